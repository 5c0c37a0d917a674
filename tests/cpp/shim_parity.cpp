// Reference-style C++ test of the qgemm_b200 drop-in (include/qgemm_b200.hpp):
// the known answers of /root/reference/proj/tests/test_gemm.cpp and README,
// written against the new namespace exactly as a reference user would.
// Built by tests/test_cpp_shim.py; run on a GPU (it calls the CUDA path).
#include <cstdio>
#include <cstdlib>

#include "qgemm_b200.hpp"

using namespace qgemm_b200;

static int failures = 0;
#define CHECK(x)                                                   \
  do {                                                             \
    if (!(x)) {                                                    \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #x);     \
      ++failures;                                                  \
    }                                                              \
  } while (0)

// SplitMix64 stream of prng.hpp:12-38 (the seeded inputs of run_bench).
static ResidueMatrix random_residue_matrix(std::size_t r, std::size_t c, std::uint32_t p, std::uint64_t seed) {
  ResidueMatrix m(r, c);
  std::uint64_t s = seed;
  for (auto& v : m.data) {
    std::uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    v = static_cast<Residue>((z ^ (z >> 31)) % p);
  }
  return m;
}

static ResidueMatrix naive(const ResidueMatrix& a, const ResidueMatrix& b, std::uint32_t p) {
  ResidueMatrix c(a.rows, b.cols);
  for (std::size_t i = 0; i < a.rows; ++i)
    for (std::size_t j = 0; j < b.cols; ++j) {
      std::uint64_t s = 0;
      for (std::size_t l = 0; l < a.cols; ++l) s += std::uint64_t(a.at(i, l)) * b.at(l, j);
      c.at(i, j) = Residue(s % p);
    }
  return c;
}

static ResidueMatrix from_rows(std::size_t r, std::size_t c, std::initializer_list<Residue> v) {
  ResidueMatrix m(r, c);
  std::copy(v.begin(), v.end(), m.data.begin());
  return m;
}

int main() {
  // test_gemm.cpp:304-306, 375-377: the hand-computed 2x2 product mod 3
  const auto kA = from_rows(2, 2, {1, 2, 0, 1});
  const auto kB = from_rows(2, 2, {2, 0, 1, 1});
  const auto kC = from_rows(2, 2, {1, 2, 1, 1});
  CompressionPlan p5;  // make_plan(3, 5, 2): Q = 32
  p5.c = {3, 5, 1, 2, 53, 7, 1.0 / 32, 0};
  CHECK(mul_common_compressed(kA, kB, p5) == kC);
  CHECK(blocked_accumulate(kA, kB, p5, 1) == kC);

  // README.md:97-99: p=3, 512^3, seed 42 -> checksum 262622
  const auto a = random_residue_matrix(512, 512, 3, 42);
  const auto b = random_residue_matrix(512, 512, 3, 43);
  const auto plan = plan_compression(3, 512);
  CHECK(plan.t() == 12 && plan.e() == 4);
  const auto c = mul_common_compressed(a, b, plan);
  CHECK(residue_checksum(c) == 262622u);
  CHECK(mul_common_compressed(a, b, plan_gpu(3, 512)) == c);

  // panel blocking (test_gemm.cpp:503-523): k twice past kmax
  const auto a14 = random_residue_matrix(3, 14, 3, 31);
  const auto b14 = random_residue_matrix(14, 5, 3, 32);
  CHECK(blocked_accumulate(a14, b14, p5, 7) == naive(a14, b14, 3));
  bool threw = false;
  try {
    blocked_accumulate(a14, b14, p5, 8);
  } catch (const PlanMismatch&) {
    threw = true;
  }
  CHECK(threw);

  // k beyond any single plan: the GPU planner blocks it (p=7, k=4096)
  const auto a7 = random_residue_matrix(64, 4096, 7, 5);
  const auto b7 = random_residue_matrix(4096, 48, 7, 6);
  CHECK(mul_common_compressed(a7, b7, plan_gpu(7, 4096)) == naive(a7, b7, 7));

  // right compression (test_gemm.cpp:417-443): CB = [[2],[33]], C = kC
  const auto cc = mul_right_compressed(kA, kB, p5);
  // C = kC: row 0 digits (1, 2) -> 1 + 2*32 = 65; row 1 digits (1, 1) -> 33
  CHECK(cc.stored_cols == 1 && cc.data[0] == 65.0 && cc.data[1] == 33.0);

  // errors: invalid modulus, dimension mismatch
  threw = false;
  try {
    plan_compression(4, 10);
  } catch (const InvalidModulus&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    mul_common_compressed(ResidueMatrix(2, 3), ResidueMatrix(2, 3), p5);
  } catch (const DimensionMismatch&) {
    threw = true;
  }
  CHECK(threw);

  if (failures) std::printf("shim_parity: %d FAILED\n", failures);
  else std::printf("shim_parity: all passed\n");
  return failures ? 1 : 0;
}
