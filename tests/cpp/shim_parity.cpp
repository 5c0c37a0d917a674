// Reference-style C++ test of the qgemm_b200 drop-in (include/qgemm_b200.hpp):
// the known answers of /root/reference/proj/tests/test_gemm.cpp and README,
// written against the new namespace exactly as a reference user would, plus
// the B200 additions (GPU plans, the multi-device entry, residue-in right /
// left products). tests/cpp/dropin_parity.cpp is the same-source comparison
// with the reference itself.
// Built by tests/test_cpp_shim.py; run on a GPU (it calls the CUDA path).
#include <cstdio>
#include <cstdlib>
#include <string>

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

// SplitMix64 stream of prng.hpp:12-38 (the seeded inputs of run_bench), on the host.
static ResidueMatrix host_random_matrix(std::size_t r, std::size_t c, std::uint32_t p, std::uint64_t seed) {
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

static ResidueMatrix host_naive(const ResidueMatrix& a, const ResidueMatrix& b, std::uint32_t p) {
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
  CompressionPlan p5{PrimeModulus(3)};  // make_plan(3, 5, 2): Q = 32
  p5.t = 5;
  p5.d = 1;
  p5.e = 2;
  p5.kmax = 7;
  p5.inv_qd = 1.0 / 32;
  const PrimeModulus m3(3), m7(7);
  CHECK(mul_common_compressed(kA, kB, p5) == kC);
  CHECK(blocked_accumulate(kA, kB, p5, 1) == kC);

  // README.md:97-99: p=3, 512^3, seed 42 -> checksum 262622
  const auto a = host_random_matrix(512, 512, 3, 42);
  const auto b = host_random_matrix(512, 512, 3, 43);
  CHECK(random_residue_matrix(512, 512, m3, 42) == a);  // the device generator, same stream
  const auto plan = plan_compression(m3, 512);
  CHECK(plan.t == 12 && plan.e == 4);
  const auto c = mul_common_compressed(a, b, plan);
  CHECK(residue_checksum(c) == 262622u);
  CHECK(mul_common_compressed(a, b, plan_gpu(m3, 512)) == c);
  CHECK(mul_common_compressed(a, b, plan_gpu(m3, 512), std::vector<int>{0}) == c);  // one-process multi-GPU entry

  // panel blocking (test_gemm.cpp:503-523): k twice past kmax
  const auto a14 = host_random_matrix(3, 14, 3, 31);
  const auto b14 = host_random_matrix(14, 5, 3, 32);
  CHECK(blocked_accumulate(a14, b14, p5, 7) == host_naive(a14, b14, 3));
  bool threw = false;
  try {
    blocked_accumulate(a14, b14, p5, 8);
  } catch (const PlanMismatch&) {
    threw = true;
  }
  CHECK(threw);

  // k beyond any single plan: the GPU planner blocks it (p=7, k=4096)
  const auto a7 = host_random_matrix(64, 4096, 7, 5);
  const auto b7 = host_random_matrix(4096, 48, 7, 6);
  CHECK(mul_common_compressed(a7, b7, plan_gpu(m7, 4096)) == host_naive(a7, b7, 7));

  // right compression (test_gemm.cpp:417-443): CB = [[2],[33]], C = kC
  const auto cc = mul_right_compressed(kA, kB, p5);
  // C = kC: row 0 digits (1, 2) -> 1 + 2*32 = 65; row 1 digits (1, 1) -> 33
  CHECK(cc.stored_cols == 1 && cc.data[0].value == 65.0 && cc.data[1].value == 33.0);

  CHECK(uncompress(cc) == kC);

  // left compression (test_gemm.cpp:177-199): CC digits [1,1] and [2,1]
  const auto cl = mul_left_compressed(kA, kB, p5);
  CHECK(cl.stored_rows == 1 && cl.data[0].value == 33.0 && cl.data[1].value == 34.0);
  CHECK(uncompress(cl) == kC);
  CHECK(uncompress(mul_left_compressed(kA, from_rows(2, 2, {1, 0, 0, 1}), p5)) == kA);

  // full compression (test_gemm.cpp:201-214): dq = dtheta = 1, Q = 32, Theta = 2^10
  CompressionPlan p54 = p5;  // make_plan(3, 5, 4)
  p54.d = 3;
  p54.e = 4;
  p54.inv_qd = 1.0 / 32768;
  FullPlan fp{p54, 1, 1, 10};
  CHECK(mul_full_compressed(kA, kB, fp) == kC);
  CHECK(mul_full_compressed(ResidueMatrix(2, 2), kB, fp) == ResidueMatrix(2, 2));
  const auto f250 = plan_full(m3, 250);  // test_plan.cpp:96-104
  CHECK(f250.base.t == 10 && f250.q_slots() == 2 && f250.theta_slots() == 2 && f250.theta_exponent == 20);
  CHECK(mul_full_compressed(a14, b14, plan_full(m3, 14)) == host_naive(a14, b14, 3));

  // naive_gemm on the device
  CHECK(naive_gemm(kA, kB, m3) == kC);
  CHECK(naive_gemm(a7, b7, m7) == host_naive(a7, b7, 7));

  // matrix files (test_io.cpp:11-37) and timing CSV rows (test_io.cpp:44-55)
  const std::string path = "/tmp/qgemm_b200_shim.mtx";
  write_matrix_file(path, a14, 3);
  const MatrixFile mf = read_matrix_file(path);
  CHECK(mf.p == 3 && mf.matrix == a14);
  threw = false;
  try {
    read_matrix_text("M 3 1 2\n0 3\n");
  } catch (const ParseError&) {
    threw = true;
  }
  CHECK(threw);
  CHECK(std::string(timing_csv_header()) == "algorithm,p,m,k,n,t,e,seconds_multiply,seconds_convert,checksum");
  TimingRecord r;
  r.algorithm = "common";
  r.p = 3; r.m = 4; r.k = 5; r.n = 6; r.t = 7; r.e = 2;
  r.seconds_multiply = 0.25;
  r.seconds_convert = 0.125;
  r.checksum = 99;
  CHECK(to_csv_row(r) == "common,3,4,5,6,7,2,0.250000,0.125000,99");
  CHECK(std::string(algorithm_name(Algorithm::FullCompressed)) == "full");

  // Int64Word backend (word.hpp:36-54) at beta = 63: same C, reference words
  const auto p63 = plan_compression(m3, 14, 63);
  CHECK(mul_common_compressed<Int64Word>(a14, b14, p63) == host_naive(a14, b14, 3));
  CHECK(blocked_accumulate<Int64Word>(a14, b14, plan_compression(m3, 7, 63), 7) == host_naive(a14, b14, 3));
  CHECK(uncompress(mul_right_compressed<Int64Word>(a14, b14, plan_packed_axis(m3, 14, 5, 63))) == host_naive(a14, b14, 3));
  CHECK(uncompress(mul_left_compressed<Int64Word>(a14, b14, plan_packed_axis(m3, 14, 3, 63))) == host_naive(a14, b14, 3));
  CHECK(mul_full_compressed<Int64Word>(a14, b14, plan_full(m3, 14, 63)) == host_naive(a14, b14, 3));
  const auto l64 = mul_left_compressed<Int64Word>(kA, kB, p5);  // test_gemm.cpp:183-185 for Int64Word
  CHECK(l64.data[0].value == 33u && l64.data[1].value == 34u);

  // errors: invalid modulus, dimension mismatch
  threw = false;
  try {
    plan_compression(PrimeModulus(4), 10);
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
