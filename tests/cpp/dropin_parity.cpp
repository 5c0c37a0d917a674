// dropin_parity.cpp — ONE reference-style program compiled twice:
//   g++ -std=c++20 -I/root/reference/proj/include dropin_parity.cpp           (namespace qgemm, the reference)
//   g++ -std=c++20 -DQG_B200 -Iinclude dropin_parity.cpp -lqgemm_b200         (namespace qgemm_b200, the GPU drop-in)
// Both builds must print byte-identical output (tests/test_cpp_shim.py; the
// reference's output is committed as tests/golden/dropin_parity.txt, made by
// tests/golden/make_dropin_golden.sh). Only the namespace switch differs: the
// body uses the reference's own types and signatures (field.hpp, plan.hpp,
// word.hpp, matrix.hpp, pack.hpp, gemm.hpp, prng.hpp, bench.hpp, verify.hpp,
// matrix_io.hpp), the way the reference's tests do (test_pack.cpp,
// test_gemm.cpp, acceptance.cpp). Exceptions are printed by class, results as
// FNV-1a hashes of their raw words / residues plus a few leading values.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <functional>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

#ifdef QG_B200
#include "qgemm_b200.hpp"
namespace Q = qgemm_b200;
#else
#include "qgemm/qgemm.hpp"
namespace Q = qgemm;
#endif
using namespace Q;

namespace {

std::uint64_t fnv(const void* p, std::size_t n, std::uint64_t h = 1469598103934665603ull) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (std::size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 1099511628211ull;
  return h;
}

template <class B>
std::uint64_t u64(PackedWord<B> w) {
  return B::to_u64(w.value);
}

template <class B>
std::string words(const std::vector<PackedWord<B>>& v) {
  std::uint64_t h = 1469598103934665603ull;
  for (const auto& w : v) {
    const std::uint64_t x = u64(w);
    h = fnv(&x, 8, h);
  }
  std::ostringstream os;
  os << "n=" << v.size() << " fnv=" << std::hex << h << std::dec << " head=";
  for (std::size_t i = 0; i < v.size() && i < 4; ++i) os << u64(v[i]) << (i + 1 < 4 && i + 1 < v.size() ? "," : "");
  return os.str();
}

template <class B>
std::string cm(const CompressedMatrix<B>& c) {
  std::ostringstream os;
  os << c.logical_rows << "x" << c.logical_cols << " stored " << c.stored_rows << "x" << c.stored_cols << " dir "
     << (c.orientation.direction == PackDirection::Reversed ? "R" : "F") << " axis "
     << (c.orientation.axis == PackAxis::Column ? "C" : "R") << " slots " << c.orientation.slots << " t "
     << c.plan.t << " e " << c.plan.e << " " << words(c.data);
  return os.str();
}

std::string rm(const ResidueMatrix& m) {
  std::ostringstream os;
  os << m.rows << "x" << m.cols << " fnv=" << std::hex << fnv(m.data.data(), m.data.size() * 4) << std::dec
     << " checksum=" << residue_checksum(m);
  return os.str();
}

std::string plan_str(const CompressionPlan& p) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%a", p.inv_qd);
  std::ostringstream os;
  os << "p=" << p.p() << " t=" << p.t << " d=" << p.d << " e=" << p.e << " beta=" << p.beta << " kmax=" << p.kmax
     << " inv_qd=" << buf << " mode=" << (p.extraction == ExtractionMode::AddHighBits ? "AHB" : "RM")
     << " q=" << p.q() << " qmask=" << p.q_mask();
  return os.str();
}

// Runs f, printing "label: <result>" or "label: throws <Class>".
void show(const std::string& label, const std::function<std::string()>& f) {
  std::string r;
  try {
    r = f();
  } catch (const InvalidModulus&) {
    r = "throws InvalidModulus";
  } catch (const NoCompression&) {
    r = "throws NoCompression";
  } catch (const SlotOverflow&) {
    r = "throws SlotOverflow";
  } catch (const DigitOverflow&) {
    r = "throws DigitOverflow";
  } catch (const DimensionMismatch&) {
    r = "throws DimensionMismatch";
  } catch (const PlanMismatch&) {
    r = "throws PlanMismatch";
  } catch (const UnsupportedAlgorithm&) {
    r = "throws UnsupportedAlgorithm";
  } catch (const ParseError&) {
    r = "throws ParseError";
  } catch (const std::invalid_argument&) {
    r = "throws invalid_argument";
  } catch (const std::exception& ex) {
    r = std::string("throws other: ") + ex.what();
  }
  std::cout << label << ": " << r << "\n";
}

// Hand-built plan, as the reference's tests build them (test_pack.cpp:15-24).
CompressionPlan make_plan(std::uint32_t p, int t, int e, int beta = 53) {
  CompressionPlan plan{PrimeModulus(p)};
  plan.t = t;
  plan.e = e;
  plan.d = e - 1;
  plan.beta = beta;
  plan.kmax = ((std::uint64_t{1} << t) - 1) / plan.modulus.pm1_squared();
  plan.inv_qd = std::ldexp(1.0, -t * plan.d);
  return plan;
}

template <class B>
void backend_suite(const char* name, int beta) {
  std::cout << "== backend " << name << "\n";
  const PrimeModulus m3(3), m5(5), m7(7);
  // scalar packing, pack.hpp:47-155
  const auto plan = make_plan(3, 5, 3, beta);  // Q = 32
  const Residue v12[] = {1, 2}, v210[] = {2, 1, 0}, v4[] = {1, 1, 1, 1}, v121[] = {1, 2, 1};
  show("compress_forward {1,2}", [&] { return std::to_string(u64(compress_forward<B>({v12, 2}, plan))); });
  show("compress_forward {}", [&] { return std::to_string(u64(compress_forward<B>({}, plan))); });
  show("compress_forward {2,1,0}", [&] { return std::to_string(u64(compress_forward<B>({v210, 3}, plan))); });
  show("compress_forward x4", [&] { return std::to_string(u64(compress_forward<B>({v4, 4}, plan))); });
  show("compress_reverse {1,2,1}", [&] { return std::to_string(u64(compress_reverse<B>({v121, 3}, plan))); });
  show("compress_reverse {1,2}", [&] { return std::to_string(u64(compress_reverse<B>({v12, 2}, plan))); });
  show("compress_reverse x4", [&] { return std::to_string(u64(compress_reverse<B>({v4, 4}, plan))); });
  const auto p2 = make_plan(3, 5, 2, beta);
  const auto w = mul(compress_reverse<B>({v12, 2}, p2), compress_forward<B>({v12, 2}, p2));
  show("extract_coefficient", [&] { return std::to_string(extract_coefficient(w, p2)); });
  show("extract_all", [&] {
    std::string s;
    for (auto d : extract_all(PackedWord<B>{B::from_u64(33 + 2 * 32 * 32)}, plan)) s += std::to_string(d) + ",";
    return s;
  });
  show("extract_all overflow", [&] { return std::to_string(extract_all(PackedWord<B>{B::from_u64(1u << 15)}, plan).size()); });
  show("redq", [&] { return std::to_string(u64(redq(PackedWord<B>{B::from_u64(31 + 17 * 32 + 4 * 1024)}, plan))); });
  show("redq overflow", [&] { return std::to_string(u64(redq(PackedWord<B>{B::from_u64(1u << 15)}, plan))); });
  show("reduce_and_compress", [&] {
    std::vector<PackedWord<B>> row;
    for (int i = 0; i < 7; ++i) row.push_back(PackedWord<B>{B::from_u64((std::uint64_t)(i * 3 + 1) << 5)});
    return words(reduce_and_compress(std::span<const PackedWord<B>>(row), p2));
  });
  show("reduce_common_entry", [&] { return std::to_string(reduce_common_entry(PackedWord<B>{B::from_u64(70)}, plan)); });

  // matrix layouts, gemm.hpp:104-204
  const ResidueMatrix a = random_residue_matrix(37, 53, m3, 42);
  const ResidueMatrix b = random_residue_matrix(53, 29, m3, 43);
  const auto pl = plan_compression(m3, 53, beta);
  std::cout << "plan " << plan_str(pl) << "\n";
  const auto ca = compress_rows_reversed<B>(a, pl);
  const auto cb = compress_cols_forward<B>(b, pl);
  std::cout << "compress_rows_reversed " << cm(ca) << "\n";
  std::cout << "compress_cols_forward " << cm(cb) << "\n";
  std::cout << "compress_outer_cols " << cm(compress_outer_cols<B>(b, pl)) << "\n";
  std::cout << "compress_outer_rows " << cm(compress_outer_rows<B>(a, pl)) << "\n";
  show("uncompress(rows_reversed)", [&] { return rm(uncompress(ca)); });
  show("uncompress(cols_forward)", [&] { return rm(uncompress(cb)); });
  show("packed_common_product", [&] { return words(packed_common_product(ca, cb)); });
  show("mul_common_compressed(ca,cb)", [&] { return rm(mul_common_compressed(ca, cb)); });
  show("mul_common_compressed(a,b,plan)", [&] { return rm(mul_common_compressed<B>(a, b, pl)); });
  show("naive_gemm", [&] { return rm(naive_gemm(a, b, m3)); });
  show("mul_common_repacked", [&] { return cm(mul_common_repacked<B>(a, b, pl)); });
  show("reduce_common_entry loop", [&] {
    const auto acc = packed_common_product(ca, cb);
    ResidueMatrix c(a.rows, b.cols);
    for (std::size_t i = 0; i < acc.size(); ++i) c.data[i] = reduce_common_entry(acc[i], pl);
    return rm(c);
  });
  // argument checks in the reference's order
  show("packed_common_product swapped", [&] { return words(packed_common_product(cb, ca)); });
  show("packed_common_product other plan", [&] {
    const auto cb2 = compress_cols_forward<B>(b, make_plan(3, 10, 3, beta));
    return words(packed_common_product(ca, cb2));
  });
  show("compress_rows_reversed k>kmax", [&] { return cm(compress_rows_reversed<B>(random_residue_matrix(2, 600, m3, 1), pl)); });
  show("mul_common_compressed dims", [&] { return rm(mul_common_compressed<B>(a, a, pl)); });

  // mixed variant, gemm.hpp:285-335
  const auto pr = plan_packed_axis(m5, 64, 50, beta);
  std::cout << "plan_packed_axis " << plan_str(pr) << "\n";
  const ResidueMatrix ar = random_residue_matrix(21, 64, m5, 7);
  const ResidueMatrix br = random_residue_matrix(64, 50, m5, 8);
  const auto cbo = compress_outer_cols<B>(br, pr);
  show("packed_right_product", [&] { return cm(packed_right_product(ar, cbo)); });
  show("redq_in_place", [&] {
    auto cc = packed_right_product(ar, cbo);
    redq_in_place(cc);
    return cm(cc);
  });
  show("mul_right_compressed(a,cb)", [&] { return cm(mul_right_compressed(ar, cbo)); });
  show("uncompress(mul_right)", [&] { return rm(uncompress(mul_right_compressed(ar, cbo))); });
  show("naive_gemm(right)", [&] { return rm(naive_gemm(ar, br, m5)); });
  show("mul_right_compressed(ca,cb)", [&] {
    const auto cao = compress_outer_cols<B>(ar, pr);  // a Forward operand, unpacked first
    return cm(mul_right_compressed(cao, cbo));
  });
  show("mul_right_compressed(reversed ca)", [&] {
    const auto car = compress_rows_reversed<B>(ar, pr);
    return cm(mul_right_compressed(car, cbo));
  });
  show("packed_right_product wrong orientation", [&] { return cm(packed_right_product(ar, compress_cols_forward<B>(br, pr))); });
  show("packed_right_product dims", [&] { return cm(packed_right_product(br, cbo)); });

  // left variant, gemm.hpp:340-371
  const auto plft = plan_packed_axis(m7, 40, 30, beta);
  const ResidueMatrix al = random_residue_matrix(30, 40, m7, 9);
  const ResidueMatrix bl = random_residue_matrix(40, 17, m7, 10);
  const auto cao = compress_outer_rows<B>(al, plft);
  show("packed_left_product", [&] { return cm(packed_left_product(cao, bl)); });
  show("mul_left_compressed", [&] { return cm(mul_left_compressed(cao, bl)); });
  show("uncompress(mul_left)", [&] { return rm(uncompress(mul_left_compressed(cao, bl))); });
  show("naive_gemm(left)", [&] { return rm(naive_gemm(al, bl, m7)); });
  show("packed_left_product wrong orientation", [&] { return cm(packed_left_product(compress_outer_cols<B>(al, plft), bl)); });

  // full compression, gemm.hpp:377-445
  show("plan_full", [&] {
    const auto fp = plan_full(m3, 100, beta);
    return plan_str(fp.base) + " dq=" + std::to_string(fp.dq) + " dtheta=" + std::to_string(fp.dtheta) +
           " theta=" + std::to_string(fp.theta_exponent) + " qs=" + std::to_string(fp.q_slots()) + " ts=" +
           std::to_string(fp.theta_slots());
  });
  show("mul_full_compressed", [&] {
    const ResidueMatrix af = random_residue_matrix(23, 100, m3, 11), bf = random_residue_matrix(100, 31, m3, 12);
    PhaseSeconds ph;
    const auto c = mul_full_compressed<B>(af, bf, plan_full(m3, 100, beta), &ph);
    return rm(c) + (c == naive_gemm(af, bf, m3) ? " ==naive" : " !=naive");
  });
  show("mul_full_compressed hand plan", [&] {
    FullPlan fp{make_plan(3, 5, 4, beta), 1, 1, 10};  // test_gemm.cpp:203
    const ResidueMatrix af = random_residue_matrix(9, 7, m3, 13), bf = random_residue_matrix(7, 11, m3, 14);
    return rm(mul_full_compressed<B>(af, bf, fp));
  });

  // blocked accumulation, gemm.hpp:450-489
  show("blocked_accumulate", [&] {
    const ResidueMatrix ab = random_residue_matrix(19, 1000, m7, 15), bb = random_residue_matrix(1000, 23, m7, 16);
    const auto pb = plan_compression(m7, 100, beta);
    PhaseSeconds ph;
    const auto c = blocked_accumulate<B>(ab, bb, pb, 100, &ph);
    return rm(c) + (c == naive_gemm(ab, bb, m7) ? " ==naive" : " !=naive");
  });
  show("blocked_accumulate kpanel 0", [&] { return rm(blocked_accumulate<B>(a, b, pl, 0)); });

  // empty and degenerate shapes (value semantics must hold at the edges)
  const ResidueMatrix e0(0, 53), e1(53, 0), e2(0, 0);
  show("compress_rows_reversed 0 rows", [&] { return cm(compress_rows_reversed<B>(e0, pl)); });
  show("compress_cols_forward 0 cols", [&] { return cm(compress_cols_forward<B>(e1, pl)); });
  show("mul_common_compressed 0 x 53 x 29", [&] { return rm(mul_common_compressed<B>(e0, b, pl)); });
  show("mul_common_compressed 37 x 53 x 0", [&] { return rm(mul_common_compressed<B>(a, e1, pl)); });
  show("packed_common_product empty", [&] {
    return words(packed_common_product(compress_rows_reversed<B>(e0, pl), compress_cols_forward<B>(b, pl)));
  });
  show("mul_right_compressed 0 rows", [&] { return cm(mul_right_compressed(ResidueMatrix(0, 64), cbo)); });
  show("uncompress empty", [&] { return rm(uncompress(compress_outer_cols<B>(e2, pr))); });
  show("mul_common_repacked 0 x 53", [&] { return cm(mul_common_repacked<B>(e0, b, pl)); });
  show("k = 1 uncompressed plan", [&] {
    const ResidueMatrix a1 = random_residue_matrix(9, 1, m3, 17), b1 = random_residue_matrix(1, 11, m3, 18);
    return rm(mul_common_compressed<B>(a1, b1, uncompressed_plan(m3, 1, beta)));
  });
  show("one row, one column", [&] {
    const ResidueMatrix a1 = random_residue_matrix(1, 40, m7, 19), b1 = random_residue_matrix(40, 1, m7, 20);
    return rm(mul_common_compressed<B>(a1, b1, plan_compression(m7, 40, beta)));
  });
  show("ragged k (k % e != 0)", [&] {
    const ResidueMatrix a1 = random_residue_matrix(13, 41, m5, 21), b1 = random_residue_matrix(41, 17, m5, 22);
    const auto p41 = plan_compression(m5, 41, beta);
    return rm(mul_common_compressed(compress_rows_reversed<B>(a1, p41), compress_cols_forward<B>(b1, p41))) +
           " e=" + std::to_string(p41.e);
  });
  show("blocked_accumulate kpanel>kmax", [&] { return rm(blocked_accumulate<B>(a, b, pl, pl.kmax + 1)); });
}

}  // namespace

int main() {
  std::cout << "== field\n";
  const PrimeModulus m7(7);
  std::cout << "PrimeModulus(7) value=" << m7.value() << " pm1sq=" << m7.pm1_squared() << " reduce(100)="
            << m7.reduce(100) << " addmul(3,4,5)=" << m7.addmul(3, 4, 5) << " eq=" << (m7 == PrimeModulus(7))
            << " prime(91)=" << PrimeModulus::is_prime(91) << "\n";
  show("PrimeModulus(8)", [] { return std::to_string(PrimeModulus(8).value()); });
  show("PrimeModulus(1)", [] { return std::to_string(PrimeModulus(1).value()); });

  std::cout << "== planners\n";
  for (auto [p, k] : std::vector<std::pair<std::uint32_t, std::uint64_t>>{
           {3, 512}, {7, 4096}, {3, 256}, {5, 8192}, {3, 32768}, {2, 1}, {251, 4}, {3, 1}}) {
    const std::string tag = "(" + std::to_string(p) + "," + std::to_string(k) + ")";
    show("plan_compression" + tag, [&] { return plan_str(plan_compression(PrimeModulus(p), k)); });
    show("plan_compression AHB" + tag,
         [&] { return plan_str(plan_compression(PrimeModulus(p), k, 53, ExtractionMode::AddHighBits)); });
    show("uncompressed_plan" + tag, [&] { return plan_str(uncompressed_plan(PrimeModulus(p), k)); });
    show("plan_packed_axis" + tag, [&] { return plan_str(plan_packed_axis(PrimeModulus(p), k, 3)); });
    show("choose_panel" + tag, [&] { return std::to_string(choose_panel(PrimeModulus(p), k)); });
    show("plan_full" + tag, [&] { return plan_str(plan_full(PrimeModulus(p), k).base); });
  }
  show("plan_compression k=0", [] { return plan_str(plan_compression(PrimeModulus(3), 0)); });
  show("plan_compression beta=1", [] { return plan_str(plan_compression(PrimeModulus(3), 4, 1)); });
  show("plan_compression beta=63", [] { return plan_str(plan_compression(PrimeModulus(3), 32768, 63)); });
  std::cout << "algorithm_name " << algorithm_name(Algorithm::CommonCompressed) << " "
            << algorithm_name(Algorithm::Blocked) << "\n";

  std::cout << "== prng\n";
  SplitMix64 rng(42);
  std::cout << "SplitMix64(42) " << rng.next() << " " << rng.next() << " below(7)=" << rng.below(7) << "\n";
  std::cout << "random_residue_matrix " << rm(random_residue_matrix(31, 17, PrimeModulus(5), 3)) << "\n";
  std::cout << "config1 checksum "
            << residue_checksum(mul_common_compressed(random_residue_matrix(512, 512, PrimeModulus(3), 42),
                                                      random_residue_matrix(512, 512, PrimeModulus(3), 43),
                                                      plan_compression(PrimeModulus(3), 512)))
            << "\n";  // README.md:97-99: 262622

  backend_suite<DoubleWord>("double", 53);
  backend_suite<Int64Word>("int64", 63);

  std::cout << "== matrix_io\n";
  {
    std::istringstream in("M 5 2 3\n1 2 3\n4 0 1\n");
    const MatrixFile mf = read_matrix(in);
    std::ostringstream out;
    write_matrix(out, mf.matrix, mf.p);
    std::cout << "roundtrip p=" << mf.p << " " << rm(mf.matrix) << " text=" << out.str().size() << "B\n";
    show("read_matrix bad header", [] {
      std::istringstream bad("X 5 2 3\n");
      return rm(read_matrix(bad).matrix);
    });
    show("read_matrix out of range", [] {
      std::istringstream bad("M 5 1 2\n1 7\n");
      return rm(read_matrix(bad).matrix);
    });
    show("read_matrix trailing", [] {
      std::istringstream bad("M 5 1 1\n1 2\n");
      return rm(read_matrix(bad).matrix);
    });
  }

  std::cout << "== bench / verify\n";
  TimingRecord r;
  r.algorithm = "common";
  r.p = 3;
  r.m = r.k = r.n = 4;
  r.t = 12;
  r.e = 4;
  r.seconds_multiply = 0.5;
  r.seconds_convert = 0.25;
  r.checksum = 99;
  std::cout << timing_csv_header() << "\n" << to_csv_row(r) << "\n";
  for (Algorithm algo : {Algorithm::Naive, Algorithm::CommonCompressed, Algorithm::RightCompressed,
                         Algorithm::LeftCompressed, Algorithm::FullCompressed, Algorithm::Blocked}) {
    show(std::string("run_bench ") + algorithm_name(algo), [&] {
      const auto recs = run_bench<DoubleWord>(algo, PrimeModulus(3), 64, 96, 48, 2, 42);
      std::string s;
      for (const auto& rec : recs)
        s += rec.algorithm + " t=" + std::to_string(rec.t) + " e=" + std::to_string(rec.e) +
             " checksum=" + std::to_string(rec.checksum) + "; ";
      return s;
    });
  }
  for (const auto& v : run_verify(PrimeModulus(5), 12, 6))
    std::cout << "verify " << algorithm_name(v.algorithm) << " " << v.backend << " cases=" << v.cases
              << " skipped=" << v.skipped << " passed=" << v.passed << "\n";
  std::cout << "done\n";
  return 0;
}
