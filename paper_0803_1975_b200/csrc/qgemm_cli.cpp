// qgemm_b200 — the reference's command line front end (tools/qgemm_main.cpp:1-273)
// on the GPU path: plan inspection, file-based multiplication, cross-checking
// every algorithm against the naive product, and benchmark CSV. Same
// subcommands, options, output text and exit codes:
//   0 success, 1 verification failure, 2 usage or parse error, 3 plan infeasible.
// Every product runs through libqgemm_b200 (sm_100a kernels); the checker of
// `verify` is the library's plain naive_gemm kernel. --bits up to 53 runs the
// DoubleWord backend (FP64 tensor cores), 54..63 the Int64Word backend (uint64
// words, integer pipes), as qgemm_main.cpp:253-266 does.
#include <cerrno>
#include <chrono>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <type_traits>
#include <map>
#include <string>
#include <vector>

#include "../../include/qgemm_b200.hpp"

using namespace qgemm_b200;

namespace {

constexpr int kExitOk = 0;
constexpr int kExitVerifyFailed = 1;
constexpr int kExitUsage = 2;
constexpr int kExitInfeasible = 3;
constexpr int kDoubleBits = 53;  // DoubleWord::exact_bits, word.hpp

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

const char* kHelp =
    "compressed matrix multiplication over small prime fields (B200 GPU path)\n"
    "Usage: qgemm_b200 SUBCOMMAND [OPTIONS]\n\n"
    "Subcommands:\n"
    "  plan     show packing parameters for (p, k)\n"
    "           --p P --k K [--bits B] [--full] [--add-high-bits]\n"
    "  gemm     multiply two matrix files\n"
    "           --algo naive|common|right|left|full|blocked --a FILE --b FILE --out FILE\n"
    "           [--p P] [--bits B] [--kpanel W]\n"
    "  verify   cross-check all algorithms against the naive product\n"
    "           --p P [--max-dim D] [--seeds S] [--bits B]\n"
    "  bench    time one algorithm, CSV to stdout\n"
    "           --p P --m M --k K --n N --algo ALGO [--reps R] [--seed S] [--bits B] [--kpanel W]\n";

// Option parsing in the style the reference's CLI11 setup accepts:
// "--name value" or "--name=value", flags without a value, --help anywhere.
struct Options {
  std::map<std::string, std::string> values;
  std::vector<std::string> flags;
  bool has(const std::string& k) const { return values.count(k) != 0; }
  bool flag(const std::string& f) const {
    for (const auto& x : flags)
      if (x == f) return true;
    return false;
  }
};

Options parse_options(int argc, char** argv, int first, const std::vector<std::string>& valued,
                      const std::vector<std::string>& flag_names) {
  Options o;
  auto is = [](const std::vector<std::string>& v, const std::string& s) {
    for (const auto& x : v)
      if (x == s) return true;
    return false;
  };
  for (int i = first; i < argc; ++i) {
    std::string a = argv[i];
    if (a.rfind("--", 0) != 0) throw UsageError("The following argument was not expected: " + a);
    std::string name = a.substr(2), val;
    const auto eq = name.find('=');
    const bool inline_val = eq != std::string::npos;
    if (inline_val) {
      val = name.substr(eq + 1);
      name = name.substr(0, eq);
    }
    if (is(flag_names, name)) {
      if (inline_val) throw UsageError("--" + name + " takes no value");
      o.flags.push_back(name);
    } else if (is(valued, name)) {
      if (!inline_val) {
        if (i + 1 >= argc) throw UsageError("--" + name + ": 1 required value missing");
        val = argv[++i];
      }
      o.values[name] = val;
    } else {
      throw UsageError("The following argument was not expected: " + a);
    }
  }
  return o;
}

template <class T>
T number(const Options& o, const std::string& name, T fallback, bool required) {
  if (!o.has(name)) {
    if (required) throw UsageError("--" + name + " is required");
    return fallback;
  }
  const std::string& v = o.values.at(name);
  char* end = nullptr;
  errno = 0;
  const bool neg = !v.empty() && v[0] == '-';
  long long s = 0;
  unsigned long long u = 0;
  if (std::is_signed<T>::value) s = std::strtoll(v.c_str(), &end, 10);
  else u = std::strtoull(v.c_str(), &end, 10);
  if (v.empty() || *end != '\0' || errno || (!std::is_signed<T>::value && neg))
    throw UsageError("--" + name + ": value " + v + " is not a valid number");
  return std::is_signed<T>::value ? (T)s : (T)u;
}

Algorithm parse_algorithm(const std::string& name) {  // qgemm_main.cpp:55-64
  if (name == "naive") return Algorithm::Naive;
  if (name == "common") return Algorithm::CommonCompressed;
  if (name == "right") return Algorithm::RightCompressed;
  if (name == "left") return Algorithm::LeftCompressed;
  if (name == "full") return Algorithm::FullCompressed;
  if (name == "blocked") return Algorithm::Blocked;
  throw std::invalid_argument("unknown algorithm '" + name + "' (expected naive|common|right|left|full|blocked)");
}

void check_modulus(std::uint32_t p) {  // PrimeModulus ctor, field.hpp:19-23
  if (p < 2) throw InvalidModulus("modulus must be >= 2, got " + std::to_string(p));
  for (std::uint64_t f = 2; f * f <= p; ++f)
    if (p % f == 0) throw InvalidModulus("modulus " + std::to_string(p) + " is not prime");
}

int cmd_plan(const Options& o) {  // qgemm_main.cpp:66-97
  const auto p = number<std::uint32_t>(o, "p", 0, true);
  const auto k = number<std::uint64_t>(o, "k", 0, true);
  const int bits = number<int>(o, "bits", 53, false);
  check_modulus(p);
  const PrimeModulus mod(p);
  if (o.flag("full")) {
    const FullPlan fp = plan_full(mod, k, bits);
    std::cout << "p        " << p << "\n"
              << "k        " << k << "\n"
              << "beta     " << fp.base.beta << "\n"
              << "t        " << fp.base.t << "\n"
              << "Q        2^" << fp.base.t << "\n"
              << "dq+1     " << fp.q_slots() << "\n"
              << "dtheta+1 " << fp.theta_slots() << "\n"
              << "Theta    2^" << fp.theta_exponent << "\n"
              << "digits   " << fp.base.e << "\n"
              << "kmax     " << fp.base.kmax << "\n";
    return kExitOk;
  }
  const auto mode = o.flag("add-high-bits") ? ExtractionMode::AddHighBits : ExtractionMode::ReciprocalMul;
  const CompressionPlan plan = plan_compression(mod, k, bits, mode);
  std::cout << "p        " << p << "\n"
            << "k        " << k << "\n"
            << "beta     " << plan.beta << "\n"
            << "t        " << plan.t << "\n"
            << "Q        2^" << plan.t << "\n"
            << "d        " << plan.d << "\n"
            << "e        " << plan.e << "\n"
            << "kmax     " << plan.kmax << "\n";
  return kExitOk;
}

// One algorithm on host matrices, with the plans the reference chooses for it
// in `gemm` and `verify` (qgemm_main.cpp:118-145, verify.hpp:29-68), on the
// DoubleWord (i64 = false) or the Int64Word backend.
ResidueMatrix run_algorithm(Algorithm algo, const ResidueMatrix& a, const ResidueMatrix& b, const PrimeModulus& mod,
                            int beta, std::uint64_t kpanel, bool verify_mode, bool i64) {
  const std::uint64_t k = a.cols;
  switch (algo) {
    case Algorithm::Naive:
      return naive_gemm(a, b, mod);
    case Algorithm::CommonCompressed: {
      const CompressionPlan plan = [&] {
        try {
          return plan_compression(mod, k, beta);
        } catch (const NoCompression&) {
          if (!verify_mode || k > 1) throw;
          return uncompressed_plan(mod, k, beta);  // verify.hpp:37-44
        }
      }();
      return i64 ? mul_common_compressed<Int64Word>(a, b, plan) : mul_common_compressed(a, b, plan);
    }
    case Algorithm::RightCompressed: {
      const CompressionPlan plan = plan_packed_axis(mod, k, b.cols, beta);
      return i64 ? uncompress(mul_right_compressed<Int64Word>(a, b, plan)) : uncompress(mul_right_compressed(a, b, plan));
    }
    case Algorithm::LeftCompressed: {
      const CompressionPlan plan = plan_packed_axis(mod, k, a.rows, beta);
      return i64 ? uncompress(mul_left_compressed<Int64Word>(a, b, plan)) : uncompress(mul_left_compressed(a, b, plan));
    }
    case Algorithm::FullCompressed:
      return i64 ? mul_full_compressed<Int64Word>(a, b, plan_full(mod, k, beta))
                 : mul_full_compressed(a, b, plan_full(mod, k, beta));
    case Algorithm::Blocked: {
      std::uint64_t kp;
      if (verify_mode) {
        kp = (k + 1) / 2;  // verify.hpp:60-66: two panels
      } else {
        kp = kpanel ? kpanel : choose_panel(mod, k, beta);
        if (kp == 0) kp = k;
      }
      const CompressionPlan plan = kp >= 2 ? plan_compression(mod, kp, beta) : uncompressed_plan(mod, 1, beta);
      return i64 ? blocked_accumulate<Int64Word>(a, b, plan, kp) : blocked_accumulate(a, b, plan, kp);
    }
  }
  throw std::invalid_argument("unknown algorithm");
}

// qgemm_main.cpp:253-266: the word backend follows --bits
bool backend_i64(int bits) {
  if (bits > 63) throw std::invalid_argument("--bits must be at most 63");
  return bits > kDoubleBits;
}

int cmd_gemm(const Options& o) {  // qgemm_main.cpp:99-148
  if (!o.has("algo")) throw UsageError("--algo is required");
  for (const char* req : {"a", "b", "out"})
    if (!o.has(req)) throw UsageError(std::string("--") + req + " is required");
  const std::string a_path = o.values.at("a"), b_path = o.values.at("b"), out_path = o.values.at("out");
  const auto want_p = number<std::uint32_t>(o, "p", 0, false);
  const int beta = number<int>(o, "bits", 53, false);
  const bool i64 = backend_i64(beta);
  const auto kpanel = number<std::uint64_t>(o, "kpanel", 0, false);
  const MatrixFile fa = read_matrix_file(a_path);
  const MatrixFile fb = read_matrix_file(b_path);
  if (fa.p != fb.p)
    throw ParseError("moduli disagree: " + a_path + " has p=" + std::to_string(fa.p) + ", " + b_path +
                     " has p=" + std::to_string(fb.p));
  if (want_p != 0 && want_p != fa.p)
    throw ParseError("--p " + std::to_string(want_p) + " does not match file modulus " + std::to_string(fa.p));
  check_modulus(fa.p);
  const ResidueMatrix& a = fa.matrix;
  const ResidueMatrix& b = fb.matrix;
  if (a.cols != b.rows)
    throw DimensionMismatch("inner dimensions disagree: " + a_path + " is " + std::to_string(a.rows) + "x" +
                            std::to_string(a.cols) + ", " + b_path + " is " + std::to_string(b.rows) + "x" +
                            std::to_string(b.cols));
  const Algorithm algo = parse_algorithm(o.values.at("algo"));
  const ResidueMatrix c = run_algorithm(algo, a, b, PrimeModulus(fa.p), beta, kpanel, false, i64);
  write_matrix_file(out_path, c, fa.p);
  return kExitOk;
}

int cmd_verify(const Options& o) {  // qgemm_main.cpp:150-170, verify.hpp:70-140
  const auto p = number<std::uint32_t>(o, "p", 0, true);
  const auto max_dim = number<std::uint64_t>(o, "max-dim", 32, false);
  const auto seeds = number<std::uint64_t>(o, "seeds", 100, false);
  const int beta = number<int>(o, "bits", 53, false);
  if (beta > 63) throw std::invalid_argument("--bits must be at most 63");
  check_modulus(p);
  const PrimeModulus mod(p);
  if (max_dim < 1) throw std::invalid_argument("--max-dim must be >= 1");
  // verify.hpp:128-137: both word backends, DoubleWord at min(beta, 53),
  // Int64Word at 63 unless a wider beta was asked for
  const int beta_double = beta < kDoubleBits ? beta : kDoubleBits;
  const int beta_int = beta <= kDoubleBits ? 63 : beta;
  bool all_ok = true;
  for (Algorithm algo : {Algorithm::CommonCompressed, Algorithm::RightCompressed, Algorithm::LeftCompressed,
                         Algorithm::FullCompressed, Algorithm::Blocked})
  for (const bool i64 : {false, true}) {
    const int bb = i64 ? beta_int : beta_double;
    std::size_t cases = 0, skipped = 0;
    bool passed = true;
    std::string detail;
    for (std::uint64_t seed = 0; seed < seeds && passed; ++seed) {
      SplitMix64 dims(seed * 0x51ab1e ^ 0xfeed);
      const std::size_t m = 1 + dims.below(max_dim);
      const std::size_t k = 1 + dims.below(max_dim);
      const std::size_t n = 1 + dims.below(max_dim);
      const ResidueMatrix a = random_residue_matrix(m, k, mod, seed * 2 + 1);
      const ResidueMatrix b = random_residue_matrix(k, n, mod, seed * 2 + 2);
      ResidueMatrix got;
      try {
        got = run_algorithm(algo, a, b, mod, bb, 0, true, i64);
      } catch (const NoCompression&) {
        ++skipped;
        continue;
      }
      const ResidueMatrix want = naive_gemm(a, b, mod);
      ++cases;
      if (!(got == want)) {
        passed = false;
        for (std::size_t i = 0; i < m && detail.empty(); ++i)
          for (std::size_t j = 0; j < n && detail.empty(); ++j)
            if (got.at(i, j) != want.at(i, j))
              detail = "FAIL seed=" + std::to_string(seed) + " dims=" + std::to_string(m) + "x" +
                       std::to_string(k) + "x" + std::to_string(n) + " at (" + std::to_string(i) + "," +
                       std::to_string(j) + "): got " + std::to_string(got.at(i, j)) + " want " +
                       std::to_string(want.at(i, j));
      }
    }
    std::cout << algorithm_name(algo) << "\t" << (i64 ? "int64" : "double") << "\t";
    if (passed) {
      std::cout << "ok (" << cases << " cases";
      if (skipped) std::cout << ", " << skipped << " skipped";
      std::cout << ")\n";
    } else {
      all_ok = false;
      std::cout << detail << "\n";
    }
  }
  return all_ok ? kExitOk : kExitVerifyFailed;
}

int cmd_bench(const Options& o) {  // qgemm_main.cpp:172-182, bench.hpp:61-166
  const auto p = number<std::uint32_t>(o, "p", 0, true);
  const auto m = number<std::uint64_t>(o, "m", 0, true);
  const auto k = number<std::uint64_t>(o, "k", 0, true);
  const auto n = number<std::uint64_t>(o, "n", 0, true);
  if (!o.has("algo")) throw UsageError("--algo is required");
  const int reps = number<int>(o, "reps", 1, false);
  const auto seed = number<std::uint64_t>(o, "seed", 0, false);
  const int beta = number<int>(o, "bits", 53, false);
  const bool i64 = backend_i64(beta);
  const auto kpanel = number<std::uint64_t>(o, "kpanel", 0, false);
  check_modulus(p);
  const PrimeModulus mod(p);
  const Algorithm algo = parse_algorithm(o.values.at("algo"));
  set_phase_timing(true);  // seconds_multiply / seconds_convert per record
  const ResidueMatrix a = random_residue_matrix(m, k, mod, seed);
  const ResidueMatrix b = random_residue_matrix(k, n, mod, seed + 1);
  std::vector<TimingRecord> out;
  for (int rep = 0; rep < reps; ++rep) {
    TimingRecord rec;
    rec.algorithm = algorithm_name(algo);
    rec.p = p;
    rec.m = m;
    rec.k = k;
    rec.n = n;
    ResidueMatrix c;
    double extra_convert = 0;
    switch (algo) {
      case Algorithm::Naive:
        c = naive_gemm(a, b, mod);
        break;
      case Algorithm::CommonCompressed: {
        const CompressionPlan plan = plan_compression(mod, k, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        c = i64 ? mul_common_compressed<Int64Word>(a, b, plan) : mul_common_compressed(a, b, plan);
        break;
      }
      case Algorithm::RightCompressed:
      case Algorithm::LeftCompressed: {  // bench.hpp:108-141: plan_compression for both
        const CompressionPlan plan = plan_compression(mod, k, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        PhaseSeconds ph;
        std::chrono::steady_clock::time_point t0;
        if (i64) {
          const auto cc = algo == Algorithm::RightCompressed ? mul_right_compressed<Int64Word>(a, b, plan)
                                                             : mul_left_compressed<Int64Word>(a, b, plan);
          ph = last_phase_seconds();
          t0 = std::chrono::steady_clock::now();
          c = uncompress(cc);
        } else {
          const auto cc = algo == Algorithm::RightCompressed ? mul_right_compressed(a, b, plan)
                                                             : mul_left_compressed(a, b, plan);
          ph = last_phase_seconds();
          t0 = std::chrono::steady_clock::now();
          c = uncompress(cc);
        }
        extra_convert = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        rec.seconds_multiply = ph.multiply;
        rec.seconds_convert = ph.convert + extra_convert;
        break;
      }
      case Algorithm::FullCompressed: {
        const FullPlan fp = plan_full(mod, k, beta);
        rec.t = fp.base.t;
        rec.e = fp.base.e;
        c = i64 ? mul_full_compressed<Int64Word>(a, b, fp) : mul_full_compressed(a, b, fp);
        break;
      }
      case Algorithm::Blocked: {
        std::uint64_t kp = kpanel ? kpanel : choose_panel(mod, k, beta);
        if (kp == 0) kp = k;
        const CompressionPlan plan = kp >= 2 ? plan_compression(mod, kp, beta) : uncompressed_plan(mod, 1, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        c = i64 ? blocked_accumulate<Int64Word>(a, b, plan, kp) : blocked_accumulate(a, b, plan, kp);
        break;
      }
    }
    if (algo != Algorithm::RightCompressed && algo != Algorithm::LeftCompressed) {
      const PhaseSeconds ph = last_phase_seconds();
      rec.seconds_multiply = ph.multiply;
      rec.seconds_convert = ph.convert;
    }
    rec.checksum = residue_checksum(c);
    out.push_back(rec);
  }
  std::cout << timing_csv_header() << "\n";
  for (const auto& r : out) std::cout << to_csv_row(r) << "\n";
  return kExitOk;
}

}  // namespace

int main(int argc, char** argv) {  // qgemm_main.cpp:186-273
  for (int i = 1; i < argc; ++i)
    if (!std::strcmp(argv[i], "--help") || !std::strcmp(argv[i], "-h")) {
      std::cout << kHelp;
      return kExitOk;
    }
  if (argc < 2) {
    std::cerr << "A subcommand is required\nRun with --help for more information.\n";
    return kExitUsage;
  }
  const std::string cmd = argv[1];
  bool infeasible_hint = cmd == "gemm" || cmd == "bench";
  try {
    if (cmd == "plan") return cmd_plan(parse_options(argc, argv, 2, {"p", "k", "bits"}, {"full", "add-high-bits"}));
    if (cmd == "gemm")
      return cmd_gemm(parse_options(argc, argv, 2, {"algo", "a", "b", "out", "p", "bits", "kpanel"}, {}));
    if (cmd == "verify") return cmd_verify(parse_options(argc, argv, 2, {"p", "max-dim", "seeds", "bits"}, {}));
    if (cmd == "bench")
      return cmd_bench(parse_options(argc, argv, 2, {"p", "m", "k", "n", "algo", "reps", "seed", "bits", "kpanel"}, {}));
    std::cerr << "The following argument was not expected: " << cmd << "\nRun with --help for more information.\n";
    return kExitUsage;
  } catch (const UsageError& e) {
    std::cerr << e.what() << "\nRun with --help for more information.\n";
    return kExitUsage;
  } catch (const NoCompression& e) {
    std::cerr << "error: " << e.what() << "\n";
    if (infeasible_hint) std::cerr << "hint: --algo blocked splits the common dimension into legal panels\n";
    return kExitInfeasible;
  } catch (const PlanMismatch& e) {
    std::cerr << "error: " << e.what() << "\n"
              << "hint: --algo blocked splits the common dimension into legal panels\n";
    return kExitInfeasible;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kExitUsage;
  }
}
