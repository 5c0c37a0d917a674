// qgemm_b200.hpp — C++ drop-in for the reference's header API (namespace
// qgemm, /root/reference/proj/include/qgemm/*.hpp), implemented over the C
// ABI (qgemm_b200.h) and therefore over the sm_100a kernels. Header-only;
// link with -lqgemm_b200 (paper_0803_1975_b200/_lib).
//
// Same types (field, public members, aggregate layout), same function
// signatures, same argument checks in the same order and the same exception
// classes as the reference, so reference-style code switches by replacing
//     #include "qgemm/qgemm.hpp"     using namespace qgemm;
// with
//     #include "qgemm_b200.hpp"      using namespace qgemm_b200;
// (tests/cpp/dropin_parity.cpp is one source compiled both ways and must
// print identical results; INTEGRATION.md lists every entry point with its
// reference file:line).
//
// Where the work happens: every matrix-level operation (packing, the packed
// products, REDQ, extraction, unpacking, the naive product, seeded input
// generation) runs in the library's CUDA kernels — the header copies operands
// to the device, calls the C ABI and copies results back, preserving the
// reference's value semantics. The single-word helpers of pack.hpp
// (compress_forward/reverse, extract_coefficient, extract_all, redq,
// reduce_and_compress) run the same kernels on one word or row. Only the
// field/word type members (PrimeModulus::reduce, DoubleWord::high_part, ...)
// and reduce_common_entry, which is PrimeModulus::reduce of a masked word,
// are inline scalar code, as in the reference's own headers.
//
// B200 additions (not in the reference): GpuPlan / plan_gpu (k-blocked plans
// for the FP64 tensor-core contraction), mul_common_compressed(a, b, GpuPlan
// [, devices]), mul_right_compressed / mul_left_compressed(a, b, plan) on
// residues, set_phase_timing / last_phase_seconds.
#pragma once

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iomanip>
#include <istream>
#include <iterator>
#include <optional>
#include <ostream>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <type_traits>
#include <vector>

#include "qgemm_b200.h"

namespace qgemm_b200 {

// ------------------------------------------------------------ errors.hpp:8-34
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct InvalidModulus : Error { using Error::Error; };
struct NoCompression : Error { using Error::Error; };
struct SlotOverflow : Error { using Error::Error; };
struct DigitOverflow : Error { using Error::Error; };
struct DimensionMismatch : Error { using Error::Error; };
struct PlanMismatch : Error { using Error::Error; };
struct UnsupportedAlgorithm : Error { using Error::Error; };
struct ParseError : Error { using Error::Error; };
struct DeviceError : Error { using Error::Error; };  // CUDA / NCCL failures (no reference analogue)

namespace detail {
inline void check(int status, const char* where) {
  if (status == QG_OK) return;
  std::string msg = std::string(where) + ": " + qg_status_string(status);
  if (status == QG_CUDA_ERROR || status == QG_NCCL_ERROR || status == QG_PARSE_ERROR)
    msg += std::string(" (") + qg_last_error() + ")";
  switch (status) {
    case QG_INVALID_MODULUS: throw InvalidModulus(msg);
    case QG_NO_COMPRESSION: throw NoCompression(msg);
    case QG_SLOT_OVERFLOW: throw SlotOverflow(msg);
    case QG_DIGIT_OVERFLOW: throw DigitOverflow(msg);
    case QG_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case QG_PLAN_MISMATCH: throw PlanMismatch(msg);
    case QG_UNSUPPORTED_ALGORITHM: throw UnsupportedAlgorithm(msg);
    case QG_PARSE_ERROR: throw ParseError(msg);
    case QG_INVALID_ARGUMENT: throw std::invalid_argument(msg);
    case QG_NOT_EXACT: throw PlanMismatch(msg);
    default: throw DeviceError(msg);
  }
}
}  // namespace detail

// ------------------------------------------------------------ field.hpp:12-53
using Residue = std::uint32_t;

class PrimeModulus {
 public:
  explicit PrimeModulus(std::uint32_t p) : p_(p) {
    if (p < 2 || !is_prime(p)) throw InvalidModulus("modulus " + std::to_string(p) + " is not prime");
    pm1sq_ = static_cast<std::uint64_t>(p - 1) * (p - 1);
  }
  std::uint32_t value() const { return p_; }
  std::uint64_t pm1_squared() const { return pm1sq_; }
  Residue reduce(std::uint64_t x) const { return static_cast<Residue>(x % p_); }
  Residue addmul(Residue acc, Residue a, Residue b) const { return reduce(acc + static_cast<std::uint64_t>(a) * b); }
  friend bool operator==(const PrimeModulus&, const PrimeModulus&) = default;
  static bool is_prime(std::uint64_t n) {
    if (n < 2) return false;
    if (n % 2 == 0) return n == 2;
    for (std::uint64_t f = 3; f * f <= n; f += 2)
      if (n % f == 0) return false;
    return true;
  }

 private:
  std::uint32_t p_;
  std::uint64_t pm1sq_;
};

// ------------------------------------------------------------ word.hpp:10-80
struct DoubleWord {
  using value_type = double;
  static constexpr int exact_bits = 53;
  static value_type from_u64(std::uint64_t x) { return static_cast<value_type>(x); }
  static std::uint64_t to_u64(value_type v) { return static_cast<std::uint64_t>(v); }
  struct HighPart {
    double inv_qd;
    std::uint64_t q_mask;
  };
  static value_type high_part(value_type a, value_type b, const HighPart& ctx) {
    return static_cast<value_type>(static_cast<std::int64_t>(a * b * ctx.inv_qd));
  }
};
struct Int64Word {
  using value_type = std::uint64_t;
  static constexpr int exact_bits = 63;
  static value_type from_u64(std::uint64_t x) { return x; }
  static std::uint64_t to_u64(value_type v) { return v; }
  struct HighPart {
    int shift;
    std::uint64_t q_mask;
  };
  static value_type high_part(value_type a, value_type b, const HighPart& ctx) {
    return ((a * b) >> ctx.shift) & ctx.q_mask;
  }
};
template <class B>
struct PackedWord {
  using backend = B;
  typename B::value_type value{};
  friend bool operator==(const PackedWord&, const PackedWord&) = default;
};
template <class B>
PackedWord<B> mul(PackedWord<B> a, PackedWord<B> b) {
  return {a.value * b.value};
}
template <class B>
PackedWord<B> add(PackedWord<B> a, PackedWord<B> b) {
  return {a.value + b.value};
}

// ------------------------------------------------------------ plan.hpp:14-92
enum class ExtractionMode { ReciprocalMul, AddHighBits };

struct CompressionPlan {
  PrimeModulus modulus;
  int t = 0;
  int d = 0;
  int e = 1;
  int beta = 53;
  std::uint64_t kmax = 0;
  double inv_qd = 1.0;
  ExtractionMode extraction = ExtractionMode::ReciprocalMul;

  std::uint64_t q() const { return std::uint64_t{1} << t; }
  std::uint64_t q_mask() const { return q() - 1; }
  std::uint32_t p() const { return modulus.value(); }
};

struct FullPlan {
  CompressionPlan base;
  int dq = 0;
  int dtheta = 0;
  int theta_exponent = 0;
  int q_slots() const { return dq + 1; }
  int theta_slots() const { return dtheta + 1; }
};

enum class Algorithm { Naive, CommonCompressed, RightCompressed, LeftCompressed, FullCompressed, Blocked };
inline const char* algorithm_name(Algorithm a) {
  switch (a) {
    case Algorithm::Naive: return "naive";
    case Algorithm::CommonCompressed: return "common";
    case Algorithm::RightCompressed: return "right";
    case Algorithm::LeftCompressed: return "left";
    case Algorithm::FullCompressed: return "full";
    case Algorithm::Blocked: return "blocked";
  }
  return "?";
}

namespace detail {
inline qg_plan to_c(const CompressionPlan& p) {
  qg_plan c{};
  c.p = p.p();
  c.t = p.t;
  c.d = p.d;
  c.e = p.e;
  c.beta = p.beta;
  c.kmax = p.kmax;
  c.inv_qd = p.inv_qd;
  c.extraction = p.extraction == ExtractionMode::AddHighBits ? QG_EXTRACT_ADD_HIGH_BITS : QG_EXTRACT_RECIPROCAL_MUL;
  return c;
}
inline CompressionPlan from_c(const qg_plan& c) {
  CompressionPlan p{PrimeModulus(c.p)};
  p.t = c.t;
  p.d = c.d;
  p.e = c.e;
  p.beta = c.beta;
  p.kmax = c.kmax;
  p.inv_qd = c.inv_qd;
  p.extraction = c.extraction == QG_EXTRACT_ADD_HIGH_BITS ? ExtractionMode::AddHighBits : ExtractionMode::ReciprocalMul;
  return p;
}
inline qg_full_plan to_c(const FullPlan& f) {
  qg_full_plan c{};
  c.base = to_c(f.base);
  c.dq = f.dq;
  c.dtheta = f.dtheta;
  c.theta_exponent = f.theta_exponent;
  return c;
}
}  // namespace detail

// plan_compression, plan.hpp:125-159
inline CompressionPlan plan_compression(const PrimeModulus& m, std::uint64_t k, int beta = 53,
                                        ExtractionMode mode = ExtractionMode::ReciprocalMul) {
  qg_plan c{};
  detail::check(qg_plan_compression(m.value(), k, beta,
                                    mode == ExtractionMode::AddHighBits ? QG_EXTRACT_ADD_HIGH_BITS
                                                                        : QG_EXTRACT_RECIPROCAL_MUL,
                                    &c),
                "plan_compression");
  return detail::from_c(c);
}
// uncompressed_plan, plan.hpp:164-179
inline CompressionPlan uncompressed_plan(const PrimeModulus& m, std::uint64_t k, int beta = 53) {
  qg_plan c{};
  detail::check(qg_uncompressed_plan(m.value(), k, beta, &c), "uncompressed_plan");
  return detail::from_c(c);
}
// plan_packed_axis, plan.hpp:186-203
inline CompressionPlan plan_packed_axis(const PrimeModulus& m, std::uint64_t k, std::uint64_t axis_len,
                                        int beta = 53) {
  qg_plan c{};
  detail::check(qg_plan_packed_axis(m.value(), k, axis_len, beta, &c), "plan_packed_axis");
  return detail::from_c(c);
}
// choose_panel, plan.hpp:209-224
inline std::uint64_t choose_panel(const PrimeModulus& m, std::uint64_t k, int beta = 53) {
  std::uint64_t out = 0;
  detail::check(qg_choose_panel(m.value(), k, beta, &out), "choose_panel");
  return out;
}
// plan_full, plan.hpp:229-252
inline FullPlan plan_full(const PrimeModulus& m, std::uint64_t k, int beta = 53) {
  qg_full_plan c{};
  detail::check(qg_plan_full(m.value(), k, beta, &c), "plan_full");
  return FullPlan{detail::from_c(c.base), c.dq, c.dtheta, c.theta_exponent};
}

// ------------------------------------------------------------ matrix.hpp:14-63
struct ResidueMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<Residue> data;
  ResidueMatrix() = default;
  ResidueMatrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0) {}
  Residue& at(std::size_t i, std::size_t j) { return data[i * cols + j]; }
  Residue at(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
  friend bool operator==(const ResidueMatrix&, const ResidueMatrix&) = default;
};

enum class PackDirection { Forward, Reversed };
enum class PackAxis { Row, Column };
struct PackOrientation {
  PackDirection direction = PackDirection::Forward;
  PackAxis axis = PackAxis::Column;
  int slots = 1;
  friend bool operator==(const PackOrientation&, const PackOrientation&) = default;
};

template <class B>
struct CompressedMatrix {
  std::size_t logical_rows;
  std::size_t logical_cols;
  std::size_t stored_rows;
  std::size_t stored_cols;
  PackOrientation orientation;
  CompressionPlan plan;
  std::vector<PackedWord<B>> data;

  CompressedMatrix(std::size_t lrows, std::size_t lcols, std::size_t srows, std::size_t scols, PackOrientation o,
                   CompressionPlan pl)
      : logical_rows(lrows),
        logical_cols(lcols),
        stored_rows(srows),
        stored_cols(scols),
        orientation(o),
        plan(std::move(pl)),
        data(srows * scols) {}

  PackedWord<B>& at(std::size_t i, std::size_t j) { return data[i * stored_cols + j]; }
  PackedWord<B> at(std::size_t i, std::size_t j) const { return data[i * stored_cols + j]; }
};

// ------------------------------------------------------------ device plumbing
namespace detail {

template <class B>
constexpr bool is_i64 = std::is_same_v<B, Int64Word>;

static_assert(sizeof(PackedWord<DoubleWord>) == sizeof(double), "PackedWord<DoubleWord> must be a bare double");
static_assert(sizeof(PackedWord<Int64Word>) == sizeof(std::uint64_t), "PackedWord<Int64Word> must be a bare uint64");

// One device allocation (freed on scope exit).
class DeviceBuffer {
 public:
  explicit DeviceBuffer(std::size_t bytes) : bytes_(bytes) { check(qg_device_alloc(bytes, &ptr_), "device alloc"); }
  template <class T>
  explicit DeviceBuffer(const std::vector<T>& host) : DeviceBuffer(host.size() * sizeof(T)) {
    check(qg_copy_to_device(ptr_, host.data(), bytes_), "copy to device");
  }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  ~DeviceBuffer() { qg_device_free(ptr_); }
  template <class T = void>
  T* get() const {
    return static_cast<T*>(ptr_);
  }
  template <class T>
  void download(std::vector<T>& host) const {
    check(qg_copy_to_host(host.data(), ptr_, host.size() * sizeof(T)), "copy to host");
  }

 private:
  void* ptr_ = nullptr;
  std::size_t bytes_ = 0;
};

inline void check_inner_dims(const ResidueMatrix& a, const ResidueMatrix& b) {  // gemm.hpp:22-27
  if (a.cols != b.rows)
    throw DimensionMismatch("inner dimensions disagree: " + std::to_string(a.rows) + "x" + std::to_string(a.cols) +
                            " times " + std::to_string(b.rows) + "x" + std::to_string(b.cols));
}
inline void check_common_dim(const CompressionPlan& plan, std::size_t k) {  // gemm.hpp:29-35
  if (k > plan.kmax)
    throw PlanMismatch("common dimension " + std::to_string(k) + " exceeds kmax=" + std::to_string(plan.kmax) +
                       " for p=" + std::to_string(plan.p()) + ", Q=2^" + std::to_string(plan.t));
}
inline bool plans_compatible(const CompressionPlan& a, const CompressionPlan& b) {  // gemm.hpp:37-39
  return a.p() == b.p() && a.t == b.t && a.e == b.e && a.beta == b.beta;
}
inline std::size_t group_count(std::size_t len, int slots) { return (len + slots - 1) / slots; }
template <class B>
void check_backend(const CompressionPlan& plan) {  // pack.hpp:19-24
  if (plan.beta > B::exact_bits)
    throw PlanMismatch("plan needs " + std::to_string(plan.beta) + " exact bits, backend has " +
                       std::to_string(B::exact_bits));
}
inline qg_orientation to_c(const PackOrientation& o) {
  qg_orientation c{};
  c.direction = o.direction == PackDirection::Reversed ? QG_REVERSED : QG_FORWARD;
  c.axis = o.axis == PackAxis::Column ? QG_COLUMN : QG_ROW;
  c.slots = o.slots;
  return c;
}

// The device pack of one reference layout (kind: gemm.hpp:104-178) into `out`.
enum class Pack { RowsReversed, ColsForward, OuterCols, OuterRows };
template <class B>
void device_pack(Pack kind, const CompressionPlan& plan, const std::vector<Residue>& src, std::size_t rows,
                 std::size_t cols, CompressedMatrix<B>& out) {
  if (out.data.empty()) return;
  DeviceBuffer ds(src);
  DeviceBuffer dw(out.data.size() * sizeof(PackedWord<B>));
  const qg_plan pc = to_c(plan);
  const std::size_t ldo = out.stored_cols;
  int st;
  if constexpr (is_i64<B>) {
    auto* w = dw.get<std::uint64_t>();
    switch (kind) {
      case Pack::RowsReversed: st = qg_compress_rows_reversed_u64(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      case Pack::ColsForward: st = qg_compress_cols_forward_u64(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      case Pack::OuterCols: st = qg_compress_outer_cols_u64(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      default: st = qg_compress_outer_rows_u64(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
    }
  } else {
    auto* w = dw.get<double>();
    switch (kind) {
      case Pack::RowsReversed: st = qg_compress_rows_reversed(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      case Pack::ColsForward: st = qg_compress_cols_forward(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      case Pack::OuterCols: st = qg_compress_outer_cols(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
      default: st = qg_compress_outer_rows(&pc, ds.get(), QG_U32, rows, cols, cols, w, ldo, nullptr); break;
    }
  }
  check(st, "compress");
  dw.download(out.data);
}

// A plan copy whose kmax admits `len` residues (the single-word pack helpers
// have no common-dimension check in the reference).
inline CompressionPlan widened(const CompressionPlan& plan, std::size_t len) {
  CompressionPlan p = plan;
  if (p.kmax < len) p.kmax = len;
  return p;
}

}  // namespace detail

// ------------------------------------------------------------ pack.hpp:47-155
// compress_forward, pack.hpp:47-54
template <class B>
PackedWord<B> compress_forward(std::span<const Residue> v, const CompressionPlan& plan) {
  detail::check_backend<B>(plan);
  if (v.size() > static_cast<std::size_t>(plan.e))
    throw SlotOverflow("compress_forward: " + std::to_string(v.size()) + " residues into " + std::to_string(plan.e) +
                       " slots");
  CompressedMatrix<B> out(1, v.size(), 1, v.empty() ? 0 : 1, {PackDirection::Forward, PackAxis::Column, plan.e}, plan);
  detail::device_pack(detail::Pack::OuterCols, plan, std::vector<Residue>(v.begin(), v.end()), 1, v.size(), out);
  return out.data.empty() ? PackedWord<B>{} : out.data[0];
}
// compress_reverse, pack.hpp:59-70 (a short group is scaled by Q^(e-len))
template <class B>
PackedWord<B> compress_reverse(std::span<const Residue> v, const CompressionPlan& plan) {
  detail::check_backend<B>(plan);
  if (v.size() > static_cast<std::size_t>(plan.e))
    throw SlotOverflow("compress_reverse: " + std::to_string(v.size()) + " residues into " + std::to_string(plan.e) +
                       " slots");
  const CompressionPlan wide = detail::widened(plan, v.size());
  CompressedMatrix<B> out(1, v.size(), 1, v.empty() ? 0 : 1, {PackDirection::Reversed, PackAxis::Column, plan.e},
                          wide);
  detail::device_pack(detail::Pack::RowsReversed, wide, std::vector<Residue>(v.begin(), v.end()), 1, v.size(), out);
  return out.data.empty() ? PackedWord<B>{} : out.data[0];
}
// extract_coefficient, pack.hpp:78-100 (both extraction modes)
template <class B>
Residue extract_coefficient(PackedWord<B> w, const CompressionPlan& plan) {
  detail::check_backend<B>(plan);
  const std::vector<PackedWord<B>> in{w};
  detail::DeviceBuffer dw(in);
  detail::DeviceBuffer dout(sizeof(std::int32_t));
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_extract_coefficients_u64(&pc, dw.get<std::uint64_t>(), 1, dout.get<std::int32_t>(), nullptr),
                  "extract_coefficient");
  else
    detail::check(qg_extract_coefficients(&pc, dw.get<double>(), 1, dout.get<std::int32_t>(), nullptr),
                  "extract_coefficient");
  std::vector<std::int32_t> out(1);
  dout.download(out);
  return static_cast<Residue>(out[0]);
}
// extract_all, pack.hpp:104-119
template <class B>
std::vector<std::uint64_t> extract_all(PackedWord<B> w, const CompressionPlan& plan) {
  detail::check_backend<B>(plan);
  const std::vector<PackedWord<B>> in{w};
  detail::DeviceBuffer dw(in);
  std::vector<std::uint64_t> digits(plan.e);
  detail::DeviceBuffer dd(digits.size() * sizeof(std::uint64_t));
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_extract_digits_u64(&pc, dw.get<std::uint64_t>(), 1, dd.get<std::uint64_t>(), nullptr),
                  "extract_all");
  else
    detail::check(qg_extract_digits(&pc, dw.get<double>(), 1, dd.get<std::uint64_t>(), nullptr), "extract_all");
  dd.download(digits);
  return digits;
}
// redq, pack.hpp:124-137
template <class B>
PackedWord<B> redq(PackedWord<B> w, const CompressionPlan& plan) {
  detail::check_backend<B>(plan);
  std::vector<PackedWord<B>> v{w};
  detail::DeviceBuffer dw(v);
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_redq_u64(&pc, dw.get<std::uint64_t>(), 1, nullptr), "redq");
  else
    detail::check(qg_redq(&pc, dw.get<double>(), 1, nullptr), "redq");
  dw.download(v);
  return v[0];
}
// reduce_and_compress, pack.hpp:141-155
template <class B>
std::vector<PackedWord<B>> reduce_and_compress(std::span<const PackedWord<B>> row, const CompressionPlan& plan) {
  if (row.empty()) return {};
  detail::check_backend<B>(plan);
  const std::size_t groups = detail::group_count(row.size(), plan.e);
  std::vector<PackedWord<B>> out(groups);
  detail::DeviceBuffer dw(std::vector<PackedWord<B>>(row.begin(), row.end()));
  detail::DeviceBuffer dout(groups * sizeof(PackedWord<B>));
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_reduce_and_compress_u64(&pc, dw.get<std::uint64_t>(), 1, row.size(), row.size(),
                                             dout.get<std::uint64_t>(), groups, nullptr),
                  "reduce_and_compress");
  else
    detail::check(qg_reduce_and_compress(&pc, dw.get<double>(), 1, row.size(), row.size(), dout.get<double>(), groups,
                                         nullptr),
                  "reduce_and_compress");
  dout.download(out);
  return out;
}

// ------------------------------------------------------------ gemm.hpp
// PhaseSeconds, gemm.hpp:49-53: multiply = device time of the contraction
// kernels, convert = the rest of the call (transfers, packing, extraction).
struct PhaseSeconds {
  double multiply = 0;
  double convert = 0;
};
inline void set_phase_timing(bool enable) { qg_set_phase_timing(enable ? 1 : 0); }
inline PhaseSeconds last_phase_seconds() {
  PhaseSeconds ph;
  qg_last_phase_seconds(&ph.multiply, &ph.convert);
  return ph;
}
namespace detail {
// Runs `call` (a host-data ABI entry) with the phase split on if `phases`
// asks for it, and adds the split to *phases (the reference's PhaseTimer adds).
template <class F>
void with_phases(PhaseSeconds* phases, F&& call) {
  if (phases) qg_set_phase_timing(1);
  call();
  if (phases) {
    const PhaseSeconds ph = last_phase_seconds();
    phases->multiply += ph.multiply;
    phases->convert += ph.convert;
  }
}
}  // namespace detail

// naive_gemm, gemm.hpp:80-100 (a plain device kernel, no packing)
inline ResidueMatrix naive_gemm(const ResidueMatrix& a, const ResidueMatrix& b, const PrimeModulus& mod) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  detail::check(qg_host_naive_gemm(mod.value(), a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                "naive_gemm");
  return c;
}

// compress_rows_reversed, gemm.hpp:104-118
template <class B>
CompressedMatrix<B> compress_rows_reversed(const ResidueMatrix& a, const CompressionPlan& plan) {
  detail::check_common_dim(plan, a.cols);
  const std::size_t groups = detail::group_count(a.cols, plan.e);
  CompressedMatrix<B> out(a.rows, a.cols, a.rows, groups, {PackDirection::Reversed, PackAxis::Column, plan.e}, plan);
  if (!out.data.empty()) detail::check_backend<B>(plan);
  detail::device_pack(detail::Pack::RowsReversed, plan, a.data, a.rows, a.cols, out);
  return out;
}
// compress_cols_forward, gemm.hpp:122-140
template <class B>
CompressedMatrix<B> compress_cols_forward(const ResidueMatrix& b, const CompressionPlan& plan) {
  detail::check_common_dim(plan, b.rows);
  const std::size_t groups = detail::group_count(b.rows, plan.e);
  CompressedMatrix<B> out(b.rows, b.cols, groups, b.cols, {PackDirection::Forward, PackAxis::Row, plan.e}, plan);
  if (!out.data.empty()) detail::check_backend<B>(plan);
  detail::device_pack(detail::Pack::ColsForward, plan, b.data, b.rows, b.cols, out);
  return out;
}
// compress_outer_cols, gemm.hpp:145-158
template <class B>
CompressedMatrix<B> compress_outer_cols(const ResidueMatrix& b, const CompressionPlan& plan) {
  const std::size_t groups = detail::group_count(b.cols, plan.e);
  CompressedMatrix<B> out(b.rows, b.cols, b.rows, groups, {PackDirection::Forward, PackAxis::Column, plan.e}, plan);
  if (!out.data.empty()) detail::check_backend<B>(plan);
  detail::device_pack(detail::Pack::OuterCols, detail::widened(plan, b.rows), b.data, b.rows, b.cols, out);
  return out;
}
// compress_outer_rows, gemm.hpp:160-178
template <class B>
CompressedMatrix<B> compress_outer_rows(const ResidueMatrix& a, const CompressionPlan& plan) {
  const std::size_t groups = detail::group_count(a.rows, plan.e);
  CompressedMatrix<B> out(a.rows, a.cols, groups, a.cols, {PackDirection::Forward, PackAxis::Row, plan.e}, plan);
  if (!out.data.empty()) detail::check_backend<B>(plan);
  detail::device_pack(detail::Pack::OuterRows, detail::widened(plan, a.cols), a.data, a.rows, a.cols, out);
  return out;
}

// uncompress, gemm.hpp:182-204
template <class B>
ResidueMatrix uncompress(const CompressedMatrix<B>& cm) {
  ResidueMatrix out(cm.logical_rows, cm.logical_cols);
  if (cm.data.empty() || out.data.empty()) return out;
  detail::check_backend<B>(cm.plan);
  const qg_plan pc = detail::to_c(cm.plan);
  int st;
  if constexpr (detail::is_i64<B>)
    st = qg_host_uncompress_u64(&pc, detail::to_c(cm.orientation), reinterpret_cast<const std::uint64_t*>(cm.data.data()),
                                cm.stored_rows, cm.stored_cols, cm.logical_rows, cm.logical_cols, out.data.data());
  else
    st = qg_host_uncompress(&pc, detail::to_c(cm.orientation), reinterpret_cast<const double*>(cm.data.data()),
                            cm.stored_rows, cm.stored_cols, cm.logical_rows, cm.logical_cols, out.data.data());
  detail::check(st, "uncompress");
  return out;
}

namespace detail {
template <class B>
void check_common_operands(const CompressedMatrix<B>& ca, const CompressedMatrix<B>& cb) {  // gemm.hpp:213-225
  if (!plans_compatible(ca.plan, cb.plan)) throw PlanMismatch("operands were packed under different plans");
  if (ca.orientation.direction != PackDirection::Reversed || ca.orientation.axis != PackAxis::Column ||
      cb.orientation.direction != PackDirection::Forward || cb.orientation.axis != PackAxis::Row)
    throw PlanMismatch("common product needs a row-reversed left operand and a column-forward right operand");
  if (ca.logical_cols != cb.logical_rows || ca.stored_cols != cb.stored_rows)
    throw DimensionMismatch("inner dimensions disagree: " + std::to_string(ca.logical_rows) + "x" +
                            std::to_string(ca.logical_cols) + " times " + std::to_string(cb.logical_rows) + "x" +
                            std::to_string(cb.logical_cols));
  check_common_dim(ca.plan, ca.logical_cols);
}
}  // namespace detail

// packed_common_product, gemm.hpp:210-244: the reference's accumulators
// (sum of per-product high parts), bit for bit, from the device.
template <class B>
std::vector<PackedWord<B>> packed_common_product(const CompressedMatrix<B>& ca, const CompressedMatrix<B>& cb) {
  detail::check_common_operands(ca, cb);
  const std::size_t m = ca.logical_rows, n = cb.logical_cols;
  std::vector<PackedWord<B>> acc(m * n);
  if (acc.empty()) return acc;
  detail::DeviceBuffer da(ca.data), db(cb.data), dacc(acc.size() * sizeof(PackedWord<B>));
  const qg_plan pc = detail::to_c(ca.plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_packed_common_product_u64(&pc, da.get<std::uint64_t>(), db.get<std::uint64_t>(), m, n,
                                               ca.stored_cols, dacc.get<std::uint64_t>(), nullptr),
                  "packed_common_product");
  else
    detail::check(qg_packed_common_product(&pc, da.get<double>(), db.get<double>(), m, n, ca.logical_cols,
                                           dacc.get<double>(), nullptr),
                  "packed_common_product");
  dacc.download(acc);
  return acc;
}

// reduce_common_entry, gemm.hpp:247-250 (PrimeModulus::reduce of the masked word)
template <class B>
Residue reduce_common_entry(PackedWord<B> w, const CompressionPlan& plan) {
  return plan.modulus.reduce(B::to_u64(w.value) & plan.q_mask());
}

// mul_common_compressed(ca, cb), gemm.hpp:263-271: the fused device product
// (FP64 tensor-core contraction, digit extraction and mod p in one kernel for
// DoubleWord words; the integer high-part kernel for Int64Word words).
template <class B>
ResidueMatrix mul_common_compressed(const CompressedMatrix<B>& ca, const CompressedMatrix<B>& cb) {
  detail::check_common_operands(ca, cb);
  const std::size_t m = ca.logical_rows, n = cb.logical_cols, k = ca.logical_cols;
  ResidueMatrix c(m, n);
  if (c.data.empty()) return c;
  detail::DeviceBuffer da(ca.data), db(cb.data), dc(c.data.size() * sizeof(Residue));
  const qg_plan pc = detail::to_c(ca.plan);
  if constexpr (detail::is_i64<B>) {
    detail::DeviceBuffer dacc(m * n * sizeof(std::uint64_t));
    detail::check(qg_packed_common_product_u64(&pc, da.get<std::uint64_t>(), db.get<std::uint64_t>(), m, n,
                                               ca.stored_cols, dacc.get<std::uint64_t>(), nullptr),
                  "mul_common_compressed");
    detail::check(qg_reduce_common_u64(&pc, dacc.get<std::uint64_t>(), m * n, dc.get<std::int32_t>(), nullptr),
                  "mul_common_compressed");
  } else {
    qg_gpu_plan gp{};
    detail::check(qg_gpu_plan_from(&pc, k, &gp), "mul_common_compressed");
    detail::check(qg_mul_common(&gp, da.get<double>(), db.get<double>(), m, n, k, dc.get<std::int32_t>(), n, nullptr),
                  "mul_common_compressed");
  }
  dc.download(c.data);
  return c;
}

// mul_common_compressed(A, B, plan), gemm.hpp:254-260: packs and the product
// in one pipelined host call (H2D / pack / contraction / D2H overlapped).
template <class B = DoubleWord>
ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  detail::check_common_dim(plan, a.cols);
  if (a.rows * detail::group_count(a.cols, plan.e) != 0 || b.cols * detail::group_count(b.rows, plan.e) != 0)
    detail::check_backend<B>(plan);
  ResidueMatrix c(a.rows, b.cols);
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_host_mul_common_i64(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                  "mul_common_compressed");
  else
    detail::check(qg_host_mul_common(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                  "mul_common_compressed");
  return c;
}

// mul_common_repacked, gemm.hpp:275-280: C reduced and its rows re-packed
// forward in groups of e, compress_outer_cols(C, plan).
template <class B = DoubleWord>
CompressedMatrix<B> mul_common_repacked(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  detail::check_common_dim(plan, a.cols);
  if constexpr (!detail::is_i64<B>) {
    const std::size_t groups = detail::group_count(b.cols, plan.e);
    CompressedMatrix<B> out(a.rows, b.cols, a.rows, groups, {PackDirection::Forward, PackAxis::Column, plan.e}, plan);
    if (a.rows * detail::group_count(a.cols, plan.e) != 0 || b.cols * detail::group_count(b.rows, plan.e) != 0 ||
        !out.data.empty())
      detail::check_backend<B>(plan);
    const qg_plan pc = detail::to_c(plan);
    detail::check(qg_host_mul_common_repacked(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols,
                                              reinterpret_cast<double*>(out.data.data())),
                  "mul_common_repacked");
    return out;
  } else {
    const ResidueMatrix c = mul_common_compressed<B>(a, b, plan);
    return compress_outer_cols<B>(c, plan);
  }
}

// packed_right_product, gemm.hpp:285-310 (pre-REDQ words)
namespace detail {
template <class B>
CompressedMatrix<B> right_product(const ResidueMatrix& a, const CompressedMatrix<B>& cb, bool reduce) {
  if (cb.orientation.direction != PackDirection::Forward || cb.orientation.axis != PackAxis::Column)
    throw PlanMismatch("right product needs the right operand packed forward on its columns");
  if (a.cols != cb.logical_rows)
    throw DimensionMismatch("inner dimensions disagree: " + std::to_string(a.rows) + "x" + std::to_string(a.cols) +
                            " times " + std::to_string(cb.logical_rows) + "x" + std::to_string(cb.logical_cols));
  check_common_dim(cb.plan, a.cols);
  const std::size_t m = a.rows, h = cb.stored_cols;
  CompressedMatrix<B> cc(m, cb.logical_cols, m, h, cb.orientation, cb.plan);
  if (cc.data.empty()) return cc;
  if (reduce) check_backend<B>(cb.plan);  // redq's check (pack.hpp:126)
  DeviceBuffer dcb(cb.data), dcc(cc.data.size() * sizeof(PackedWord<B>));
  const qg_plan pc = to_c(cb.plan);
  const std::size_t n = h * cb.plan.e < cb.logical_cols ? cb.logical_cols : h * cb.plan.e;
  int st;
  if constexpr (is_i64<B>) {
    DeviceBuffer da(a.data);
    st = (reduce ? qg_mul_right_u64 : qg_packed_right_product_u64)(&pc, da.get(), QG_U32, a.cols,
                                                                    dcb.get<std::uint64_t>(), m, a.cols, n,
                                                                    dcc.get<std::uint64_t>(), nullptr);
  } else {
    DeviceBuffer da(std::vector<double>(a.data.begin(), a.data.end()));  // residues as exact doubles
    st = (reduce ? qg_mul_right : qg_packed_right_product)(&pc, da.get<double>(), a.cols, dcb.get<double>(), m,
                                                            a.cols, n, dcc.get<double>(), nullptr);
  }
  check(st, reduce ? "mul_right_compressed" : "packed_right_product");
  dcc.download(cc.data);
  return cc;
}
template <class B>
CompressedMatrix<B> left_product(const CompressedMatrix<B>& ca, const ResidueMatrix& b, bool reduce) {
  if (ca.orientation.direction != PackDirection::Forward || ca.orientation.axis != PackAxis::Row)
    throw PlanMismatch("left product needs the left operand packed forward on its rows");
  if (ca.logical_cols != b.rows)
    throw DimensionMismatch("inner dimensions disagree: " + std::to_string(ca.logical_rows) + "x" +
                            std::to_string(ca.logical_cols) + " times " + std::to_string(b.rows) + "x" +
                            std::to_string(b.cols));
  check_common_dim(ca.plan, b.rows);
  const std::size_t g = ca.stored_rows, n = b.cols;
  CompressedMatrix<B> cc(ca.logical_rows, n, g, n, ca.orientation, ca.plan);
  if (cc.data.empty()) return cc;
  if (reduce) check_backend<B>(ca.plan);
  DeviceBuffer dca(ca.data), db(b.data), dcc(cc.data.size() * sizeof(PackedWord<B>));
  const qg_plan pc = to_c(ca.plan);
  const std::size_t m = g * ca.plan.e < ca.logical_rows ? ca.logical_rows : g * ca.plan.e;
  int st;
  if constexpr (is_i64<B>)
    st = (reduce ? qg_mul_left_u64 : qg_packed_left_product_u64)(&pc, dca.get<std::uint64_t>(), db.get(), QG_U32, n,
                                                                  m, b.rows, n, dcc.get<std::uint64_t>(), nullptr);
  else
    st = (reduce ? qg_mul_left : qg_packed_left_product)(&pc, dca.get<double>(), b.rows, db.get(), QG_U32, n, m,
                                                          b.rows, n, dcc.get<double>(), nullptr);
  check(st, reduce ? "mul_left_compressed" : "packed_left_product");
  dcc.download(cc.data);
  return cc;
}
}  // namespace detail

template <class B>
CompressedMatrix<B> packed_right_product(const ResidueMatrix& a, const CompressedMatrix<B>& cb) {
  return detail::right_product(a, cb, false);
}
// redq_in_place, gemm.hpp:313-316
template <class B>
void redq_in_place(CompressedMatrix<B>& cm) {
  if (cm.data.empty()) return;
  detail::check_backend<B>(cm.plan);
  detail::DeviceBuffer dw(cm.data);
  const qg_plan pc = detail::to_c(cm.plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_redq_u64(&pc, dw.get<std::uint64_t>(), cm.data.size(), nullptr), "redq_in_place");
  else
    detail::check(qg_redq(&pc, dw.get<double>(), cm.data.size(), nullptr), "redq_in_place");
  dw.download(cm.data);
}
// mul_right_compressed(a, cb), gemm.hpp:320-325 (product + REDQ fused on the device)
template <class B>
CompressedMatrix<B> mul_right_compressed(const ResidueMatrix& a, const CompressedMatrix<B>& cb) {
  return detail::right_product(a, cb, true);
}
// mul_right_compressed(ca, cb), gemm.hpp:329-335: the left operand is unpacked first
template <class B>
CompressedMatrix<B> mul_right_compressed(const CompressedMatrix<B>& ca, const CompressedMatrix<B>& cb) {
  if (ca.orientation.direction != PackDirection::Forward)
    throw PlanMismatch("left operand must be packed forward to be unpacked");
  return mul_right_compressed(uncompress(ca), cb);
}
// packed_left_product, gemm.hpp:340-364
template <class B>
CompressedMatrix<B> packed_left_product(const CompressedMatrix<B>& ca, const ResidueMatrix& b) {
  return detail::left_product(ca, b, false);
}
// mul_left_compressed, gemm.hpp:366-371
template <class B>
CompressedMatrix<B> mul_left_compressed(const CompressedMatrix<B>& ca, const ResidueMatrix& b) {
  return detail::left_product(ca, b, true);
}

// mul_full_compressed, gemm.hpp:377-445
template <class B = DoubleWord>
ResidueMatrix mul_full_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const FullPlan& fp,
                                  PhaseSeconds* phases = nullptr) {
  detail::check_inner_dims(a, b);
  detail::check_backend<B>(fp.base);
  detail::check_common_dim(fp.base, a.cols);
  ResidueMatrix c(a.rows, b.cols);
  const qg_full_plan fc = detail::to_c(fp);
  detail::with_phases(phases, [&] {
    if constexpr (detail::is_i64<B>)
      detail::check(qg_host_mul_full_i64(&fc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                    "mul_full_compressed");
    else
      detail::check(qg_host_mul_full(&fc, 0, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                    "mul_full_compressed");
  });
  return c;
}

// blocked_accumulate, gemm.hpp:450-489
template <class B = DoubleWord>
ResidueMatrix blocked_accumulate(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan,
                                 std::size_t kpanel, PhaseSeconds* phases = nullptr) {
  detail::check_inner_dims(a, b);
  if (kpanel < 1) throw std::invalid_argument("blocked_accumulate: kpanel must be >= 1");
  detail::check_common_dim(plan, kpanel);
  ResidueMatrix c(a.rows, b.cols);
  if (a.rows * a.cols != 0 || b.rows * b.cols != 0) detail::check_backend<B>(plan);
  const qg_plan pc = detail::to_c(plan);
  detail::with_phases(phases, [&] {
    if constexpr (detail::is_i64<B>)
      detail::check(qg_host_blocked_accumulate_i64(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, kpanel,
                                                   c.data.data()),
                    "blocked_accumulate");
    else
      detail::check(qg_host_blocked_accumulate(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, kpanel,
                                               c.data.data()),
                    "blocked_accumulate");
  });
  return c;
}

// ------------------------------------------------------------ prng.hpp:12-38
class SplitMix64 {
 public:
  explicit SplitMix64(std::uint64_t seed) : state_(seed) {}
  std::uint64_t next() {
    std::uint64_t z = (state_ += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
  }
  std::uint64_t below(std::uint64_t bound) { return next() % bound; }

 private:
  std::uint64_t state_;
};
// random_residue_matrix, prng.hpp:31-38: the same sequence, generated on the
// device (element i is SplitMix64 output number i, counter-based).
inline ResidueMatrix random_residue_matrix(std::size_t rows, std::size_t cols, const PrimeModulus& mod,
                                           std::uint64_t seed) {
  ResidueMatrix m(rows, cols);
  if (!m.data.empty())
    detail::check(qg_host_random_residue_matrix(rows, cols, mod.value(), seed, m.data.data()),
                  "random_residue_matrix");
  return m;
}

// ------------------------------------------------------------ matrix_io.hpp:14-77
struct MatrixFile {
  std::uint32_t p;
  ResidueMatrix matrix;
};
namespace detail {
inline MatrixFile adopt(int status, const char* where, std::uint32_t p, std::size_t rows, std::size_t cols,
                        std::uint32_t* data) {
  if (status != QG_OK) {
    if (status == QG_PARSE_ERROR) throw ParseError(qg_last_error());
    check(status, where);
  }
  MatrixFile mf{p, ResidueMatrix(rows, cols)};
  if (rows * cols != 0) std::copy(data, data + rows * cols, mf.matrix.data.begin());
  qg_free(data);
  return mf;
}
}  // namespace detail
inline MatrixFile read_matrix(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::uint32_t p = 0, *data = nullptr;
  std::size_t rows = 0, cols = 0;
  const int st = qg_parse_matrix(text.data(), text.size(), &p, &rows, &cols, &data);
  return detail::adopt(st, "read_matrix", p, rows, cols, data);
}
inline MatrixFile read_matrix_file(const std::string& path) {
  std::uint32_t p = 0, *data = nullptr;
  std::size_t rows = 0, cols = 0;
  const int st = qg_read_matrix_file(path.c_str(), &p, &rows, &cols, &data);
  return detail::adopt(st, "read_matrix_file", p, rows, cols, data);
}
inline void write_matrix(std::ostream& out, const ResidueMatrix& m, std::uint32_t p) {
  out << "M " << p << ' ' << m.rows << ' ' << m.cols << '\n';
  for (std::size_t i = 0; i < m.rows; ++i)
    for (std::size_t j = 0; j < m.cols; ++j) out << m.at(i, j) << (j + 1 == m.cols ? '\n' : ' ');
}
inline void write_matrix_file(const std::string& path, const ResidueMatrix& m, std::uint32_t p) {
  const int st = qg_write_matrix_file(path.c_str(), p, m.data.data(), m.rows, m.cols);
  if (st == QG_PARSE_ERROR) throw ParseError(qg_last_error());
  detail::check(st, "write_matrix_file");
}

// ------------------------------------------------------------ bench.hpp:19-171
struct TimingRecord {
  std::string algorithm;
  std::uint32_t p = 0;
  std::size_t m = 0, k = 0, n = 0;
  int t = 0;
  int e = 1;
  double seconds_multiply = 0;
  double seconds_convert = 0;
  std::uint32_t checksum = 0;
};
inline const char* timing_csv_header() { return "algorithm,p,m,k,n,t,e,seconds_multiply,seconds_convert,checksum"; }
inline std::string to_csv_row(const TimingRecord& r) {
  std::ostringstream os;
  os << r.algorithm << ',' << r.p << ',' << r.m << ',' << r.k << ',' << r.n << ',' << r.t << ',' << r.e << ','
     << std::fixed << std::setprecision(6) << r.seconds_multiply << ',' << r.seconds_convert << ',' << r.checksum;
  return os.str();
}
inline std::uint32_t residue_checksum(const ResidueMatrix& m) {
  std::uint32_t sum = 0;
  for (Residue v : m.data) sum += v;
  return sum;
}

// run_bench, bench.hpp:61-166: each algorithm through this header's device
// calls; seconds_multiply is the contraction kernels' device time (the
// library's phase split), seconds_convert the rest of the call.
template <class B = DoubleWord>
std::vector<TimingRecord> run_bench(Algorithm algo, const PrimeModulus& mod, std::size_t m, std::size_t k,
                                    std::size_t n, int reps, std::uint64_t seed, int beta = 53,
                                    std::uint64_t kpanel = 0, const CompressionPlan* common_plan = nullptr) {
  const ResidueMatrix a = random_residue_matrix(m, k, mod, seed);
  const ResidueMatrix b = random_residue_matrix(k, n, mod, seed + 1);
  std::vector<TimingRecord> out;
  set_phase_timing(true);
  for (int rep = 0; rep < reps; ++rep) {
    TimingRecord rec;
    rec.algorithm = algorithm_name(algo);
    rec.p = mod.value();
    rec.m = m;
    rec.k = k;
    rec.n = n;
    ResidueMatrix c;
    PhaseSeconds ph;
    auto timed = [](auto&& f) {
      const auto t0 = std::chrono::steady_clock::now();
      f();
      return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    };
    switch (algo) {
      case Algorithm::Naive:
        rec.seconds_multiply = timed([&] { c = naive_gemm(a, b, mod); });
        break;
      case Algorithm::CommonCompressed: {
        const CompressionPlan plan = common_plan ? *common_plan : plan_compression(mod, k, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        c = mul_common_compressed<B>(a, b, plan);
        ph = last_phase_seconds();
        rec.seconds_multiply = ph.multiply;
        rec.seconds_convert = ph.convert;
        break;
      }
      case Algorithm::RightCompressed:
      case Algorithm::LeftCompressed: {
        const CompressionPlan plan = plan_compression(mod, k, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        const double conv0 = timed([&] {
          if (algo == Algorithm::RightCompressed) {
            const auto cb = compress_outer_cols<B>(b, plan);
            rec.seconds_multiply = timed([&] { c = uncompress(mul_right_compressed(a, cb)); });
          } else {
            const auto ca = compress_outer_rows<B>(a, plan);
            rec.seconds_multiply = timed([&] { c = uncompress(mul_left_compressed(ca, b)); });
          }
        });
        rec.seconds_convert = conv0 - rec.seconds_multiply;
        break;
      }
      case Algorithm::FullCompressed: {
        const FullPlan fp = plan_full(mod, k, beta);
        rec.t = fp.base.t;
        rec.e = fp.base.e;
        c = mul_full_compressed<B>(a, b, fp, &ph);
        rec.seconds_multiply = ph.multiply;
        rec.seconds_convert = ph.convert;
        break;
      }
      case Algorithm::Blocked: {
        std::uint64_t kp = kpanel ? kpanel : choose_panel(mod, k, beta);
        if (kp == 0) kp = k;
        const CompressionPlan plan = kp >= 2 ? plan_compression(mod, kp, beta) : uncompressed_plan(mod, 1, beta);
        rec.t = plan.t;
        rec.e = plan.e;
        c = blocked_accumulate<B>(a, b, plan, kp, &ph);
        rec.seconds_multiply = ph.multiply;
        rec.seconds_convert = ph.convert;
        break;
      }
    }
    rec.checksum = residue_checksum(c);
    out.push_back(rec);
  }
  set_phase_timing(false);
  return out;
}

// ------------------------------------------------------------ verify.hpp:14-131
struct VerifyResult {
  Algorithm algorithm = Algorithm::Naive;
  std::string backend;
  std::size_t cases = 0;
  std::size_t skipped = 0;
  bool passed = true;
  std::uint64_t seed = 0;
  std::size_t m = 0, k = 0, n = 0;
  std::size_t row = 0, col = 0;
  Residue got = 0, want = 0;
};
namespace detail {
template <class B>
ResidueMatrix run_algorithm(Algorithm algo, const ResidueMatrix& a, const ResidueMatrix& b, const PrimeModulus& mod,
                            int beta) {  // verify.hpp:29-68
  const std::size_t k = a.cols;
  switch (algo) {
    case Algorithm::Naive:
      return naive_gemm(a, b, mod);
    case Algorithm::CommonCompressed: {
      CompressionPlan plan = [&] {
        try {
          return plan_compression(mod, k, beta);
        } catch (const NoCompression&) {
          if (k > 1) throw;
          return uncompressed_plan(mod, k, beta);
        }
      }();
      return mul_common_compressed<B>(a, b, plan);
    }
    case Algorithm::RightCompressed: {
      const auto plan = plan_packed_axis(mod, k, b.cols, beta);
      return uncompress(mul_right_compressed(a, compress_outer_cols<B>(b, plan)));
    }
    case Algorithm::LeftCompressed: {
      const auto plan = plan_packed_axis(mod, k, a.rows, beta);
      return uncompress(mul_left_compressed(compress_outer_rows<B>(a, plan), b));
    }
    case Algorithm::FullCompressed:
      return mul_full_compressed<B>(a, b, plan_full(mod, k, beta));
    case Algorithm::Blocked: {
      const std::uint64_t kp = (k + 1) / 2;
      const auto plan = kp >= 2 ? plan_compression(mod, kp, beta) : uncompressed_plan(mod, 1, beta);
      return blocked_accumulate<B>(a, b, plan, kp);
    }
  }
  throw std::invalid_argument("unknown algorithm");
}
template <class B>
VerifyResult verify_algorithm(Algorithm algo, const char* backend_name, const PrimeModulus& mod, std::size_t max_dim,
                              std::uint64_t seeds, int beta) {  // verify.hpp:70-110
  VerifyResult res;
  res.algorithm = algo;
  res.backend = backend_name;
  for (std::uint64_t seed = 0; seed < seeds; ++seed) {
    SplitMix64 dims(seed * 0x51ab1e ^ 0xfeed);
    const std::size_t m = 1 + dims.below(max_dim);
    const std::size_t k = 1 + dims.below(max_dim);
    const std::size_t n = 1 + dims.below(max_dim);
    const ResidueMatrix a = random_residue_matrix(m, k, mod, seed * 2 + 1);
    const ResidueMatrix b = random_residue_matrix(k, n, mod, seed * 2 + 2);
    ResidueMatrix got(0, 0);
    try {
      got = run_algorithm<B>(algo, a, b, mod, beta);
    } catch (const NoCompression&) {
      ++res.skipped;
      continue;
    }
    const ResidueMatrix want = naive_gemm(a, b, mod);
    ++res.cases;
    if (got != want) {
      res.passed = false;
      res.seed = seed;
      res.m = m;
      res.k = k;
      res.n = n;
      bool found = false;
      for (std::size_t i = 0; i < m && !found; ++i)
        for (std::size_t j = 0; j < n && !found; ++j)
          if (got.at(i, j) != want.at(i, j)) {
            res.row = i;
            res.col = j;
            res.got = got.at(i, j);
            res.want = want.at(i, j);
            found = true;
          }
      return res;
    }
  }
  return res;
}
}  // namespace detail
// run_verify, verify.hpp:115-131
inline std::vector<VerifyResult> run_verify(const PrimeModulus& mod, std::size_t max_dim, std::uint64_t seeds,
                                            int beta = 53) {
  std::vector<VerifyResult> out;
  const int beta_double = std::min(beta, DoubleWord::exact_bits);
  const int beta_int = beta <= DoubleWord::exact_bits ? Int64Word::exact_bits : beta;
  for (Algorithm algo : {Algorithm::CommonCompressed, Algorithm::RightCompressed, Algorithm::LeftCompressed,
                         Algorithm::FullCompressed, Algorithm::Blocked}) {
    out.push_back(detail::verify_algorithm<DoubleWord>(algo, "double", mod, max_dim, seeds, beta_double));
    out.push_back(detail::verify_algorithm<Int64Word>(algo, "int64", mod, max_dim, seeds, beta_int));
  }
  return out;
}

// ------------------------------------------------------------ B200 additions
// A plan k-blocked for the FP64 tensor-core contraction (qg_plan_gpu): the
// contraction flushes every kblock_words packed words, so k may exceed
// plan.kmax; balanced = residues enter as signed digits.
struct GpuPlan {
  CompressionPlan plan;
  std::uint64_t kblock_words = 0;
  std::uint64_t max_exact_words = 0;
  bool balanced = false;
  bool anchored = false;  // anchored accumulation (integer-pipe block flush)
};
namespace detail {
inline qg_gpu_plan to_c(const GpuPlan& g) {
  qg_gpu_plan c{};
  c.plan = to_c(g.plan);
  c.kblock_words = g.kblock_words;
  c.max_exact_words = g.max_exact_words;
  c.balanced = g.balanced ? 1 : 0;
  c.anchored = g.anchored ? 1 : 0;
  return c;
}
}  // namespace detail
// flags: QG_PLAN_UNSIGNED_ONLY, QG_PLAN_NO_ANCHOR (qg_plan_gpu_ex)
inline GpuPlan plan_gpu(const PrimeModulus& m, std::uint64_t k, int flags = 0) {
  qg_gpu_plan c{};
  detail::check(qg_plan_gpu_ex(m.value(), k, flags, &c), "plan_gpu");
  return GpuPlan{detail::from_c(c.plan), c.kblock_words, c.max_exact_words, c.balanced != 0, c.anchored != 0};
}
// mul_common_compressed(A, B) under a GPU plan (k-blocked on the device).
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const GpuPlan& plan) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  const qg_gpu_plan g = detail::to_c(plan);
  detail::check(qg_host_mul_common_gpu(&g, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
                "mul_common_compressed");
  return c;
}
// The same over several GPUs of this process (qg_host_mul_common_multi): rows
// of A and C sharded over `devices`, the packed B sent over NCCL.
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const GpuPlan& plan,
                                           const std::vector<int>& devices) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  const qg_gpu_plan g = detail::to_c(plan);
  detail::check(qg_host_mul_common_multi(&g, devices.data(), (int)devices.size(), a.data.data(), b.data.data(), a.rows,
                                         a.cols, b.cols, c.data.data()),
                "mul_common_compressed");
  return c;
}
// mul_right_compressed(A, compress_outer_cols<B>(B, plan)) in one pipelined
// host call (residues in, post-REDQ words out; no packed-B round trip).
template <class B = DoubleWord>
CompressedMatrix<B> mul_right_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  detail::check_common_dim(plan, a.cols);
  CompressedMatrix<B> cc(a.rows, b.cols, a.rows, detail::group_count(b.cols, plan.e),
                         {PackDirection::Forward, PackAxis::Column, plan.e}, plan);
  if (!cc.data.empty()) detail::check_backend<B>(plan);
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_host_mul_right_i64(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols,
                                        reinterpret_cast<std::uint64_t*>(cc.data.data())),
                  "mul_right_compressed");
  else
    detail::check(qg_host_mul_right(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols,
                                    reinterpret_cast<double*>(cc.data.data())),
                  "mul_right_compressed");
  return cc;
}
// mul_left_compressed(compress_outer_rows<B>(A, plan), B) in one host call.
template <class B = DoubleWord>
CompressedMatrix<B> mul_left_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  detail::check_common_dim(plan, b.rows);
  CompressedMatrix<B> cc(a.rows, b.cols, detail::group_count(a.rows, plan.e), b.cols,
                         {PackDirection::Forward, PackAxis::Row, plan.e}, plan);
  if (!cc.data.empty()) detail::check_backend<B>(plan);
  const qg_plan pc = detail::to_c(plan);
  if constexpr (detail::is_i64<B>)
    detail::check(qg_host_mul_left_i64(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols,
                                       reinterpret_cast<std::uint64_t*>(cc.data.data())),
                  "mul_left_compressed");
  else
    detail::check(qg_host_mul_left(&pc, a.data.data(), b.data.data(), a.rows, a.cols, b.cols,
                                   reinterpret_cast<double*>(cc.data.data())),
                  "mul_left_compressed");
  return cc;
}
// read_matrix on an in-memory text (the CLI's and tests' convenience)
inline MatrixFile read_matrix_text(const std::string& text) {
  std::istringstream in(text);
  return read_matrix(in);
}

}  // namespace qgemm_b200
