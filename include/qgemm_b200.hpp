// qgemm_b200.hpp — C++ drop-in for the reference's qgemm header API,
// implemented over the C ABI (qgemm_b200.h) and therefore over the sm_100a
// kernels. Header-only; link with -lqgemm_b200 (paper_0803_1975_b200/_lib).
//
// Same names, argument meaning and error behaviour as
// /root/reference/proj/include/qgemm/*.hpp for the dot-product and mixed
// paths: value types in, value types out, exceptions on error
// (errors.hpp:8-34, std::invalid_argument for bad arguments). A reference
// caller switches by replacing
//     #include "qgemm/qgemm.hpp"     using namespace qgemm;
// with
//     #include "qgemm_b200.hpp"      using namespace qgemm_b200;
// for the entry points below (INTEGRATION.md lists them with their
// reference file:line).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <type_traits>
#include <string>
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
struct DeviceError : Error { using Error::Error; };  // CUDA failures (no reference analogue)

inline void check(int status, const char* where) {
  if (status == QG_OK) return;
  std::string msg = std::string(where) + ": " + qg_status_string(status);
  if (status == QG_CUDA_ERROR) msg += std::string(" (") + qg_last_error() + ")";
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
    default: throw DeviceError(msg);
  }
}

// ------------------------------------------------------------ field / plan
using Residue = std::uint32_t;  // field.hpp:12

enum class ExtractionMode { ReciprocalMul = QG_EXTRACT_RECIPROCAL_MUL, AddHighBits = QG_EXTRACT_ADD_HIGH_BITS };

// CompressionPlan, plan.hpp:29-42 (the modulus is carried as its value).
struct CompressionPlan {
  qg_plan c{};
  std::uint32_t p() const { return c.p; }
  int t() const { return c.t; }
  int d() const { return c.d; }
  int e() const { return c.e; }
  int beta() const { return c.beta; }
  std::uint64_t kmax() const { return c.kmax; }
  double inv_qd() const { return c.inv_qd; }
  std::uint64_t q() const { return std::uint64_t{1} << c.t; }
  std::uint64_t q_mask() const { return q() - 1; }
};

// A plan k-blocked for the FP64 tensor-core contraction (qg_plan_gpu).
struct GpuPlan {
  qg_gpu_plan c{};
  CompressionPlan plan() const { return CompressionPlan{c.plan}; }
  std::uint64_t kblock_words() const { return c.kblock_words; }
};

// plan_compression, plan.hpp:125-159
inline CompressionPlan plan_compression(std::uint32_t p, std::uint64_t k, int beta = 53,
                                        ExtractionMode mode = ExtractionMode::ReciprocalMul) {
  CompressionPlan pl;
  check(qg_plan_compression(p, k, beta, static_cast<int>(mode), &pl.c), "plan_compression");
  return pl;
}
// uncompressed_plan, plan.hpp:164-179
inline CompressionPlan uncompressed_plan(std::uint32_t p, std::uint64_t k, int beta = 53) {
  CompressionPlan pl;
  check(qg_uncompressed_plan(p, k, beta, &pl.c), "uncompressed_plan");
  return pl;
}
// plan_packed_axis, plan.hpp:186-203
inline CompressionPlan plan_packed_axis(std::uint32_t p, std::uint64_t k, std::uint64_t axis_len,
                                        int beta = 53) {
  CompressionPlan pl;
  check(qg_plan_packed_axis(p, k, axis_len, beta, &pl.c), "plan_packed_axis");
  return pl;
}
// choose_panel, plan.hpp:209-224
inline std::uint64_t choose_panel(std::uint32_t p, std::uint64_t k, int beta = 53) {
  std::uint64_t out = 0;
  check(qg_choose_panel(p, k, beta, &out), "choose_panel");
  return out;
}
// The GPU planner: (t, e, k-block) chosen for the tensor-core path.
inline GpuPlan plan_gpu(std::uint32_t p, std::uint64_t k) {
  GpuPlan g;
  check(qg_plan_gpu(p, k, &g.c), "plan_gpu");
  return g;
}

// ------------------------------------------------------------ matrix.hpp:14-26
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

// Packed words of a right-compressed product (CompressedMatrix<DoubleWord>
// of packed_right_product / mul_right_compressed, m x ceil(n/e), matrix.hpp:44-63).
struct CompressedWords {
  std::size_t logical_rows = 0, logical_cols = 0, stored_rows = 0, stored_cols = 0;
  qg_orientation orientation{QG_FORWARD, QG_COLUMN, 1};  // PackOrientation, matrix.hpp:33-39
  CompressionPlan plan;
  std::vector<double> data;
};

namespace detail {
inline void check_inner_dims(const ResidueMatrix& a, const ResidueMatrix& b) {  // gemm.hpp:22-27
  if (a.cols != b.rows)
    throw DimensionMismatch("inner dimensions disagree: " + std::to_string(a.rows) + "x" +
                            std::to_string(a.cols) + " times " + std::to_string(b.rows) + "x" +
                            std::to_string(b.cols));
}
}  // namespace detail

// ------------------------------------------------------------ gemm.hpp entry points
// mul_common_compressed(A, B, plan), gemm.hpp:254-260: on the device, k-blocked
// for exactness where the plan requires it.
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b,
                                           const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_mul_common(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
        "mul_common_compressed");
  return c;
}
// Same product under a GPU plan: k may exceed plan().kmax() (in-kernel k-blocks).
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b,
                                           const GpuPlan& plan) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_mul_common_gpu(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
        "mul_common_compressed");
  return c;
}
// The same over several GPUs of this process (qg_host_mul_common_multi): rows
// of A and C sharded over `devices`, the packed B broadcast over NCCL.
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const GpuPlan& plan,
                                           const std::vector<int>& devices) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_mul_common_multi(&plan.c, devices.data(), (int)devices.size(), a.data.data(), b.data.data(), a.rows,
                                 a.cols, b.cols, c.data.data()),
        "mul_common_compressed");
  return c;
}
// blocked_accumulate, gemm.hpp:450-489.
inline ResidueMatrix blocked_accumulate(const ResidueMatrix& a, const ResidueMatrix& b,
                                        const CompressionPlan& plan, std::size_t kpanel) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_blocked_accumulate(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, kpanel,
                                   c.data.data()),
        "blocked_accumulate");
  return c;
}
// mul_right_compressed(A, compress_outer_cols(B, plan)), gemm.hpp:320-325:
// the post-REDQ words, bit-identical to the reference's.
inline CompressedWords mul_right_compressed(const ResidueMatrix& a, const ResidueMatrix& b,
                                            const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  CompressedWords cc;
  cc.logical_rows = cc.stored_rows = a.rows;
  cc.logical_cols = b.cols;
  cc.stored_cols = (b.cols + plan.e() - 1) / plan.e();
  cc.orientation = qg_orientation{QG_FORWARD, QG_COLUMN, plan.e()};
  cc.plan = plan;
  cc.data.resize(cc.stored_rows * cc.stored_cols);
  check(qg_host_mul_right(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, cc.data.data()),
        "mul_right_compressed");
  return cc;
}

// mul_left_compressed(compress_outer_rows(A, plan), B), gemm.hpp:340-371:
// ceil(m/e) x n post-REDQ words, {Forward, Row, e}.
inline CompressedWords mul_left_compressed(const ResidueMatrix& a, const ResidueMatrix& b,
                                           const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  CompressedWords cc;
  cc.logical_rows = a.rows;
  cc.logical_cols = cc.stored_cols = b.cols;
  cc.stored_rows = (a.rows + plan.e() - 1) / plan.e();
  cc.orientation = qg_orientation{QG_FORWARD, QG_ROW, plan.e()};
  cc.plan = plan;
  cc.data.resize(cc.stored_rows * cc.stored_cols);
  check(qg_host_mul_left(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, cc.data.data()),
        "mul_left_compressed");
  return cc;
}

// uncompress, gemm.hpp:182-204 (on the device).
inline ResidueMatrix uncompress(const CompressedWords& cm) {
  ResidueMatrix c(cm.logical_rows, cm.logical_cols);
  check(qg_host_uncompress(&cm.plan.c, cm.orientation, cm.data.data(), cm.stored_rows, cm.stored_cols,
                           cm.logical_rows, cm.logical_cols, c.data.data()),
        "uncompress");
  return c;
}

// FullPlan, plan.hpp:44-57, and plan_full, plan.hpp:229-252.
struct FullPlan {
  qg_full_plan c{};
  CompressionPlan base() const { return CompressionPlan{c.base}; }
  int dq() const { return c.dq; }
  int dtheta() const { return c.dtheta; }
  int theta_exponent() const { return c.theta_exponent; }
  int q_slots() const { return c.dq + 1; }
  int theta_slots() const { return c.dtheta + 1; }
};
inline FullPlan plan_full(std::uint32_t p, std::uint64_t k, int beta = 53) {
  FullPlan fp;
  check(qg_plan_full(p, k, beta, &fp.c), "plan_full");
  return fp;
}
// mul_full_compressed(A, B, fp), gemm.hpp:377-445.
inline ResidueMatrix mul_full_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const FullPlan& fp) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_mul_full(&fp.c, 0, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
        "mul_full_compressed");
  return c;
}

// naive_gemm, gemm.hpp:80-100 (a plain device kernel, no packing).
inline ResidueMatrix naive_gemm(const ResidueMatrix& a, const ResidueMatrix& b, std::uint32_t p) {
  detail::check_inner_dims(a, b);
  ResidueMatrix c(a.rows, b.cols);
  check(qg_host_naive_gemm(p, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()), "naive_gemm");
  return c;
}

// PhaseSeconds of the last product call on this thread (see qg_last_phase_seconds).
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

// ------------------------------------------------------------ plan.hpp:59-78
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
// The same seeded matrix as the reference's, generated on the device.
inline ResidueMatrix random_residue_matrix(std::size_t rows, std::size_t cols, std::uint32_t p, std::uint64_t seed) {
  ResidueMatrix m(rows, cols);
  check(qg_host_random_residue_matrix(rows, cols, p, seed, m.data.data()), "random_residue_matrix");
  return m;
}

// ------------------------------------------------------------ matrix_io.hpp:14-77
struct MatrixFile {
  std::uint32_t p = 0;
  ResidueMatrix matrix;
};
namespace detail {
inline MatrixFile adopt(int status, const char* where, std::uint32_t p, std::size_t rows, std::size_t cols,
                        std::uint32_t* data) {
  if (status != QG_OK) {
    const std::string msg = qg_last_error();
    if (status == QG_PARSE_ERROR) throw ParseError(msg);
    check(status, where);
  }
  MatrixFile mf;
  mf.p = p;
  mf.matrix = ResidueMatrix(rows, cols);
  if (rows * cols != 0) std::copy(data, data + rows * cols, mf.matrix.data.begin());
  qg_free(data);
  return mf;
}
}  // namespace detail
inline MatrixFile read_matrix_text(const std::string& text) {
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
inline void write_matrix_file(const std::string& path, const ResidueMatrix& m, std::uint32_t p) {
  const int st = qg_write_matrix_file(path.c_str(), p, m.data.data(), m.rows, m.cols);
  if (st == QG_PARSE_ERROR) throw ParseError(qg_last_error());
  check(st, "write_matrix_file");
}

// ------------------------------------------------------------ bench.hpp:19-41
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
  char buf[64];
  std::string s = r.algorithm + ',' + std::to_string(r.p) + ',' + std::to_string(r.m) + ',' + std::to_string(r.k) +
                  ',' + std::to_string(r.n) + ',' + std::to_string(r.t) + ',' + std::to_string(r.e) + ',';
  std::snprintf(buf, sizeof buf, "%.6f,%.6f,", r.seconds_multiply, r.seconds_convert);
  return s + buf + std::to_string(r.checksum);
}

// ------------------------------------------------------------ word backends
// word.hpp:10-54. Without a template argument every entry point above runs
// the DoubleWord backend (the FP64 tensor-core path); mul_*<Int64Word>(...)
// runs the reference's Int64Word semantics (uint64 words, wrapping products,
// beta up to 63) on the device's integer pipes.
struct DoubleWord {
  static constexpr int exact_bits = 53;
};
struct Int64Word {
  static constexpr int exact_bits = 63;
};

// Words of an Int64Word right/left product (CompressedMatrix<Int64Word>).
struct CompressedWords64 {
  std::size_t logical_rows = 0, logical_cols = 0, stored_rows = 0, stored_cols = 0;
  qg_orientation orientation{QG_FORWARD, QG_COLUMN, 1};
  CompressionPlan plan;
  std::vector<std::uint64_t> data;
};

template <class B>
inline ResidueMatrix mul_common_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan) {
  if constexpr (std::is_same_v<B, Int64Word>) {
    detail::check_inner_dims(a, b);
    ResidueMatrix c(a.rows, b.cols);
    check(qg_host_mul_common_i64(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
          "mul_common_compressed<Int64Word>");
    return c;
  } else {
    return mul_common_compressed(a, b, plan);
  }
}
template <class B>
inline ResidueMatrix blocked_accumulate(const ResidueMatrix& a, const ResidueMatrix& b, const CompressionPlan& plan,
                                        std::size_t kpanel) {
  if constexpr (std::is_same_v<B, Int64Word>) {
    detail::check_inner_dims(a, b);
    ResidueMatrix c(a.rows, b.cols);
    check(qg_host_blocked_accumulate_i64(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, kpanel,
                                         c.data.data()),
          "blocked_accumulate<Int64Word>");
    return c;
  } else {
    return blocked_accumulate(a, b, plan, kpanel);
  }
}
template <class B>
inline ResidueMatrix mul_full_compressed(const ResidueMatrix& a, const ResidueMatrix& b, const FullPlan& fp) {
  if constexpr (std::is_same_v<B, Int64Word>) {
    detail::check_inner_dims(a, b);
    ResidueMatrix c(a.rows, b.cols);
    check(qg_host_mul_full_i64(&fp.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, c.data.data()),
          "mul_full_compressed<Int64Word>");
    return c;
  } else {
    return mul_full_compressed(a, b, fp);
  }
}
// mul_right_compressed / mul_left_compressed <Int64Word>: post-REDQ uint64 words
inline CompressedWords64 mul_right_compressed_i64(const ResidueMatrix& a, const ResidueMatrix& b,
                                                  const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  CompressedWords64 cc;
  cc.logical_rows = cc.stored_rows = a.rows;
  cc.logical_cols = b.cols;
  cc.stored_cols = (b.cols + plan.e() - 1) / plan.e();
  cc.orientation = qg_orientation{QG_FORWARD, QG_COLUMN, plan.e()};
  cc.plan = plan;
  cc.data.resize(cc.stored_rows * cc.stored_cols);
  check(qg_host_mul_right_i64(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, cc.data.data()),
        "mul_right_compressed<Int64Word>");
  return cc;
}
inline CompressedWords64 mul_left_compressed_i64(const ResidueMatrix& a, const ResidueMatrix& b,
                                                 const CompressionPlan& plan) {
  detail::check_inner_dims(a, b);
  CompressedWords64 cc;
  cc.logical_rows = a.rows;
  cc.logical_cols = cc.stored_cols = b.cols;
  cc.stored_rows = (a.rows + plan.e() - 1) / plan.e();
  cc.orientation = qg_orientation{QG_FORWARD, QG_ROW, plan.e()};
  cc.plan = plan;
  cc.data.resize(cc.stored_rows * cc.stored_cols);
  check(qg_host_mul_left_i64(&plan.c, a.data.data(), b.data.data(), a.rows, a.cols, b.cols, cc.data.data()),
        "mul_left_compressed<Int64Word>");
  return cc;
}
inline ResidueMatrix uncompress(const CompressedWords64& cm) {
  ResidueMatrix c(cm.logical_rows, cm.logical_cols);
  check(qg_host_uncompress_u64(&cm.plan.c, cm.orientation, cm.data.data(), cm.stored_rows, cm.stored_cols,
                               cm.logical_rows, cm.logical_cols, c.data.data()),
        "uncompress<Int64Word>");
  return c;
}

// residue_checksum, bench.hpp:43-47.
inline std::uint32_t residue_checksum(const ResidueMatrix& m) {
  std::uint32_t s = 0;
  for (Residue v : m.data) s += v;
  return s;
}

}  // namespace qgemm_b200
