// ref_harness.cpp — C-ABI wrapper around the UNMODIFIED reference headers
// (/root/reference/proj/include/qgemm, included read-only via -I; nothing is
// copied). Built by oracle/Makefile into oracle/_ref/libqgref.so.
//
// TEST INFRASTRUCTURE ONLY: used (a) to pin the C restatement
// (oracle/qg_oracle.c) and generate tests/golden/, and (b) as bench.py's CPU
// baseline ("kind": "reference"): the reference's own dot-product path
// compress_rows_reversed -> compress_cols_forward -> packed_common_product ->
// reduce_common_entry (bench.hpp:127-146), with output rows sharded over host
// threads exactly as SURVEY.md §6 did (each thread runs the unmodified
// routines on its row shard; CB is packed once).
#include <chrono>
#include <sstream>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "qgemm/qgemm.hpp"
#include "qg_oracle.h"  // for the qgo_plan / status layout only

using namespace qgemm;

namespace {

int status_of(const std::exception& ex) {
  if (dynamic_cast<const InvalidModulus*>(&ex)) return QGO_INVALID_MODULUS;
  if (dynamic_cast<const NoCompression*>(&ex)) return QGO_NO_COMPRESSION;
  if (dynamic_cast<const SlotOverflow*>(&ex)) return QGO_SLOT_OVERFLOW;
  if (dynamic_cast<const DigitOverflow*>(&ex)) return QGO_DIGIT_OVERFLOW;
  if (dynamic_cast<const DimensionMismatch*>(&ex)) return QGO_DIMENSION_MISMATCH;
  if (dynamic_cast<const PlanMismatch*>(&ex)) return QGO_PLAN_MISMATCH;
  if (dynamic_cast<const UnsupportedAlgorithm*>(&ex)) return QGO_UNSUPPORTED_ALGORITHM;
  if (dynamic_cast<const ParseError*>(&ex)) return QGO_PARSE_ERROR;
  if (dynamic_cast<const std::invalid_argument*>(&ex)) return QGO_INVALID_ARGUMENT;
  return 99;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return QGO_OK;
  } catch (const std::exception& ex) {
    return status_of(ex);
  }
}

void export_plan(const CompressionPlan& p, qgo_plan* out) {
  std::memset(out, 0, sizeof *out);
  out->p = p.p();
  out->t = p.t;
  out->d = p.d;
  out->e = p.e;
  out->beta = p.beta;
  out->kmax = p.kmax;
  out->inv_qd = p.inv_qd;
  out->extraction = p.extraction == ExtractionMode::AddHighBits ? 1 : 0;
}

CompressionPlan import_plan(const qgo_plan* in) {
  CompressionPlan p{PrimeModulus(in->p)};
  p.t = in->t;
  p.d = in->d;
  p.e = in->e;
  p.beta = in->beta;
  p.kmax = in->kmax;
  p.inv_qd = in->inv_qd;
  p.extraction = in->extraction ? ExtractionMode::AddHighBits : ExtractionMode::ReciprocalMul;
  return p;
}

ResidueMatrix wrap(const uint32_t* v, size_t rows, size_t cols) {
  ResidueMatrix m(rows, cols);
  std::memcpy(m.data.data(), v, rows * cols * sizeof(uint32_t));
  return m;
}

template <class T>
void copy_words(const CompressedMatrix<DoubleWord>& cm, T* out) {
  for (size_t i = 0; i < cm.data.size(); ++i) out[i] = cm.data[i].value;
}

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

template <class F>
void shard_rows(size_t rows, int threads, F&& f) {
  if (threads <= 1 || rows < 2) {
    f(0, rows);
    return;
  }
  if (size_t(threads) > rows) threads = int(rows);
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] { f(rows * t / threads, rows * (t + 1) / threads); });
  for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int qgref_plan_compression(uint32_t p, uint64_t k, int beta, int mode, qgo_plan* out) {
  return guarded([&] {
    export_plan(plan_compression(PrimeModulus(p), k, beta,
                                 mode ? ExtractionMode::AddHighBits : ExtractionMode::ReciprocalMul),
                out);
  });
}

int qgref_uncompressed_plan(uint32_t p, uint64_t k, int beta, qgo_plan* out) {
  return guarded([&] { export_plan(uncompressed_plan(PrimeModulus(p), k, beta), out); });
}

int qgref_plan_packed_axis(uint32_t p, uint64_t k, uint64_t axis, int beta, qgo_plan* out) {
  return guarded([&] { export_plan(plan_packed_axis(PrimeModulus(p), k, axis, beta), out); });
}

int qgref_choose_panel(uint32_t p, uint64_t k, int beta, uint64_t* out) {
  return guarded([&] { *out = choose_panel(PrimeModulus(p), k, beta); });
}

void qgref_random_residue_matrix(size_t rows, size_t cols, uint32_t p, uint64_t seed, uint32_t* out) {
  const ResidueMatrix m = random_residue_matrix(rows, cols, PrimeModulus(p), seed);
  std::memcpy(out, m.data.data(), rows * cols * sizeof(uint32_t));
}

int qgref_compress_forward(const qgo_plan* plan, const uint32_t* v, size_t len, double* out) {
  return guarded([&] {
    *out = compress_forward<DoubleWord>(std::span<const Residue>(v, len), import_plan(plan)).value;
  });
}

int qgref_compress_reverse(const qgo_plan* plan, const uint32_t* v, size_t len, double* out) {
  return guarded([&] {
    *out = compress_reverse<DoubleWord>(std::span<const Residue>(v, len), import_plan(plan)).value;
  });
}

int qgref_extract_coefficient(const qgo_plan* plan, double w, uint32_t* out) {
  return guarded([&] { *out = extract_coefficient(PackedWord<DoubleWord>{w}, import_plan(plan)); });
}

int qgref_extract_all(const qgo_plan* plan, double w, uint64_t* digits) {
  return guarded([&] {
    const auto d = extract_all(PackedWord<DoubleWord>{w}, import_plan(plan));
    for (size_t i = 0; i < d.size(); ++i) digits[i] = d[i];
  });
}

int qgref_redq(const qgo_plan* plan, double w, double* out) {
  return guarded([&] { *out = redq(PackedWord<DoubleWord>{w}, import_plan(plan)).value; });
}

int qgref_compress_rows_reversed(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k, double* out) {
  return guarded([&] { copy_words(compress_rows_reversed<DoubleWord>(wrap(a, m, k), import_plan(plan)), out); });
}

int qgref_compress_cols_forward(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n, double* out) {
  return guarded([&] { copy_words(compress_cols_forward<DoubleWord>(wrap(b, k, n), import_plan(plan)), out); });
}

int qgref_compress_outer_cols(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n, double* out) {
  return guarded([&] { copy_words(compress_outer_cols<DoubleWord>(wrap(b, k, n), import_plan(plan)), out); });
}

int qgref_compress_outer_rows(const qgo_plan* plan, const uint32_t* a, size_t m, size_t k, double* out) {
  return guarded([&] { copy_words(compress_outer_rows<DoubleWord>(wrap(a, m, k), import_plan(plan)), out); });
}

// packed_common_product on reference-packed operands: the pre-mask accumulators.
int qgref_packed_common_product(const qgo_plan* plan, const uint32_t* a, const uint32_t* b,
                                size_t m, size_t k, size_t n, double* acc) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const auto ca = compress_rows_reversed<DoubleWord>(wrap(a, m, k), pl);
    const auto cb = compress_cols_forward<DoubleWord>(wrap(b, k, n), pl);
    const auto w = packed_common_product(ca, cb);
    for (size_t i = 0; i < w.size(); ++i) acc[i] = w[i].value;
  });
}

// The reference's dot-product path (bench.hpp:127-146), rows sharded over threads.
int qgref_mul_common(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                     size_t k, size_t n, uint32_t* c, int threads, double* sec_multiply,
                     double* sec_convert) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const ResidueMatrix bm = wrap(b, k, n);
    double conv = 0, mul = 0;
    auto t0 = std::chrono::steady_clock::now();
    const auto cb = compress_cols_forward<DoubleWord>(bm, pl);
    conv += seconds_since(t0);
    // per-shard phase times; the wall clock of the slowest shard is what counts
    std::vector<double> shard_conv(threads > 0 ? threads : 1, 0.0), shard_mul(threads > 0 ? threads : 1, 0.0);
    const int nth = threads > 0 ? threads : 1;
    auto body = [&](size_t r0, size_t r1) {
      if (r0 >= r1) return;
      const int slot = int(r0 * nth / (m ? m : 1));
      auto s0 = std::chrono::steady_clock::now();
      ResidueMatrix as(r1 - r0, k);
      std::memcpy(as.data.data(), a + r0 * k, (r1 - r0) * k * sizeof(uint32_t));
      const auto ca = compress_rows_reversed<DoubleWord>(as, pl);
      double cv = seconds_since(s0);
      s0 = std::chrono::steady_clock::now();
      const auto acc = packed_common_product(ca, cb);
      double mu = seconds_since(s0);
      s0 = std::chrono::steady_clock::now();
      for (size_t i = 0; i < acc.size(); ++i) c[r0 * n + i] = reduce_common_entry(acc[i], pl);
      cv += seconds_since(s0);
      shard_conv[slot < nth ? slot : nth - 1] = cv;
      shard_mul[slot < nth ? slot : nth - 1] = mu;
    };
    t0 = std::chrono::steady_clock::now();
    shard_rows(m, nth, body);
    const double wall = seconds_since(t0);
    double mx_mul = 0;
    for (double v : shard_mul) mx_mul = v > mx_mul ? v : mx_mul;
    mul = mx_mul;
    conv += wall - mx_mul;
    if (sec_multiply) *sec_multiply = mul;
    if (sec_convert) *sec_convert = conv;
  });
}

// The same dot-product path with the packed B kept between calls, so that a
// row sample can be charged its pro-rata share of compress_cols_forward(B)
// (a full-size run packs B once for all m rows, bench.hpp:127-146):
//   qgref_cb_create  packs B (the reference's single-threaded call) and
//                    reports its seconds;
//   qgref_mul_common_cb  compress_rows_reversed + packed_common_product +
//                    reduce_common_entry on `m` rows, sharded over threads.
void* qgref_cb_create(const qgo_plan* plan, const uint32_t* b, size_t k, size_t n, double* sec_pack) {
  CompressedMatrix<DoubleWord>* out = nullptr;
  const int st = guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const ResidueMatrix bm = wrap(b, k, n);
    const auto t0 = std::chrono::steady_clock::now();
    out = new CompressedMatrix<DoubleWord>(compress_cols_forward<DoubleWord>(bm, pl));
    if (sec_pack) *sec_pack = seconds_since(t0);
  });
  return st == QGO_OK ? out : nullptr;
}

void qgref_cb_free(void* cb) { delete static_cast<CompressedMatrix<DoubleWord>*>(cb); }

int qgref_mul_common_cb(const qgo_plan* plan, const void* cbh, const uint32_t* a, size_t m, size_t k,
                        uint32_t* c, int threads, double* sec_wall) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const auto& cb = *static_cast<const CompressedMatrix<DoubleWord>*>(cbh);
    const size_t n = cb.logical_cols;
    const int nth = threads > 0 ? threads : 1;
    const auto t0 = std::chrono::steady_clock::now();
    shard_rows(m, nth, [&](size_t r0, size_t r1) {
      if (r0 >= r1) return;
      ResidueMatrix as(r1 - r0, k);
      std::memcpy(as.data.data(), a + r0 * k, (r1 - r0) * k * sizeof(uint32_t));
      const auto ca = compress_rows_reversed<DoubleWord>(as, pl);
      const auto acc = packed_common_product(ca, cb);
      for (size_t i = 0; i < acc.size(); ++i) c[r0 * n + i] = reduce_common_entry(acc[i], pl);
    });
    if (sec_wall) *sec_wall = seconds_since(t0);
  });
}

// Mixed/right variant (bench.hpp:148-165): compress_outer_cols, packed_right_product,
// redq_in_place; cc gets the post-REDQ words (m x ceil(n/e)), c (optional) the uncompressed C.
int qgref_mul_right(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                    size_t k, size_t n, double* cc, uint32_t* c, int threads,
                    double* sec_multiply, double* sec_convert) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    auto t0 = std::chrono::steady_clock::now();
    const auto cb = compress_outer_cols<DoubleWord>(wrap(b, k, n), pl);
    double conv = seconds_since(t0);
    const size_t h = cb.stored_cols;
    std::vector<double> mul_s(threads > 0 ? threads : 1, 0.0);
    const int nth = threads > 0 ? threads : 1;
    t0 = std::chrono::steady_clock::now();
    shard_rows(m, nth, [&](size_t r0, size_t r1) {
      if (r0 >= r1) return;
      const int slot = int(r0 * nth / (m ? m : 1));
      ResidueMatrix as(r1 - r0, k);
      std::memcpy(as.data.data(), a + r0 * k, (r1 - r0) * k * sizeof(uint32_t));
      auto s0 = std::chrono::steady_clock::now();
      auto part = packed_right_product(as, cb);
      mul_s[slot < nth ? slot : nth - 1] = seconds_since(s0);
      redq_in_place(part);
      for (size_t i = 0; i < part.data.size(); ++i) cc[r0 * h + i] = part.data[i].value;
      if (c) {
        const ResidueMatrix u = uncompress(part);
        std::memcpy(c + r0 * n, u.data.data(), u.data.size() * sizeof(uint32_t));
      }
    });
    const double wall = seconds_since(t0);
    double mx = 0;
    for (double v : mul_s) mx = v > mx ? v : mx;
    if (sec_multiply) *sec_multiply = mx;
    if (sec_convert) *sec_convert = conv + wall - mx;
  });
}

int qgref_plan_full(uint32_t p, uint64_t k, int beta, qgo_full_plan* out) {
  return guarded([&] {
    const FullPlan fp = plan_full(PrimeModulus(p), k, beta);
    export_plan(fp.base, &out->base);
    out->dq = fp.dq;
    out->dtheta = fp.dtheta;
    out->theta_exponent = fp.theta_exponent;
  });
}

// mul_left_compressed(compress_outer_rows(A, plan), B), gemm.hpp:366-371: post-REDQ words.
int qgref_mul_left(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                   double* cc) {
  return guarded([&] {
    const auto ca = compress_outer_rows<DoubleWord>(wrap(a, m, k), import_plan(plan));
    const auto r = mul_left_compressed(ca, wrap(b, k, n));
    for (size_t i = 0; i < r.data.size(); ++i) cc[i] = r.data[i].value;
  });
}

// mul_full_compressed, gemm.hpp:377-445.
int qgref_mul_full(const qgo_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                   uint32_t* c) {
  return guarded([&] {
    FullPlan f{import_plan(&fp->base), fp->dq, fp->dtheta, fp->theta_exponent};
    const auto r = mul_full_compressed<DoubleWord>(wrap(a, m, k), wrap(b, k, n), f);
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

// read_matrix / write_matrix, matrix_io.hpp:27-75 (to pin the file format).
int qgref_parse_matrix(const char* text, size_t len, uint32_t* p, size_t* rows, size_t* cols, uint32_t* data,
                       size_t cap, char* msg, size_t msglen) {
  try {
    std::istringstream in(std::string(text, len));
    const MatrixFile mf = read_matrix(in);
    *p = mf.p;
    *rows = mf.matrix.rows;
    *cols = mf.matrix.cols;
    for (size_t i = 0; i < mf.matrix.data.size() && i < cap; ++i) data[i] = mf.matrix.data[i];
    return QGO_OK;
  } catch (const std::exception& ex) {
    std::snprintf(msg, msglen, "%s", ex.what());
    return status_of(ex);
  }
}

size_t qgref_write_matrix(const uint32_t* data, size_t rows, size_t cols, uint32_t p, char* out, size_t cap) {
  std::ostringstream os;
  write_matrix(os, wrap(data, rows, cols), p);
  const std::string s = os.str();
  if (s.size() <= cap) std::memcpy(out, s.data(), s.size());
  return s.size();
}

// ---- Int64Word instantiations (word.hpp:36-54), to pin the i64 restatement
// kind 0 rows_reversed, 1 cols_forward, 2 outer_cols, 3 outer_rows
int qgref_pack_i64(int kind, const qgo_plan* plan, const uint32_t* src, size_t rows, size_t cols, uint64_t* out) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const ResidueMatrix m = wrap(src, rows, cols);
    CompressedMatrix<Int64Word> cm = kind == 0   ? compress_rows_reversed<Int64Word>(m, pl)
                                     : kind == 1 ? compress_cols_forward<Int64Word>(m, pl)
                                     : kind == 2 ? compress_outer_cols<Int64Word>(m, pl)
                                                 : compress_outer_rows<Int64Word>(m, pl);
    for (size_t i = 0; i < cm.data.size(); ++i) out[i] = cm.data[i].value;
  });
}

int qgref_common_i64(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                     uint64_t* acc, uint32_t* c) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const auto ca = compress_rows_reversed<Int64Word>(wrap(a, m, k), pl);
    const auto cb = compress_cols_forward<Int64Word>(wrap(b, k, n), pl);
    const auto w = packed_common_product(ca, cb);
    for (size_t i = 0; i < w.size(); ++i) acc[i] = w[i].value;
    const ResidueMatrix r = mul_common_compressed<Int64Word>(wrap(a, m, k), wrap(b, k, n), pl);
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

int qgref_right_i64(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                    uint64_t* pre, uint64_t* cc) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const auto cbo = compress_outer_cols<Int64Word>(wrap(b, k, n), pl);
    const auto p0 = packed_right_product(wrap(a, m, k), cbo);
    for (size_t i = 0; i < p0.data.size(); ++i) pre[i] = p0.data[i].value;
    const auto r = mul_right_compressed(wrap(a, m, k), cbo);
    for (size_t i = 0; i < r.data.size(); ++i) cc[i] = r.data[i].value;
  });
}

int qgref_left_i64(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                   uint64_t* pre, uint64_t* cc) {
  return guarded([&] {
    const CompressionPlan pl = import_plan(plan);
    const auto ca = compress_outer_rows<Int64Word>(wrap(a, m, k), pl);
    const auto p0 = packed_left_product(ca, wrap(b, k, n));
    for (size_t i = 0; i < p0.data.size(); ++i) pre[i] = p0.data[i].value;
    const auto r = mul_left_compressed(ca, wrap(b, k, n));
    for (size_t i = 0; i < r.data.size(); ++i) cc[i] = r.data[i].value;
  });
}

int qgref_full_i64(const qgo_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                   uint32_t* c) {
  return guarded([&] {
    FullPlan f{import_plan(&fp->base), fp->dq, fp->dtheta, fp->theta_exponent};
    const auto r = mul_full_compressed<Int64Word>(wrap(a, m, k), wrap(b, k, n), f);
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

int qgref_blocked_i64(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                      size_t kpanel, uint32_t* c) {
  return guarded([&] {
    const auto r = blocked_accumulate<Int64Word>(wrap(a, m, k), wrap(b, k, n), import_plan(plan), kpanel);
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

int qgref_extract_i64(const qgo_plan* plan, uint64_t w, uint32_t* out) {
  return guarded([&] { *out = extract_coefficient(PackedWord<Int64Word>{w}, import_plan(plan)); });
}

int qgref_redq_i64(const qgo_plan* plan, uint64_t w, uint64_t* out) {
  return guarded([&] { *out = redq(PackedWord<Int64Word>{w}, import_plan(plan)).value; });
}

int qgref_blocked_accumulate(const qgo_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                             size_t k, size_t n, size_t kpanel, uint32_t* c) {
  return guarded([&] {
    const auto r = blocked_accumulate<DoubleWord>(wrap(a, m, k), wrap(b, k, n), import_plan(plan), kpanel);
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

int qgref_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                     size_t n, uint32_t* c) {
  return guarded([&] {
    const auto r = naive_gemm(wrap(a, m, k), wrap(b, k, n), PrimeModulus(p));
    std::memcpy(c, r.data.data(), r.data.size() * sizeof(uint32_t));
  });
}

}  // extern "C"
