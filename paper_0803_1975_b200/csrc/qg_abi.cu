// qg_abi.cu — the C ABI (include/qgemm_b200.h): argument checks in the
// reference's order, plan -> kernel dispatch, and the host-buffer entry points.
// Every computation is a kernel launch on the caller's stream; nothing here
// computes results on the CPU.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <vector>

#include "../../include/qgemm_b200.h"
#include "qg_internal.h"
#include "qg_kernels.h"
#include "qg_stage.h"

namespace qg {
bool is_prime(uint64_t n);
uint64_t max_exact_block(uint32_t p, int t, int e);
uint64_t stage_block(uint64_t limit, int* bk);
uint64_t stage_block_tiled(uint64_t limit, int* bk);
uint64_t stage_block_redq(uint64_t limit, int* bk);
int stage_single(uint64_t K);
uint64_t max_exact_block_balanced(uint32_t p, int t, int e);
uint64_t max_exact_block_anchored(uint32_t p, int t, int e);
int anchored_exponent(uint32_t p, int t, int e, uint64_t kb);
int anchored_stage(uint64_t kb);
uint64_t largest_common_dim(uint32_t p, int t);
uint64_t largest_common_dim_balanced(uint32_t p, int t);
}  // namespace qg

namespace qgk {
static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
}  // namespace qgk

namespace {

thread_local const char* g_last_kernel = "none";
thread_local cudaError_t g_last_cuda_error = cudaSuccess;

int cuda_status(cudaError_t e) {
  if (e == cudaSuccess) return QG_OK;
  g_last_cuda_error = e;
  qg::last_message() = cudaGetErrorString(e);
  return QG_CUDA_ERROR;
}
cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
#define QG_TRY(x)                       \
  do {                                  \
    cudaError_t e_ = (x);               \
    if (e_ != cudaSuccess) return cuda_status(e_); \
  } while (0)
size_t ceil_div(size_t a, size_t b) { return (a + b - 1) / b; }

// CompressionPlan usable by the DoubleWord backend (pack.hpp:19-24).
int check_plan(const qg_plan* plan) {
  if (!plan) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !qg::is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->beta > 53) return QG_PLAN_MISMATCH;
  if (plan->t < 1 || plan->e < 1 || plan->d != plan->e - 1 || plan->t * plan->e > 63)
    return QG_PLAN_MISMATCH;
  return QG_OK;
}

// kernel arguments carry dimensions as int: larger ones are refused, not wrapped
// Eq. 3 bound of a GPU plan, recomputed from (p, t) instead of trusting the
// struct's kmax field: balanced digits (|v| <= p/2) have their own, ~4x
// larger bound; an unsigned plan keeps a caller's smaller kmax (the
// AddHighBits reduction, plan.hpp:150-157) but never exceeds plan.hpp:113-115.
uint64_t gpu_kmax(const qg_gpu_plan* gp) {
  const qg_plan& pl = gp->plan;
  if (gp->balanced) return qg::largest_common_dim_balanced(pl.p, pl.t);
  const uint64_t lcd = qg::largest_common_dim(pl.p, pl.t);
  return pl.kmax < lcd ? pl.kmax : lcd;
}

bool dims_ok(size_t a, size_t b, size_t c = 0) {
  const size_t lim = 0x7FFFFFFF;
  return a <= lim && b <= lim && c <= lim;
}

// stream-ordered device buffer, freed on its stream
struct DevBuf {
  void* p = nullptr;
  cudaStream_t s;
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaError_t alloc(size_t bytes) { return bytes ? cudaMallocAsync(&p, bytes, s) : cudaSuccess; }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, s);
  }
};

int check_dtype(qg_dtype d) { return (d == QG_F64 || d == QG_U32 || d == QG_I32) ? QG_OK : QG_INVALID_ARGUMENT; }

// Device flag for DigitOverflow (redq / extract_all throw it in the reference).
struct DeviceFlag {
  // one persistent device int per host thread: a stream-ordered allocation
  // per call costs a pool map/unmap round trip on every uncompress / redq
  int* ptr = nullptr;
  cudaStream_t s;
  explicit DeviceFlag(cudaStream_t st) : s(st) {
    // keyed by device: a thread may call the library on several GPUs
    static thread_local std::map<int, int*> flags;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return;
    int*& flag = flags[dev];
    if (!flag && cudaMalloc(&flag, sizeof(int)) != cudaSuccess) flag = nullptr;
    ptr = flag;
    if (ptr && cudaMemsetAsync(ptr, 0, sizeof(int), s) != cudaSuccess) ptr = nullptr;
  }
  int read(int* value) {
    int v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, ptr, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
    *value = v;
    return cuda_status(e);
  }
};

// The common-variant contraction, dispatched on the block structure. Blocks
// may always be made shorter than asked (Eq. 3 and Eq. G only get easier), so
// the DMMA kernel runs with blocks of min(kblock, Eq. G bound) words rounded
// down to whole pipeline stages; only when that leaves less than one 4-word
// k-step does the reference's per-product high-part kernel take over.
int run_common(const qg_plan& pl, uint64_t kblock, const double* ca, size_t ldca, const double* cb,
               size_t ldcb, size_t m, size_t n, size_t K, int32_t* c, size_t ldc, cudaStream_t s) {
  if (m == 0 || n == 0) return QG_OK;
  const uint64_t exact = qg::max_exact_block(pl.p, pl.t, pl.e);
  const uint32_t qmask = (uint32_t)((1ull << pl.t) - 1);
  uint64_t kb = kblock < K ? kblock : K;
  if (kb > exact) return QG_NOT_EXACT;  // a block past Eq. G: refused, never clamped silently
  int bk = 32;
  uint64_t blk = K;  // words per k-block
  bool dmma = kb >= K;
  if (!dmma) {
    blk = qg::stage_block(kb, &bk);
    dmma = blk >= 4;
  }
  if (dmma) {
    qgk::GemmArgs a;
    std::memset(&a, 0, sizeof a);
    a.lda = ldca;
    a.b = cb;
    a.ldb = ldcb;
    if (!dims_ok(m, n, K)) return QG_INVALID_ARGUMENT;
    a.M = (int)m;
    a.N = (int)n;
    a.kb_stages = blk >= K ? 0 : (int)(blk / bk);
    a.anchor = std::ldexp(1.0, pl.t * pl.d + 52);
    a.qmask = qmask;
    a.p = pl.p;
    a.c = c;
    a.ldc = ldc;
    // digit sums are uint32: split k into launches of at most this many blocks,
    // each adding its residues onto C (mod p)
    const uint64_t max_blocks = ((1ull << 32) - 1 - pl.p) / (qmask ? qmask : 1);
    const uint64_t chunk_words = a.kb_stages ? max_blocks * blk : K;
    for (uint64_t w0 = 0; w0 < K; w0 += chunk_words) {
      const uint64_t wn = (K - w0) < chunk_words ? (K - w0) : chunk_words;
      a.a = ca + w0;
      a.b = cb + w0 * ldcb;
      a.K = (int)wn;
      a.accumulate = w0 > 0;
      cudaError_t e = qgk::launch_dot_dmma(a, bk, s, &g_last_kernel);
      if (e) return cuda_status(e);
    }
    return QG_OK;
  }
  qgk::HighArgs h;
  h.ca = ca;
  h.ldca = ldca;
  h.cb = cb;
  h.ldcb = ldcb;
  if (!dims_ok(m, n, K)) return QG_INVALID_ARGUMENT;
  h.M = (int)m;
  h.N = (int)n;
  h.K = (int)K;
  h.inv_qd = pl.inv_qd;
  h.kb_words = kblock >= K ? 0 : (int)kblock;
  h.qmask = qmask;
  h.p = pl.p;
  h.acc = nullptr;
  h.c = c;
  h.ldc = ldc;
  return cuda_status(qgk::launch_dot_highpart(h, s, &g_last_kernel));
}

// Tiled path: stage depth and blocks for a plan. Single-block plans take the
// stage depth with the least padded work (qg::stage_single); blocked plans use
// the deepest stage that divides the (Eq. G / Eq. 3) block.
int tiled_geometry(const qg_gpu_plan* gp, uint64_t K, int* bk, int* kb_stages) {
  const qg_plan& pl = gp->plan;
  const uint64_t exact = gp->balanced ? qg::max_exact_block_balanced(pl.p, pl.t, pl.e)
                                      : qg::max_exact_block(pl.p, pl.t, pl.e);
  const uint64_t kb = gp->kblock_words < K ? gp->kblock_words : K;
  if (kb > exact) return QG_NOT_EXACT;  // a block past Eq. G: refused, never clamped silently
  if (gp->anchored && gp->balanced && kb < K) {  // anchored plan: blocks of exactly kb words = the stage depth
    if (!qg::anchored_exponent(pl.p, pl.t, pl.e, kb)) return QG_NOT_EXACT;
    const int b = qg::anchored_stage(kb);
    if (!b) return QG_INVALID_ARGUMENT;
    *bk = b;
    *kb_stages = 1;
    return QG_OK;
  }
  if (kb >= K) {
    const char* e = getenv("QG_TILED_SINGLE_BK");  // experiments
    *bk = e ? atoi(e) : qg::stage_single(K);
    *kb_stages = 0;
    return QG_OK;
  }
  const uint64_t blk = qg::stage_block_tiled(kb, bk);
  if (blk < 4) return QG_NOT_EXACT;
  *kb_stages = (int)(blk / *bk);
  return QG_OK;
}

}  // namespace

extern "C" {

int qg_gpu_plan_kmax(const qg_gpu_plan* gplan, uint64_t* kmax) {
  if (!gplan || !kmax) return QG_INVALID_ARGUMENT;
  int st = check_plan(&gplan->plan);
  if (st) return st;
  *kmax = gpu_kmax(gplan);
  return QG_OK;
}

int qg_tiled_stage_words(const qg_gpu_plan* gplan, uint64_t k, uint32_t* bk) {
  if (!gplan || !bk) return QG_INVALID_ARGUMENT;
  int st = check_plan(&gplan->plan);
  if (st) return st;
  const uint64_t K = ceil_div(k, gplan->plan.e), kb = gplan->kblock_words, kmax = gpu_kmax(gplan);
  if (kb < K && kb * (uint64_t)gplan->plan.e > kmax) return QG_PLAN_MISMATCH;  // Eq. 3 first, as the contraction
  int b = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &b, &kbs))) return st;
  *bk = (uint32_t)b;
  return QG_OK;
}

size_t qg_tiled_words(size_t rows, size_t k, int e, uint32_t bk) {
  if (e < 1 || bk == 0) return 0;
  const size_t K = ceil_div(k, (size_t)e);
  return ceil_div(rows, 128) * 128 * ceil_div(K, bk) * bk;
}

int qg_pack_a_tiled(const qg_gpu_plan* gplan, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k,
                    size_t lda, double* ca_t, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan* plan = &gplan->plan;
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < k) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(false, a, dtype, m, k, lda, plan->t, plan->e, (int)bk, ca_t,
                                            as_stream(stream), plan->p, gplan->balanced != 0));
}

int qg_pack_b_tiled(const qg_gpu_plan* gplan, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n,
                    size_t ldb, double* cb_t, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan* plan = &gplan->plan;
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (ldb < n) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(true, b, dtype, k, n, ldb, plan->t, plan->e, (int)bk, cb_t,
                                            as_stream(stream), plan->p, gplan->balanced != 0));
}

// ---- mixed variant on the tiled layout
static int right_tiled_geometry(const qg_gpu_plan* gp, uint64_t k, int* bk, int* kb_stages) {
  const uint64_t kb = gp->kblock_words;
  if (kb == 0) return QG_INVALID_ARGUMENT;
  if (kb >= k) {
    *bk = 28;
    *kb_stages = 0;
    return QG_OK;
  }
  const uint64_t blk = qg::stage_block_redq(kb, bk);
  if (blk < 4) return QG_INVALID_ARGUMENT;
  *kb_stages = (int)(blk / *bk);
  return QG_OK;
}

int qg_right_tiled_stage(const qg_gpu_plan* gplan, uint64_t k, uint32_t* bk) {
  if (!gplan || !bk) return QG_INVALID_ARGUMENT;
  int b = 0, kbs = 0;
  int st = right_tiled_geometry(gplan, k, &b, &kbs);
  if (st) return st;
  *bk = (uint32_t)b;
  return QG_OK;
}

int qg_pack_residues_tiled(uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda, double* a_t,
                           void* stream) {
  int st = check_dtype(dtype);
  if (st) return st;
  if (lda < k) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(false, a, dtype, m, k, lda, 1, 1, (int)bk, a_t, as_stream(stream)));
}

// the stage depths the REDQ-epilogue kernels and their packs are built for
static bool redq_stage_ok(uint32_t bk) { return bk == 4 || bk == 12 || bk == 20 || bk == 28 || bk == 36; }

int qg_pack_outer_cols_tiled(const qg_plan* plan, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n,
                             size_t ldb, double* bo_t, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (ldb < n || !redq_stage_ok(bk)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_outer_tiled(b, dtype, k, n, ldb, plan->t, plan->e, (int)bk, bo_t,
                                                  as_stream(stream)));
}

// The exact contraction with in-place REDQ shared by the right, left and
// full variants: cc (M x N words) = REDQ(A_t x B_t^T), the accumulators REDQ'd
// every kblock residues of k. Every digit of a block stays below Q while
// (p-1) + kb (p-1)^2 < Q (the previous block's REDQ'd digit plus the block's
// sum); a single block needs k <= kmax (gemm.hpp:295).
static int redq_product(const qg_gpu_plan* gplan, const double* a_t, const double* b_t, size_t M, size_t k,
                        size_t N, double* cc, size_t ldcc, void* stream, bool accumulate = false) {
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if (pl.t * pl.e > 53) return QG_PLAN_MISMATCH;  // sums must stay exact
  const bool bal = gplan->balanced != 0;
  if (bal && (pl.t > 31 || pl.t * pl.e > 52 || pl.t < 2)) return QG_PLAN_MISMATCH;
  const uint64_t h = bal ? pl.p / 2 : pl.p - 1;  // largest |digit| of an operand
  const uint64_t pm = h * h;
  const uint64_t Q = 1ull << pl.t, lim = bal ? Q / 2 : Q;  // digits stay in (-Q/2, Q/2) resp. [0, Q)
  int bk = 0, kbs = 0;
  if ((st = right_tiled_geometry(gplan, k, &bk, &kbs))) return st;
  if (kbs == 0) {
    if (bal ? (uint64_t)k * pm >= lim : k > pl.kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:295 for unsigned
    // continuing from REDQ'd words: their digits (< p) add to the block's sums
    if (accumulate && h + (uint64_t)k * pm >= lim) return QG_PLAN_MISMATCH;
  } else if (h + (uint64_t)gplan->kblock_words * pm >= lim) {
    // the plan's block (before rounding down to whole stages) would overflow
    // a digit after the in-place REDQ: refused, never rounded into range
    return QG_PLAN_MISMATCH;
  }
  if (ldcc < N) return QG_INVALID_ARGUMENT;
  if (M == 0 || N == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  if (k == 0) {
    if (cudaMemset2DAsync(cc, ldcc * sizeof(double), 0, N * sizeof(double), M, s) != cudaSuccess)
      return QG_CUDA_ERROR;
    return QG_OK;
  }
  qgk::GemmArgs r;
  std::memset(&r, 0, sizeof r);
  r.a = a_t;
  r.b = b_t;
  if (!dims_ok(M, N, k)) return QG_INVALID_ARGUMENT;
  r.M = (int)M;
  r.N = (int)N;
  r.K = (int)k;
  r.kb_stages = kbs;
  r.t = pl.t;
  r.e = pl.e;
  r.p = pl.p;
  r.cc = cc;
  r.ldcc = ldcc;
  if (accumulate) {  // start from the (REDQ'd, digits < p) words in cc: unsigned plans only
    if (bal) return QG_PLAN_MISMATCH;
    r.accumulate = 1;
  }
  if (bal) {  // constants of the balanced in-place REDQ (qg_dot.cu, redq_words_inplace_bal)
    r.balanced = 1;
    const uint64_t half = Q / 2;
    uint64_t off = 0;
    for (int d = 0; d < pl.e; ++d) off |= half << (pl.t * d);
    r.redq_off2 = (double)off + 4503599627370496.0;  // exact: off < 2^52
    r.redq_ybias = (uint32_t)((half + pl.p - 1) / pl.p * pl.p - half);
  }
  return cuda_status(qgk::launch_right_tiled(r, bk, true, s, &g_last_kernel));
}

int qg_mul_right_tiled(const qg_gpu_plan* gplan, const double* a_t, const double* bo_t, size_t m, size_t k,
                       size_t n, double* cc, size_t ldcc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  if (gplan->plan.e < 1) return QG_PLAN_MISMATCH;
  return redq_product(gplan, a_t, bo_t, m, k, ceil_div(n, (size_t)gplan->plan.e), cc, ldcc, stream);
}

// ---- left and full compression (gemm.hpp:340-445) on the same contraction

int qg_pack_outer_rows_tiled(const qg_plan* plan, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k,
                             size_t lda, double* ao_t, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < k || !redq_stage_ok(bk)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_outer_rows_tiled(a, dtype, m, k, lda, plan->t, plan->e, (int)bk, ao_t,
                                                       as_stream(stream)));
}

int qg_pack_residues_b_tiled(uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n, size_t ldb,
                             double* b_t, void* stream) {
  int st = check_dtype(dtype);
  if (st) return st;
  if (ldb < n) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(true, b, dtype, k, n, ldb, 1, 1, (int)bk, b_t, as_stream(stream), 2,
                                            false));
}

// Balanced-digit operands for plans with gplan->balanced (residue v enters as
// v - p when v > p/2): the same layouts as the entries above.
int qg_pack_residues_tiled_bal(uint32_t p, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda,
                               double* a_t, void* stream) {
  int st = check_dtype(dtype);
  if (st) return st;
  if (p < 2 || !qg::is_prime(p)) return QG_INVALID_MODULUS;
  if (lda < k) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(false, a, dtype, m, k, lda, 1, 1, (int)bk, a_t, as_stream(stream), p, true));
}
int qg_pack_residues_b_tiled_bal(uint32_t p, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n, size_t ldb,
                                 double* b_t, void* stream) {
  int st = check_dtype(dtype);
  if (st) return st;
  if (p < 2 || !qg::is_prime(p)) return QG_INVALID_MODULUS;
  if (ldb < n) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_tiled(true, b, dtype, k, n, ldb, 1, 1, (int)bk, b_t, as_stream(stream), p, true));
}
int qg_pack_outer_cols_tiled_bal(const qg_plan* plan, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n,
                                 size_t ldb, double* bo_t, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (ldb < n || !redq_stage_ok(bk)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_outer_tiled_bal(b, dtype, k, n, ldb, plan->t, plan->e, (int)bk, bo_t, plan->p,
                                                      as_stream(stream)));
}
int qg_pack_outer_rows_tiled_bal(const qg_plan* plan, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k,
                                 size_t lda, double* ao_t, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < k || !redq_stage_ok(bk)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack_outer_rows_tiled_bal(a, dtype, m, k, lda, plan->t, plan->e, (int)bk, ao_t,
                                                           plan->p, as_stream(stream)));
}

int qg_mul_left_tiled(const qg_gpu_plan* gplan, const double* ao_t, const double* b_t, size_t m, size_t k,
                      size_t n, double* cc, size_t ldcc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  if (gplan->plan.e < 1) return QG_PLAN_MISMATCH;
  return redq_product(gplan, ao_t, b_t, ceil_div(m, (size_t)gplan->plan.e), k, n, cc, ldcc, stream);
}

static int full_gpu_plan(const qg_full_plan* fp, uint64_t kblock_words, uint64_t k, qg_gpu_plan* gp) {
  if (!fp) return QG_INVALID_ARGUMENT;
  int st = check_plan(&fp->base);
  if (st) return st;
  const int qs = fp->dq + 1, ts = fp->dtheta + 1;
  if (qs < 1 || ts < 1 || fp->base.e != qs * ts || fp->theta_exponent != fp->base.t * qs)
    return QG_PLAN_MISMATCH;
  std::memset(gp, 0, sizeof *gp);
  gp->plan = fp->base;
  gp->kblock_words = kblock_words ? kblock_words : (k ? k : 1);
  gp->max_exact_words = gp->kblock_words;
  return QG_OK;
}

int qg_full_tiled_stage(const qg_full_plan* fp, uint64_t kblock_words, uint64_t k, uint32_t* bk) {
  qg_gpu_plan gp;
  int st = full_gpu_plan(fp, kblock_words, k, &gp);
  if (st) return st;
  return qg_right_tiled_stage(&gp, k, bk);
}

int qg_mul_full_tiled(const qg_full_plan* fp, uint64_t kblock_words, const double* ao_t, const double* bo_t,
                      size_t m, size_t k, size_t n, double* cc, size_t ldcc, void* stream) {
  qg_gpu_plan gp;
  int st = full_gpu_plan(fp, kblock_words, k, &gp);
  if (st) return st;
  return redq_product(&gp, ao_t, bo_t, ceil_div(m, (size_t)fp->dq + 1), k, ceil_div(n, (size_t)fp->dtheta + 1),
                      cc, ldcc, stream);
}

int qg_uncompress_full(const qg_full_plan* fp, const double* cc, size_t ldcc, size_t m, size_t n, int32_t* c,
                       size_t ldc, void* stream) {
  qg_gpu_plan gp;
  int st = full_gpu_plan(fp, 0, 1, &gp);
  if (st) return st;
  if (ldc < n || ldcc < ceil_div(n, (size_t)fp->dtheta + 1)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_uncompress_full(cc, ldcc, m, n, fp->base.t, fp->dq + 1, fp->dtheta + 1, fp->base.p,
                                                 c, ldc, as_stream(stream)));
}

}  // extern "C"

namespace {

// Keep freed stream-ordered allocations mapped across calls on this device
// (the default release threshold of 0 re-maps workspaces on every call).
void keep_pool_mapped() {
  static std::atomic<uint64_t> done{0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev >= 64) return;
  if (done.load() & (1ull << dev)) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done.fetch_or(1ull << dev);
}

int device_sms() {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms > 0 ? sms : 148;
}

// The one-launch small path (qg_small.cu) takes products whose 128x128 tiles
// would occupy less than half of the SMs (config 1: 16 tiles), and odd n
// (the tiled epilogue stores column pairs). QG_SMALL=0/1 forces it off/on.
bool use_small_path(size_t m, size_t n) {
  const char* e = getenv("QG_SMALL");
  if (e && e[0] == '0') return n % 2 != 0;
  if (e && e[0] == '1') return true;
  return n % 2 != 0 || ceil_div(m, 128) * ceil_div(n, 128) * 2 < (size_t)device_sms();
}

// Geometry of the small path on a tiled layout of stage depth bk (Kt stages,
// k-blocks of kbs stages): the stages split over a cluster of CTAs (<= 8,
// about one CTA per SM). Blocks restart at split starts; any partition of k
// into pieces of <= the exact block is exact.
void small_geometry(size_t m, size_t n, size_t Kt, int kbs, int* splits, int* split_stages, uint64_t* extractions) {
  const size_t tiles = ceil_div(m, 64) * ceil_div(n, 64);
  size_t S = (size_t)device_sms() / (tiles ? tiles : 1);
  if (const char* e = getenv("QG_SMALL_SPLITS")) S = (size_t)atoi(e);  // experiments
  S = S < 1 ? 1 : (S > 8 ? 8 : S);
  if (S > Kt) S = Kt;
  const size_t Ls = ceil_div(Kt, S);
  S = ceil_div(Kt, Ls);
  uint64_t ex = 0;
  for (size_t s = 0; s < S; ++s) {
    const uint64_t nst = ((s + 1) * Ls < Kt ? (s + 1) * Ls : Kt) - s * Ls;
    ex += kbs ? (nst - 1) / kbs + 1 : 1;
  }
  *splits = (int)S;
  *split_stages = (int)Ls;
  *extractions = ex;
}

}  // namespace

extern "C" {

// K4A (qg_anchor.cu): anchor pair, digit position and block length of an anchored
// plan's contraction; the block was validated by tiled_geometry. The digit sums (scaled by 2^shift)
// of all extractions must fit the kernel's uint32 accumulators.
static int set_anchored_args(const qg_plan& pl, size_t K, uint64_t kb, qgk::GemmArgs* a) {
  const int E = qg::anchored_exponent(pl.p, pl.t, pl.e, kb);
  if (!E) return QG_NOT_EXACT;
  const int sh = pl.t * pl.d - (E - 52);
  a->anchored_kb = (int)kb;
  a->anch_shift = sh;
  a->anchor = std::ldexp(1.5, E) + std::ldexp(1.0, pl.t * pl.d - 1) + std::ldexp(1.0, pl.t * pl.d + pl.t - 1);
  a->anchor1 = a->anchor + std::ldexp(1.0, pl.t * pl.d + pl.t);  // second anchor: + Q^(d+1), above the digit field
  const uint64_t nex = ceil_div(K, (size_t)kb) + 3;  // extractions per output (<= 2 zero blocks + the final one)
  if (((unsigned __int128)nex * a->qmask << sh) + 2 * pl.p >= ((unsigned __int128)1 << 32)) return QG_NOT_EXACT;
  return QG_OK;
}

int qg_mul_common_tiled(const qg_gpu_plan* gplan, const double* ca_t, const double* cb_t, size_t m, size_t n,
                        size_t k, int32_t* c, size_t ldc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if (ldc < n) return QG_INVALID_ARGUMENT;
  // the main kernel stores column pairs; odd n / ldc or an unaligned C take the small kernel
  const bool pairs_ok = !(ldc % 2) && !(n % 2) && ((((uintptr_t)c) & 7) == 0);
  const size_t K = ceil_div(k, pl.e);
  const uint64_t kb = gplan->kblock_words;
  if (kb == 0) return QG_INVALID_ARGUMENT;
  const uint64_t kmax = gpu_kmax(gplan);
  if (kb < K && kb * (uint64_t)pl.e > kmax) return QG_PLAN_MISMATCH;  // Eq. 3 per block
  if (kb >= K && k > kmax) return QG_PLAN_MISMATCH;
  if (m == 0 || n == 0) return QG_OK;
  int bk = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &bk, &kbs))) return st;
  qgk::GemmArgs a;
  std::memset(&a, 0, sizeof a);
  a.a = ca_t;
  a.b = cb_t;
  if (!dims_ok(m, n, K)) return QG_INVALID_ARGUMENT;
  a.M = (int)m;
  a.N = (int)n;
  a.K = (int)K;
  a.kb_stages = kbs;
  a.balanced = gplan->balanced != 0;
  // unsigned: round-toward-zero against 2^(td+52) gives floor(S/Q^d); balanced:
  // round-to-nearest against 1.5*2^(td+52) + Q^d*Q/2 gives round(S/Q^d) + Q/2
  a.anchor = a.balanced ? std::ldexp(1.5, pl.t * pl.d + 52) + std::ldexp(1.0, pl.t * pl.d + pl.t - 1)
                        : std::ldexp(1.0, pl.t * pl.d + 52);
  a.qmask = (uint32_t)((1ull << pl.t) - 1);
  a.p = pl.p;
  a.c = c;
  a.ldc = ldc;
  if (K == 0) {
    for (size_t i = 0; i < m; ++i)
      if (cudaMemsetAsync(c + i * ldc, 0, n * sizeof(int32_t), as_stream(stream)) != cudaSuccess) return QG_CUDA_ERROR;
    return QG_OK;
  }
  if (!pairs_ok || use_small_path(m, n)) {  // 64x64 tiles, k stages split over a cluster (qg_small.cu)
    qgk::SmallArgs sa;
    std::memset(&sa, 0, sizeof sa);
    sa.a = ca_t;
    sa.b = cb_t;
    sa.M = (int)m;
    sa.N = (int)n;
    sa.K = (int)K;
    sa.Kt = (int)ceil_div(K, (size_t)bk);
    sa.balanced = a.balanced;
    sa.kb_stages = kbs;
    sa.anchor = a.anchor;
    sa.qmask = a.qmask;
    sa.p = pl.p;
    sa.c = c;
    sa.ldc = ldc;
    int splits = 1, ls = 1;
    uint64_t ex = 0;
    small_geometry(m, n, (size_t)sa.Kt, kbs, &splits, &ls, &ex);
    sa.split_stages = ls;
    if ((unsigned __int128)ex * sa.qmask + 2 * pl.p >= ((unsigned __int128)1 << 32)) return QG_NOT_EXACT;
    if (sa.balanced) {  // remove the Q/2 bias of every extraction, mod p
      const uint64_t halfq = ((uint64_t)sa.qmask + 1) / 2;
      sa.corr = (uint32_t)((pl.p - (ex % pl.p) * (halfq % pl.p) % pl.p) % pl.p);
    }
    return cuda_status(qgk::launch_small_tiled(sa, bk, splits, as_stream(stream), &g_last_kernel));
  }
  // digit sums are uint32 (planner keeps nblocks * (Q-1) < 2^32); the fused
  // flush packs two per register as 16-bit lanes, reduced mod p in time
  if (gplan->anchored && a.balanced && kb < K) {  // K4A (qg_anchor.cu)
    if ((st = set_anchored_args(pl, K, kb, &a))) return st;
    return cuda_status(qgk::launch_dot_tiled(a, bk, as_stream(stream), &g_last_kernel));
  }
  if (pl.t <= 16) a.pack_period = (int)((65535u - (pl.p - 1)) / a.qmask);
  const uint64_t nblocks = (kbs ? ceil_div(K, (size_t)kbs * bk) : 1) + 1;
  if ((unsigned __int128)nblocks * a.qmask + 2 * pl.p >= ((unsigned __int128)1 << 32)) return QG_NOT_EXACT;
  return cuda_status(qgk::launch_dot_tiled(a, bk, as_stream(stream), &g_last_kernel));
}

// mul_common_repacked, gemm.hpp:275-280, on the tiled layout: C's rows leave
// the contraction as forward-packed words of e adjacent residues
// (ReduceAndCompress, pack.hpp:141-155, under gplan->plan's t and e). The
// 128x128-tile kernel does it in its epilogue (EPI_REPACK: no int32 C in
// HBM); products that take the small cluster kernel, or p >= 256, go through
// an int32 workspace and the outer-cols pack instead.
int qg_mul_common_repacked_tiled(const qg_gpu_plan* gplan, const double* ca_t, const double* cb_t, size_t m,
                                 size_t n, size_t k, double* cc, size_t ldcc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if (pl.t * pl.e > 53) return QG_PLAN_MISMATCH;  // output words must be exact doubles
  const size_t H = ceil_div(n, (size_t)pl.e);
  if (ldcc < H) return QG_INVALID_ARGUMENT;
  const size_t K = ceil_div(k, pl.e);
  const uint64_t kb = gplan->kblock_words;
  if (kb == 0) return QG_INVALID_ARGUMENT;
  const uint64_t kmax = gpu_kmax(gplan);
  if (kb < K && kb * (uint64_t)pl.e > kmax) return QG_PLAN_MISMATCH;  // Eq. 3 per block
  if (kb >= K && k > kmax) return QG_PLAN_MISMATCH;
  if (m == 0 || n == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  if (K == 0) return cuda_status(cudaMemset2DAsync(cc, ldcc * 8, 0, H * 8, m, s));
  int bk = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &bk, &kbs))) return st;
  if (pl.p > 255 || use_small_path(m, n)) {
    DevBuf ws(s);
    QG_TRY(ws.alloc(m * n * sizeof(int32_t)));
    if ((st = qg_mul_common_tiled(gplan, ca_t, cb_t, m, n, k, (int32_t*)ws.p, n, stream))) return st;
    return cuda_status(qgk::launch_pack(qgk::PACK_OUTER_COLS, ws.p, QG_I32, m, n, n, pl.t, pl.e, cc, ldcc, 0, 0, s));
  }
  qgk::GemmArgs a;
  std::memset(&a, 0, sizeof a);
  a.a = ca_t;
  a.b = cb_t;
  if (!dims_ok(m, n, K) || !dims_ok(ldcc, 1)) return QG_INVALID_ARGUMENT;
  a.M = (int)m;
  a.N = (int)n;
  a.K = (int)K;
  a.kb_stages = kbs;
  a.balanced = gplan->balanced != 0;
  a.anchor = a.balanced ? std::ldexp(1.5, pl.t * pl.d + 52) + std::ldexp(1.0, pl.t * pl.d + pl.t - 1)
                        : std::ldexp(1.0, pl.t * pl.d + 52);
  a.qmask = (uint32_t)((1ull << pl.t) - 1);
  a.p = pl.p;
  a.t = pl.t;
  a.e = pl.e;
  a.cc = cc;
  a.ldcc = ldcc;
  if (gplan->anchored && a.balanced && kb < K) {  // K4A with the ReduceAndCompress epilogue
    if ((st = set_anchored_args(pl, K, kb, &a))) return st;
  } else {
    const uint64_t nblocks = (kbs ? ceil_div(K, (size_t)kbs * bk) : 1) + 1;
    if ((unsigned __int128)nblocks * a.qmask + 2 * pl.p >= ((unsigned __int128)1 << 32)) return QG_NOT_EXACT;
  }
  // words cut by a 32-column warp segment are summed atomically from zero
  if (32 % pl.e) QG_TRY(cudaMemset2DAsync(cc, ldcc * 8, 0, H * 8, m, s));
  return cuda_status(qgk::launch_dot_tiled_repack(a, bk, s, &g_last_kernel));
}

// mul_common_repacked(A, B, plan) on device residues in one call: tiled packs
// into stream-ordered workspaces, then qg_mul_common_repacked_tiled.
int qg_mul_common_repacked_compressed(const qg_gpu_plan* gplan, const void* a, size_t lda, const void* b, size_t ldb,
                                      qg_dtype dtype, size_t m, size_t k, size_t n, double* cc, size_t ldcc,
                                      void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < k || ldb < n || ldcc < ceil_div(n, (size_t)pl.e)) return QG_INVALID_ARGUMENT;
  if (pl.t * pl.e > 53 || pl.t > 31) return QG_PLAN_MISMATCH;
  const size_t K = ceil_div(k, (size_t)pl.e);
  if (m == 0 || n == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  if (K == 0) return cuda_status(cudaMemset2DAsync(cc, ldcc * 8, 0, ceil_div(n, (size_t)pl.e) * 8, m, s));
  keep_pool_mapped();
  int bk = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &bk, &kbs))) return st;
  DevBuf ca(s), cb(s);
  QG_TRY(ca.alloc(qg_tiled_words(m, k, pl.e, bk) * 8));
  QG_TRY(cb.alloc(qg_tiled_words(n, k, pl.e, bk) * 8));
  if ((st = qg_pack_a_tiled(gplan, bk, a, dtype, m, k, lda, (double*)ca.p, stream))) return st;
  if ((st = qg_pack_b_tiled(gplan, bk, b, dtype, k, n, ldb, (double*)cb.p, stream))) return st;
  return qg_mul_common_repacked_tiled(gplan, (const double*)ca.p, (const double*)cb.p, m, n, k, cc, ldcc, stream);
}

int qg_mul_common_compressed(const qg_gpu_plan* gplan, const void* a, size_t lda, const void* b, size_t ldb,
                             qg_dtype dtype, size_t m, size_t k, size_t n, int32_t* c, size_t ldc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < k || ldb < n || ldc < n) return QG_INVALID_ARGUMENT;
  const size_t K = ceil_div(k, (size_t)pl.e);
  const uint64_t kb = gplan->kblock_words;
  if (kb == 0) return QG_INVALID_ARGUMENT;
  const uint64_t kmax = gpu_kmax(gplan);
  if (kb < K && kb * (uint64_t)pl.e > kmax) return QG_PLAN_MISMATCH;  // Eq. 3 per block
  if (kb >= K && k > kmax) return QG_PLAN_MISMATCH;
  if (pl.t * pl.e > 53) return QG_PLAN_MISMATCH;  // DoubleWord words only
  if (!dims_ok(m, n, k) || !dims_ok(lda, ldb, ldc)) return QG_INVALID_ARGUMENT;
  if (m == 0 || n == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  if (K == 0) {
    for (size_t i = 0; i < m; ++i)
      if (cudaMemsetAsync(c + i * ldc, 0, n * sizeof(int32_t), s) != cudaSuccess) return QG_CUDA_ERROR;
    return QG_OK;
  }
  if (pl.t > 31) {
    // t * e <= 53 makes e = 1: one residue per word, and Eq. 3 keeps the whole
    // dot product below Q = 2^t < 2^53 — C is the exact integer sum mod p.
    // Integer contraction (64-bit sums, qg_word64.cu) + reduction.
    keep_pool_mapped();
    DevBuf acc(s), cw(s), bw(s);
    QG_TRY(acc.alloc(m * n * 8));
    QG_TRY(bw.alloc(k * n * 8));
    // B's residues as one-residue uint64 words (compress_cols_forward at e = 1)
    if ((st = cuda_status(qgk::launch_pack_u64(qgk::PACK_COLS_FORWARD, b, dtype, k, n, ldb, pl.t, 1,
                                               (uint64_t*)bw.p, n, 0, 0, s))))
      return st;
    int32_t* cdst = c;
    if (ldc != n) {
      QG_TRY(cw.alloc(m * n * 4));
      cdst = (int32_t*)cw.p;
    }
    if ((st = cuda_status(qgk::launch_gemm_u64(1, a, dtype, lda, bw.p, -1, n, m, n, k, 0, 0, (uint64_t*)acc.p, n, s))))
      return st;
    if ((st = cuda_status(qgk::launch_word_reduce_u64((const uint64_t*)acc.p, m * n, 0, 0, (1ull << pl.t) - 1, pl.p,
                                                      cdst, 0, s))))
      return st;
    if (ldc != n)
      return cuda_status(cudaMemcpy2DAsync(c, ldc * 4, cdst, n * 4, n * 4, m, cudaMemcpyDeviceToDevice, s));
    return QG_OK;
  }
  // tiled packs into stream-ordered workspaces, then the tiled contraction
  // (64x64-tile cluster kernel for small products, qg_small.cu)
  keep_pool_mapped();
  int bk = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &bk, &kbs))) return st;
  DevBuf ca(s), cb(s);
  QG_TRY(ca.alloc(qg_tiled_words(m, k, pl.e, bk) * 8));
  QG_TRY(cb.alloc(qg_tiled_words(n, k, pl.e, bk) * 8));
  if ((st = qg_pack_a_tiled(gplan, bk, a, dtype, m, k, lda, (double*)ca.p, stream))) return st;
  if ((st = qg_pack_b_tiled(gplan, bk, b, dtype, k, n, ldb, (double*)cb.p, stream))) return st;
  return qg_mul_common_tiled(gplan, (const double*)ca.p, (const double*)cb.p, m, n, k, c, ldc, stream);
}


uint64_t qg_kernel_launches(void) { return qgk::g_launches.load(); }
void qg_set_dynamic_tiles(int enable) { qgk::set_dynamic_tiles(enable); }
const char* qg_last_error(void) {
  const std::string& m = qg::last_message();
  return m.empty() ? cudaGetErrorString(g_last_cuda_error) : m.c_str();
}
const char* qg_last_kernel(void) { return g_last_kernel; }

int qg_gen_residues(uint64_t seed, uint32_t p, size_t row0, size_t rows, size_t cols, void* dst,
                    qg_dtype dtype, void* stream) {
  if (p < 2 || !qg::is_prime(p)) return QG_INVALID_MODULUS;  // PrimeModulus, field.hpp:19-21
  if (dtype != QG_F64 && dtype != QG_U32) return QG_INVALID_ARGUMENT;
  if (!dst && rows * cols) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_gen_residues(seed, p, row0, rows, cols, dst, dtype, as_stream(stream)));
}

int qg_compress_rows_reversed(const qg_plan* plan, const void* a, qg_dtype dtype, size_t m,
                              size_t k, size_t lda, double* ca, size_t ldca, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // check_common_dim, gemm.hpp:29-35
  const size_t K = ceil_div(k, plan->e);
  if (lda < k || ldca < K) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack(qgk::PACK_ROWS_REVERSED, a, dtype, m, k, lda, plan->t,
                                      plan->e, ca, ldca, 0, 0, as_stream(stream)));
}

int qg_compress_cols_forward(const qg_plan* plan, const void* b, qg_dtype dtype, size_t k,
                             size_t n, size_t ldb, double* cb, size_t ldcb, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;
  if (ldb < n || ldcb < n) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack(qgk::PACK_COLS_FORWARD, b, dtype, k, n, ldb, plan->t,
                                      plan->e, cb, ldcb, 0, 0, as_stream(stream)));
}

int qg_compress_outer_cols(const qg_plan* plan, const void* b, qg_dtype dtype, size_t rows,
                           size_t cols, size_t ldb, double* cb, size_t ldcb, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (ldb < cols || ldcb < ceil_div(cols, plan->e)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack(qgk::PACK_OUTER_COLS, b, dtype, rows, cols, ldb, plan->t,
                                      plan->e, cb, ldcb, 0, 0, as_stream(stream)));
}

int qg_compress_outer_rows(const qg_plan* plan, const void* a, qg_dtype dtype, size_t rows,
                           size_t cols, size_t lda, double* ca, size_t ldca, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (lda < cols || ldca < cols) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_pack(qgk::PACK_OUTER_ROWS, a, dtype, rows, cols, lda, plan->t,
                                      plan->e, ca, ldca, 0, 0, as_stream(stream)));
}

int qg_packed_common_product(const qg_plan* plan, const double* ca, const double* cb, size_t m,
                             size_t n, size_t k, double* acc, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:225
  qgk::HighArgs h;
  h.ca = ca;
  h.ldca = ceil_div(k, plan->e);
  h.cb = cb;
  h.ldcb = n;
  if (!dims_ok(m, n, k)) return QG_INVALID_ARGUMENT;
  h.M = (int)m;
  h.N = (int)n;
  h.K = (int)ceil_div(k, plan->e);
  h.inv_qd = plan->inv_qd;
  h.kb_words = 0;
  h.qmask = (uint32_t)((1ull << plan->t) - 1);
  h.p = plan->p;
  h.acc = acc;
  h.c = nullptr;
  h.ldc = n;
  if (m == 0 || n == 0) return QG_OK;
  if (h.K == 0) return cuda_status(cudaMemsetAsync(acc, 0, m * n * sizeof(double), as_stream(stream)));
  return cuda_status(qgk::launch_dot_highpart(h, as_stream(stream), &g_last_kernel));
}

int qg_reduce_common(const qg_plan* plan, const double* acc, size_t count, int32_t* c, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  return cuda_status(qgk::launch_reduce_common(acc, count, (uint32_t)((1ull << plan->t) - 1),
                                               plan->p, c, as_stream(stream)));
}

int qg_mul_common(const qg_gpu_plan* gplan, const double* ca, const double* cb, size_t m, size_t n,
                  size_t k, int32_t* c, size_t ldc, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  if (gplan->balanced) return QG_PLAN_MISMATCH;  // reference-layout words are unsigned
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if (ldc < n) return QG_INVALID_ARGUMENT;
  const size_t K = ceil_div(k, pl.e);
  uint64_t kb = gplan->kblock_words;
  if (kb == 0) return QG_INVALID_ARGUMENT;
  // Eq. 3 per block (gemm.hpp:456): a block may hold at most kmax residues.
  const uint64_t kmax = gpu_kmax(gplan);
  if (kb < K && kb * (uint64_t)pl.e > kmax) return QG_PLAN_MISMATCH;
  if (kb >= K && k > kmax) return QG_PLAN_MISMATCH;
  if (K == 0) {
    cudaStream_t s = as_stream(stream);
    for (size_t i = 0; i < m; ++i)
      if (cudaMemsetAsync(c + i * ldc, 0, n * sizeof(int32_t), s) != cudaSuccess) return QG_CUDA_ERROR;
    return QG_OK;
  }
  return run_common(pl, kb, ca, K, cb, n, m, n, K, c, ldc, as_stream(stream));
}

int qg_mul_common_repacked(const qg_gpu_plan* gplan, const double* ca, const double* cb, size_t m,
                           size_t n, size_t k, double* cc, int32_t* workspace, void* stream) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  int32_t* ws = workspace;
  if (!ws && m * n) {
    if (cudaMallocAsync(&ws, m * n * sizeof(int32_t), s) != cudaSuccess) return QG_CUDA_ERROR;
  }
  int st = qg_mul_common(gplan, ca, cb, m, n, k, ws, n, stream);
  if (!st)  // compress_outer_cols(C, plan), gemm.hpp:279
    st = cuda_status(qgk::launch_pack(qgk::PACK_OUTER_COLS, ws, QG_I32, m, n, n, gplan->plan.t,
                                      gplan->plan.e, cc, ceil_div(n, gplan->plan.e), 0, 0, s));
  if (!workspace && ws) cudaFreeAsync(ws, s);
  return st;
}

static int right_common(const qg_plan* plan, const double* a, size_t lda, const double* cbo,
                        size_t m, size_t k, size_t n, double* cc, int redq, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:295
  if (plan->t * plan->e > 53) return QG_PLAN_MISMATCH;  // sums must stay exact
  if (lda < k) return QG_INVALID_ARGUMENT;
  const size_t H = ceil_div(n, plan->e);
  if (m == 0 || H == 0) return QG_OK;
  if (k == 0) return cuda_status(cudaMemsetAsync(cc, 0, m * H * sizeof(double), as_stream(stream)));
  qgk::GemmArgs r;
  std::memset(&r, 0, sizeof r);
  r.a = a;
  r.lda = lda;
  r.b = cbo;
  r.ldb = H;
  if (!dims_ok(m, H, k)) return QG_INVALID_ARGUMENT;
  r.M = (int)m;
  r.N = (int)H;
  r.K = (int)k;
  r.t = plan->t;
  r.e = plan->e;
  r.p = plan->p;
  r.cc = cc;
  r.ldcc = H;
  return cuda_status(qgk::launch_right_dmma(r, redq != 0, as_stream(stream), &g_last_kernel));
}

int qg_mul_right(const qg_plan* plan, const double* a, size_t lda, const double* cbo, size_t m,
                 size_t k, size_t n, double* cc, void* stream) {
  return right_common(plan, a, lda, cbo, m, k, n, cc, 1, stream);
}

int qg_packed_right_product(const qg_plan* plan, const double* a, size_t lda, const double* cbo,
                            size_t m, size_t k, size_t n, double* cc, void* stream) {
  return right_common(plan, a, lda, cbo, m, k, n, cc, 0, stream);
}

// packed_left_product / mul_left_compressed (DoubleWord, reference layout),
// gemm.hpp:340-371: CC (ceil(m/e) x n words) = CA (compress_outer_rows words,
// ceil(m/e) x k, ldca) x B (k x n residues). Both this and the right product
// are row-major word matrix x row-major word matrix with exact sums < Q^e, so
// the right variant's DMMA contraction runs it with the operands' roles
// swapped; residues that are not float64 are widened on the device first
// (an e = 1 forward pack is the identity on values).
static int left_common(const qg_plan* plan, const double* ca, size_t ldca, const void* b, qg_dtype dtype,
                       size_t ldb, size_t m, size_t k, size_t n, double* cc, int redq, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;          // gemm.hpp:349 check_common_dim
  if (plan->t * plan->e > 53) return QG_PLAN_MISMATCH;  // sums must stay exact
  if (ldca < k || ldb < n) return QG_INVALID_ARGUMENT;
  const size_t G = ceil_div(m, (size_t)plan->e);
  if (G == 0 || n == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  if (k == 0) return cuda_status(cudaMemsetAsync(cc, 0, G * n * sizeof(double), s));
  DevBuf wide(s);
  const double* bd = static_cast<const double*>(b);
  size_t ldbd = ldb;
  if (dtype != QG_F64) {
    QG_TRY(wide.alloc(k * n * sizeof(double)));
    QG_TRY(qgk::launch_pack(qgk::PACK_OUTER_COLS, b, dtype, k, n, ldb, 1, 1, (double*)wide.p, n, 0, 0, s));
    bd = (const double*)wide.p;
    ldbd = n;
  }
  qgk::GemmArgs r;
  std::memset(&r, 0, sizeof r);
  r.a = ca;
  r.lda = ldca;
  r.b = bd;
  r.ldb = ldbd;
  if (!dims_ok(G, n, k)) return QG_INVALID_ARGUMENT;
  r.M = (int)G;
  r.N = (int)n;
  r.K = (int)k;
  r.t = plan->t;
  r.e = plan->e;
  r.p = plan->p;
  r.cc = cc;
  r.ldcc = n;
  return cuda_status(qgk::launch_right_dmma(r, redq != 0, s, &g_last_kernel));
}

int qg_packed_left_product(const qg_plan* plan, const double* ca, size_t ldca, const void* b, qg_dtype dtype,
                           size_t ldb, size_t m, size_t k, size_t n, double* cc, void* stream) {
  return left_common(plan, ca, ldca, b, dtype, ldb, m, k, n, cc, 0, stream);
}

int qg_mul_left(const qg_plan* plan, const double* ca, size_t ldca, const void* b, qg_dtype dtype, size_t ldb,
                size_t m, size_t k, size_t n, double* cc, void* stream) {
  return left_common(plan, ca, ldca, b, dtype, ldb, m, k, n, cc, 1, stream);
}

static int extract_digits(const qg_plan* plan, const void* words, bool u64, size_t count, uint64_t* digits,
                          void* stream) {
  if (!plan) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !qg::is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->t < 1 || plan->e < 1 || plan->t * plan->e > (u64 ? 64 : 53)) return QG_PLAN_MISMATCH;
  if (count == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  DeviceFlag flag(s);
  if (!flag.ptr) return QG_CUDA_ERROR;
  int st = cuda_status(qgk::launch_extract_digits(words, u64, count, plan->t, plan->e, digits, flag.ptr, s));
  if (st) return st;
  int over = 0;
  if ((st = flag.read(&over))) return st;
  return over ? QG_DIGIT_OVERFLOW : QG_OK;
}

int qg_extract_digits(const qg_plan* plan, const double* words, size_t count, uint64_t* digits, void* stream) {
  return extract_digits(plan, words, false, count, digits, stream);
}

int qg_extract_digits_u64(const qg_plan* plan, const uint64_t* words, size_t count, uint64_t* digits,
                          void* stream) {
  return extract_digits(plan, words, true, count, digits, stream);
}

// Device memory for callers without the CUDA runtime headers (the C++
// drop-in): synchronous, on the legacy default stream that the entry points
// run on when passed a NULL stream.
int qg_device_alloc(size_t bytes, void** ptr) {
  if (!ptr) return QG_INVALID_ARGUMENT;
  *ptr = nullptr;
  if (bytes == 0) return QG_OK;
  return cuda_status(cudaMalloc(ptr, bytes));
}
int qg_device_free(void* ptr) { return ptr ? cuda_status(cudaFree(ptr)) : QG_OK; }
int qg_copy_to_device(void* dst, const void* src, size_t bytes) {
  return bytes ? cuda_status(cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice)) : QG_OK;
}
int qg_copy_to_host(void* dst, const void* src, size_t bytes) {
  return bytes ? cuda_status(cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost)) : QG_OK;
}

int qg_redq(const qg_plan* plan, double* words, size_t count, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (count == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  DeviceFlag flag(s);
  if (!flag.ptr) return QG_CUDA_ERROR;
  if ((st = cuda_status(qgk::launch_redq(words, count, plan->t, plan->e, plan->p, flag.ptr, s)))) return st;
  int over = 0;
  if ((st = flag.read(&over))) return st;
  return over ? QG_DIGIT_OVERFLOW : QG_OK;
}

int qg_uncompress(const qg_plan* plan, qg_orientation o, const double* words, size_t stored_rows,
                  size_t stored_cols, size_t logical_rows, size_t logical_cols, int32_t* out,
                  void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (o.slots < 1 || o.slots > plan->e) return QG_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  DeviceFlag flag(s);
  if (!flag.ptr) return QG_CUDA_ERROR;
  if ((st = cuda_status(qgk::launch_uncompress(words, stored_rows, stored_cols, logical_rows,
                                               logical_cols, plan->t, plan->e, o.slots,
                                               o.direction == 1, o.axis == 1, plan->p, out,
                                               flag.ptr, s))))
    return st;
  int over = 0;
  if ((st = flag.read(&over))) return st;
  return over ? QG_DIGIT_OVERFLOW : QG_OK;
}

// ------------------------------------------------------------ host buffers

namespace {

// Phase split of the last host-data call, the reference's PhaseSeconds
// (gemm.hpp, bench.hpp:67-152): multiply = device time of the contraction
// kernels (event pairs on the stream they run on), convert = the rest of the
// call's wall time (transfers, packing, extraction, reduction).
struct PhaseLog {
  double multiply = 0, convert = 0;
};
thread_local PhaseLog g_phase;
// Recording timing events between the pipelined path's kernels costs ~0.36 ms
// of a config-2 host call (measured), so the split is measured only on request.
std::atomic<int> g_phase_timing{0};

struct PhaseScope {
  static constexpr int kPairs = 512;  // host_pipeline2d: up to 64 chunks x 8 panels
  // timing events created once per thread: creating them per call stalls the
  // host's enqueue loop of the pipelined path (measured +0.36 ms on config 2)
  static cudaEvent_t* pool() {
    if (!g_phase_timing.load(std::memory_order_relaxed)) return nullptr;
    // events belong to a device: one pool per (thread, device)
    static thread_local std::map<int, std::vector<cudaEvent_t>> pools;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
    std::vector<cudaEvent_t>& ev = pools[dev];
    if (ev.empty()) {
      ev.assign(2 * kPairs, nullptr);
      for (auto& e : ev)
        if (cudaEventCreate(&e) != cudaSuccess) e = nullptr;
    }
    return ev.data();
  }
  std::chrono::steady_clock::time_point t0 = std::chrono::steady_clock::now();
  cudaEvent_t* ev = pool();
  int n = 0;
  const bool on = g_phase_timing.load(std::memory_order_relaxed) != 0;
  void begin(cudaStream_t s) {
    if (!on || n + 2 > 2 * kPairs || !ev[n] || !ev[n + 1]) return;
    cudaEventRecord(ev[n], s);
  }
  void end(cudaStream_t s) {
    if (!on || n + 2 > 2 * kPairs || !ev[n] || !ev[n + 1]) return;
    cudaEventRecord(ev[n + 1], s);
    n += 2;
  }
  void finish() {  // after the call's final synchronize
    double mul = 0;
    if (!on) n = 0;
    for (int i = 0; i < n; i += 2) {
      float ms = 0;
      if (cudaEventElapsedTime(&ms, ev[i], ev[i + 1]) == cudaSuccess) mul += ms * 1e-3;
    }
    const double wall = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    g_phase.multiply = mul;
    g_phase.convert = wall > mul ? wall - mul : 0.0;
  }
};

}  // namespace

// Streams and events of the pipelined host path, created once per thread.
struct HostPipe {
  cudaStream_t in = nullptr, comp = nullptr, out = nullptr;
  // chunk contractions rotate over kComp compute streams: a chunk with fewer
  // output tiles than SMs then shares the GPU with the next one
  static constexpr int kComp = 3;
  cudaStream_t comps[kComp] = {};
  static constexpr int kMaxChunks = 64;
  cudaEvent_t b_ready = nullptr, b_packed = nullptr, a_ready[kMaxChunks] = {}, c_ready[kMaxChunks] = {},
              done = nullptr;
  std::vector<cudaEvent_t> pool;  // host_pipeline2d's per-item and per-tile events, grown on demand
  cudaEvent_t event(size_t i) {
    while (pool.size() <= i) {
      cudaEvent_t e = nullptr;
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return nullptr;
      pool.push_back(e);
    }
    return pool[i];
  }
  cudaEvent_t join[kComp + 1] = {};  // PipeJoin: one per compute stream + out
  qg::HostStager stage;               // pinned slots for pageable host buffers (allocated on first use)
  bool ok = false;
  HostPipe() {
    ok = cudaStreamCreateWithFlags(&in, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&comp, cudaStreamNonBlocking) == cudaSuccess &&
         cudaStreamCreateWithFlags(&out, cudaStreamNonBlocking) == cudaSuccess &&
         cudaEventCreateWithFlags(&b_ready, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&b_packed, cudaEventDisableTiming) == cudaSuccess &&
         cudaEventCreateWithFlags(&done, cudaEventDisableTiming) == cudaSuccess;
    comps[0] = comp;
    for (int i = 1; ok && i < kComp; ++i) ok = cudaStreamCreateWithFlags(&comps[i], cudaStreamNonBlocking) == cudaSuccess;
    for (int i = 0; ok && i <= kComp; ++i)
      ok = cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming) == cudaSuccess;
    for (int i = 0; ok && i < kMaxChunks; ++i)
      ok = cudaEventCreateWithFlags(&a_ready[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaEventCreateWithFlags(&c_ready[i], cudaEventDisableTiming) == cudaSuccess;
    // keep freed stream-ordered allocations mapped across calls (the default
    // release threshold of 0 would unmap and re-map the buffers every call)
    int dev = 0;
    cudaMemPool_t pool;
    if (ok && cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
};

// Pipelined host products (common, right, left, full): B goes up first and is
// packed; A streams up in row chunks (a multiple of `align` rows, so every
// chunk maps to whole 128-row blocks of the packed layout) while the earlier
// chunks are packed and contracted; each chunk's output streams back on its
// own stream, so both PCIe directions overlap the contraction.
// One pipeline (streams, events) per host thread AND device: its streams and
// events belong to the device that was current when it was made, so a thread
// that moves to another GPU gets that GPU's own set.
static HostPipe& host_pipe() {
  static thread_local std::map<int, std::unique_ptr<HostPipe>> pipes;
  int dev = 0;
  cudaGetDevice(&dev);
  std::unique_ptr<HostPipe>& hp = pipes[dev];
  if (!hp) hp.reset(new HostPipe());
  return *hp;
}

// Joins every stream of the pipeline into hp.in when a pipelined call
// returns, on success and on every early error return alike: the call's
// buffers are freed stream-ordered on hp.in (DevBuf), so the frees then wait
// for every pack, contraction and copy already queued on the compute streams
// and on hp.out. Declare it after the call's DevBufs (destroyed before them).
struct PipeJoin {
  HostPipe& hp;
  explicit PipeJoin(HostPipe& h) : hp(h) {}
  PipeJoin(const PipeJoin&) = delete;
  PipeJoin& operator=(const PipeJoin&) = delete;
  ~PipeJoin() {
    for (int i = 0; i <= HostPipe::kComp; ++i) {
      cudaStream_t st = i < HostPipe::kComp ? hp.comps[i] : hp.out;
      if (hp.join[i] && st && cudaEventRecord(hp.join[i], st) == cudaSuccess) cudaStreamWaitEvent(hp.in, hp.join[i], 0);
    }
    hp.stage.finish();  // no staged copy into the caller's buffers outlives the call
  }
};

struct ChunkOut {
  const void* src = nullptr;
  void* dst = nullptr;
  size_t bytes = 0;
};

static int host_pipeline(size_t m, size_t k, size_t n, size_t align, size_t col_tiles, const uint32_t* a,
                         const uint32_t* b,
                         const std::function<int(const uint32_t* db, cudaStream_t s)>& pack_b,
                         const std::function<int(size_t r0, size_t rows, const uint32_t* da, cudaStream_t s,
                                                 PhaseScope& ps, ChunkOut* out)>& chunk) {
  HostPipe& hp = host_pipe();
  if (!hp.ok) return QG_CUDA_ERROR;
  PhaseScope ps;
  size_t rows_per = (512 + align - 1) / align * align;
  size_t nchunks = ceil_div(m, rows_per);
  if (nchunks > (size_t)HostPipe::kMaxChunks) {
    rows_per = ceil_div(ceil_div(m, (size_t)HostPipe::kMaxChunks), align) * align;
    nchunks = ceil_div(m, rows_per);
  }
  // a chunk that already fills most SMs runs alone (overlapping kernels only
  // contend: config 2); smaller ones rotate over up to kComp streams (config 4)
  int sms = 148;
  {
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  }
  const size_t chunk_tiles = (rows_per / align) * (col_tiles ? col_tiles : 1);
  int ncomp = chunk_tiles * 4 >= (size_t)sms * 3 ? 1 : (int)ceil_div((size_t)sms, chunk_tiles ? chunk_tiles : 1);
  if (ncomp > HostPipe::kComp) ncomp = HostPipe::kComp;
  DevBuf da(hp.in), db(hp.in);
  PipeJoin join(hp);  // after the buffers: joins the streams before they are freed
  QG_TRY(da.alloc(m * k * 4));
  if (b) {  // b == NULL: the right operand is already packed on the device (pack_b only orders on it)
    QG_TRY(db.alloc(k * n * 4));
    if (k * n) QG_TRY(hp.stage.h2d(db.p, 0, b, 0, k * n * 4, 1, hp.in));
  }
  QG_TRY(cudaEventRecord(hp.b_ready, hp.in));
  QG_TRY(cudaStreamWaitEvent(hp.comp, hp.b_ready, 0));
  int st = pack_b((const uint32_t*)db.p, hp.comp);
  if (st) return st;
  QG_TRY(cudaEventRecord(hp.b_packed, hp.comp));
  for (int j = 1; j < ncomp; ++j) QG_TRY(cudaStreamWaitEvent(hp.comps[j], hp.b_packed, 0));
  // chunk i goes up, then its contraction and its copy back are queued: from
  // pinned buffers every copy is async anyway; from pageable ones (staged,
  // the host copies into pinned slots) chunk i+1 is staged while chunk i runs
  for (size_t i = 0; i < nchunks; ++i) {
    const size_t r0 = i * rows_per, rows = (m - r0) < rows_per ? (m - r0) : rows_per;
    if (rows * k) QG_TRY(hp.stage.h2d((uint32_t*)da.p + r0 * k, 0, a + r0 * k, 0, rows * k * 4, 1, hp.in));
    QG_TRY(cudaEventRecord(hp.a_ready[i], hp.in));
    cudaStream_t cs = hp.comps[i % ncomp];
    QG_TRY(cudaStreamWaitEvent(cs, hp.a_ready[i], 0));
    ChunkOut out;
    if ((st = chunk(r0, rows, (const uint32_t*)da.p + r0 * k, cs, ps, &out))) return st;
    QG_TRY(cudaEventRecord(hp.c_ready[i], cs));
    QG_TRY(cudaStreamWaitEvent(hp.out, hp.c_ready[i], 0));
    if (out.bytes) QG_TRY(hp.stage.d2h(out.dst, 0, out.src, 0, out.bytes, 1, hp.out));
  }
  QG_TRY(cudaEventRecord(hp.done, hp.out));
  QG_TRY(cudaStreamWaitEvent(hp.in, hp.done, 0));  // buffers are freed on `in` after everything
  QG_TRY(cudaStreamSynchronize(hp.out));
  QG_TRY(hp.stage.finish());
  ps.finish();
  return QG_OK;
}

// The 2-D pipeline pays off when the contraction is long against B's
// transfer (config 5: B is 78 ms of PCIe against a 0.36 s product, 448 ->
// 403 ms); where the transfer dominates anyway (config 2) or the tiles get
// too small for the GPU (config 4, 3.5 % at best) the 1-D pipeline stays.
// Estimates: contraction at 30 TFLOP/s of packed FP64, PCIe at 50 GB/s.
// QG_HOST_2D=0/1 forces it off/on.
static bool use_pipeline2d(double packed_flop, size_t b_bytes) {
  const char* e = getenv("QG_HOST_2D");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return packed_flop / 30e12 > 3.0 * ((double)b_bytes / 50e9);
}

// Two-dimensional variant of host_pipeline: A streams up in row chunks and B
// in column panels, the two interleaved by bytes sent, so the contraction of
// tile (chunk r, panel c) starts as soon as both have arrived and been packed
// instead of after all of B (config 4: B alone is 4.7 ms of PCIe). Tiles
// rotate over the compute streams; each tile's output leaves as a 2-D copy.
struct TileOut {
  const void* src = nullptr;
  size_t spitch = 0;
  void* dst = nullptr;
  size_t dpitch = 0, width = 0, height = 0;
};

static int host_pipeline2d(
    size_t m, size_t k, size_t n, size_t align, size_t col_align, size_t out_tiles_per_block, const uint32_t* a,
    const uint32_t* b,
    const std::function<int(size_t c0, size_t cols, const uint32_t* dbp, cudaStream_t s)>& pack_b_panel,
    const std::function<int(size_t r0, size_t rows, const uint32_t* da, cudaStream_t s)>& pack_a_chunk,
    const std::function<int(size_t r0, size_t rows, size_t c0, size_t cols, cudaStream_t s, PhaseScope& ps,
                            TileOut* out)>& tile) {
  HostPipe& hp = host_pipe();
  if (!hp.ok) return QG_CUDA_ERROR;
  PhaseScope ps;
  // column panels (whole multiples of col_align columns; one col_align block =
  // out_tiles_per_block 128-wide output tile columns)
  const size_t col_blocks = ceil_div(n, col_align);
  // up to 16 panels of >= 16 tile columns (config 5: 4 / 8 / 16 / 32 panels at
  // two waves of tiles per launch: 403 / 390 / 389 / 389 ms e2e, tools/e2e_c5_sweep.py)
  size_t want_p = col_blocks * out_tiles_per_block / 16;
  // (pageable B: at most 8 — its panels are staged row by row on the host)
  const size_t max_p = qg::host_pinned(b) ? 16 : 8;
  want_p = want_p < 2 ? 2 : (want_p > max_p ? max_p : want_p);
  if (const char* e = getenv("QG_HOST_PANELS")) want_p = (size_t)atoi(e);  // experiments
  const size_t npanels = col_blocks < want_p ? (col_blocks ? col_blocks : 1) : (want_p ? want_p : 1);
  const size_t blocks_per = ceil_div(col_blocks, npanels);
  // row chunks large enough that one tile launch has ~two waves of 128 x 128
  // output tiles (a tile launch on a few SMs would leave the GPU idle; config 5:
  // 96 / 148 / 296 / 444 tiles per launch at 16 panels: 395 / 389 / 389 / 391 ms)
  size_t want_tiles = 2 * (size_t)device_sms();
  if (const char* e = getenv("QG_HOST_TILES")) want_tiles = (size_t)atoi(e);  // experiments
  const size_t tc = blocks_per * out_tiles_per_block;
  size_t rows_per = ceil_div(want_tiles, tc ? tc : 1) * 128;
  if (rows_per < 512) rows_per = 512;
  rows_per = (rows_per + align - 1) / align * align;
  size_t nchunks = ceil_div(m, rows_per);
  if (nchunks > (size_t)HostPipe::kMaxChunks) {
    rows_per = ceil_div(ceil_div(m, (size_t)HostPipe::kMaxChunks), align) * align;
    nchunks = ceil_div(m, rows_per);
  }
  auto panel = [&](size_t j, size_t* c0, size_t* cols) {
    *c0 = j * blocks_per * col_align;
    const size_t c1 = (j + 1) * blocks_per * col_align;
    *cols = (c1 < n ? c1 : n) - (*c0 < n ? *c0 : n);
  };
  DevBuf da(hp.in), db(hp.in);
  PipeJoin join(hp);  // after the buffers: joins the streams before they are freed
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));  // panel j: k x cols_j contiguous at column offset c0_j * k
  size_t ev = 0;
  std::vector<cudaEvent_t> a_packed(nchunks, nullptr), b_packed(npanels, nullptr);
  std::vector<char> a_sent(nchunks, 0), b_sent(npanels, 0);
  size_t ia = 0, ib = 0, bytes_a = 0, bytes_b = 0, ntile = 0, npack = 0;
  while (ia < nchunks || ib < npanels) {
    // the stream (A rows or B columns) that has sent fewer bytes goes next
    const bool send_b = ib < npanels && (ia >= nchunks || bytes_b <= bytes_a);
    cudaEvent_t ready = hp.event(ev++), packed = hp.event(ev++);
    if (!ready || !packed) return QG_CUDA_ERROR;
    cudaStream_t ps_s = hp.comps[npack++ % HostPipe::kComp];
    if (send_b) {
      size_t c0, cols;
      panel(ib, &c0, &cols);
      const uint32_t* dbp = (const uint32_t*)db.p + c0 * k;
      if (k * cols)
        QG_TRY(hp.stage.h2d((void*)dbp, cols * 4, b + c0, n * 4, cols * 4, k, hp.in));
      QG_TRY(cudaEventRecord(ready, hp.in));
      QG_TRY(cudaStreamWaitEvent(ps_s, ready, 0));
      int st = pack_b_panel(c0, cols, dbp, ps_s);
      if (st) return st;
      QG_TRY(cudaEventRecord(packed, ps_s));
      b_packed[ib] = packed;
      b_sent[ib] = 1;
      bytes_b += k * cols * 4;
    } else {
      const size_t r0 = ia * rows_per, rows = (m - r0) < rows_per ? (m - r0) : rows_per;
      const uint32_t* dap = (const uint32_t*)da.p + r0 * k;
      if (rows * k) QG_TRY(hp.stage.h2d((void*)dap, 0, a + r0 * k, 0, rows * k * 4, 1, hp.in));
      QG_TRY(cudaEventRecord(ready, hp.in));
      QG_TRY(cudaStreamWaitEvent(ps_s, ready, 0));
      int st = pack_a_chunk(r0, rows, dap, ps_s);
      if (st) return st;
      QG_TRY(cudaEventRecord(packed, ps_s));
      a_packed[ia] = packed;
      a_sent[ia] = 1;
      bytes_a += rows * k * 4;
    }
    // every tile the new item completes
    const size_t r_lo = send_b ? 0 : ia, r_hi = send_b ? ia : ia + 1;
    const size_t c_lo = send_b ? ib : 0, c_hi = send_b ? ib + 1 : ib;
    for (size_t r = r_lo; r < r_hi; ++r)
      for (size_t c = c_lo; c < c_hi; ++c) {
        if (!a_sent[r] || !b_sent[c]) continue;
        const size_t r0 = r * rows_per, rows = (m - r0) < rows_per ? (m - r0) : rows_per;
        size_t c0, cols;
        panel(c, &c0, &cols);
        cudaStream_t cs = hp.comps[ntile++ % HostPipe::kComp];
        QG_TRY(cudaStreamWaitEvent(cs, a_packed[r], 0));
        QG_TRY(cudaStreamWaitEvent(cs, b_packed[c], 0));
        TileOut out;
        int st = tile(r0, rows, c0, cols, cs, ps, &out);
        if (st) return st;
        cudaEvent_t done_t = hp.event(ev++);
        if (!done_t) return QG_CUDA_ERROR;
        QG_TRY(cudaEventRecord(done_t, cs));
        QG_TRY(cudaStreamWaitEvent(hp.out, done_t, 0));
        if (out.width && out.height)
          QG_TRY(hp.stage.d2h(out.dst, out.dpitch, out.src, out.spitch, out.width, out.height, hp.out));
      }
    if (send_b) ++ib;
    else ++ia;
  }
  QG_TRY(cudaEventRecord(hp.done, hp.out));
  QG_TRY(cudaStreamWaitEvent(hp.in, hp.done, 0));  // buffers are freed on `in` after everything
  QG_TRY(cudaStreamSynchronize(hp.out));
  QG_TRY(hp.stage.finish());
  ps.finish();
  return QG_OK;
}

// mul_common_compressed on host data, pipelined over three streams: B goes
// up first and is packed; A then streams up in row chunks of 512 while the
// previous chunks are packed and contracted, and C streams back per chunk on
// its own stream (the two PCIe directions overlap). Exact same kernels and
// results as the device path.
static int host_common(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m,
                       size_t k, size_t n, uint32_t* c) {
  const qg_plan& pl = gp->plan;
  int st;
  const size_t K = ceil_div(k, pl.e);
  int bk = 0, kbs = 0;
  const bool tiled = (n % 2 == 0) && K > 0 && tiled_geometry(gp, K, &bk, &kbs) == QG_OK;
  if (tiled && m * n > 0) {
    const size_t Kt = ceil_div(K, (size_t)bk);
    cudaStream_t s0 = host_pipe().in;
    DevBuf dca(s0), dcb(s0), dc(s0);
    QG_TRY(dc.alloc(m * n * 4));
    QG_TRY(dca.alloc(qg_tiled_words(m, k, pl.e, bk) * 8));
    QG_TRY(dcb.alloc(qg_tiled_words(n, k, pl.e, bk) * 8));
    const size_t Wt = Kt * 128 * bk;  // words per 128-row (column) block of CA_t (CB_t)
    if (use_pipeline2d(2.0 * m * n * K, k * n * 4))
      return host_pipeline2d(
          m, k, n, 128, 128, 1, a, b,
          [&](size_t c0, size_t cols, const uint32_t* dbp, cudaStream_t s2) {
            return cuda_status(qgk::launch_pack_tiled(true, dbp, QG_U32, k, cols, cols, pl.t, pl.e, bk,
                                                      (double*)dcb.p + (c0 / 128) * Wt, s2, pl.p, gp->balanced != 0));
          },
          [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s2) {
            return cuda_status(qgk::launch_pack_tiled(false, da, QG_U32, rows, k, k, pl.t, pl.e, bk,
                                                      (double*)dca.p + (r0 / 128) * Wt, s2, pl.p, gp->balanced != 0));
          },
          [&](size_t r0, size_t rows, size_t c0, size_t cols, cudaStream_t s2, PhaseScope& ps, TileOut* out) {
            ps.begin(s2);
            int st2 = qg_mul_common_tiled(gp, (const double*)dca.p + (r0 / 128) * Wt,
                                          (const double*)dcb.p + (c0 / 128) * Wt, rows, cols, k,
                                          (int32_t*)dc.p + r0 * n + c0, n, s2);
            if (st2) return st2;
            ps.end(s2);
            out->src = (const int32_t*)dc.p + r0 * n + c0;
            out->dst = c + r0 * n + c0;
            out->spitch = out->dpitch = n * 4;
            out->width = cols * 4;
            out->height = rows;
            return (int)QG_OK;
          });
    return host_pipeline(
        m, k, n, 128, ceil_div(n, (size_t)128), a, b,
        [&](const uint32_t* db, cudaStream_t s2) {
          return cuda_status(qgk::launch_pack_tiled(true, db, QG_U32, k, n, n, pl.t, pl.e, bk, (double*)dcb.p, s2,
                                                    pl.p, gp->balanced != 0));
        },
        [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s2, PhaseScope& ps, ChunkOut* out) {
          double* ca_chunk = (double*)dca.p + (r0 / 128) * Kt * 128 * bk;
          int st2 = cuda_status(qgk::launch_pack_tiled(false, da, QG_U32, rows, k, k, pl.t, pl.e, bk, ca_chunk, s2,
                                                       pl.p, gp->balanced != 0));
          if (st2) return st2;
          ps.begin(s2);
          if ((st2 = qg_mul_common_tiled(gp, ca_chunk, (const double*)dcb.p, rows, n, k, (int32_t*)dc.p + r0 * n, n,
                                         s2)))
            return st2;
          ps.end(s2);
          out->src = (const int32_t*)dc.p + r0 * n;
          out->dst = c + r0 * n;
          out->bytes = rows * n * 4;
          return (int)QG_OK;
        });
  }
  if (gp->balanced) {  // the row-layout kernels need unsigned words: re-plan
    qg_gpu_plan up;
    if ((st = qg_plan_gpu_ex(pl.p, k, 1, &up))) return st;
    return host_common(&up, a, b, m, k, n, c);
  }
  cudaStream_t s = nullptr;
  PhaseScope ps;
  DevBuf da(s), db(s), dca(s), dcb(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  // reference layout: packing itself does not depend on kmax; the blocks enforce Eq. 3
  QG_TRY(dca.alloc(m * K * 8));
  QG_TRY(dcb.alloc(K * n * 8));
  QG_TRY(qgk::launch_pack(qgk::PACK_ROWS_REVERSED, da.p, QG_U32, m, k, k, pl.t, pl.e, (double*)dca.p, K, 0, 0, s));
  QG_TRY(qgk::launch_pack(qgk::PACK_COLS_FORWARD, db.p, QG_U32, k, n, n, pl.t, pl.e, (double*)dcb.p, n, 0, 0, s));
  ps.begin(s);
  if ((st = qg_mul_common(gp, (const double*)dca.p, (const double*)dcb.p, m, n, k, (int32_t*)dc.p, n, s)))
    return st;
  ps.end(s);
  if (m * n) QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

// mul_common_repacked on host data (gemm.hpp:275-280): the 1-D host
// pipeline of host_common with the repacking contraction per row chunk, each
// chunk's CC words streamed back while later chunks run. Plans the tiled
// kernels cannot run exactly take the reference-layout path (two passes).
static int host_common_repacked(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                size_t n, double* cc) {
  const qg_plan& pl = gp->plan;
  const size_t K = ceil_div(k, pl.e), H = ceil_div(n, (size_t)pl.e);
  if (m * H == 0) return QG_OK;
  int bk = 0, kbs = 0;
  const int geo = K > 0 ? tiled_geometry(gp, K, &bk, &kbs) : QG_OK;
  if (geo != QG_OK && gp->balanced) return geo;
  if (geo != QG_OK) {
    cudaStream_t s = nullptr;
    DevBuf da(s), db(s), dca(s), dcb(s), dcc(s);
    QG_TRY(da.alloc(m * k * 4));
    QG_TRY(db.alloc(k * n * 4));
    QG_TRY(dca.alloc(m * K * 8));
    QG_TRY(dcb.alloc(K * n * 8));
    QG_TRY(dcc.alloc(m * H * 8));
    QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
    QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
    QG_TRY(qgk::launch_pack(qgk::PACK_ROWS_REVERSED, da.p, QG_U32, m, k, k, pl.t, pl.e, (double*)dca.p, K, 0, 0, s));
    QG_TRY(qgk::launch_pack(qgk::PACK_COLS_FORWARD, db.p, QG_U32, k, n, n, pl.t, pl.e, (double*)dcb.p, n, 0, 0, s));
    int st = qg_mul_common_repacked(gp, (const double*)dca.p, (const double*)dcb.p, m, n, k, (double*)dcc.p, nullptr, s);
    if (st) return st;
    QG_TRY(cudaMemcpyAsync(cc, dcc.p, m * H * 8, cudaMemcpyDeviceToHost, s));
    return cuda_status(cudaStreamSynchronize(s));
  }
  if (K == 0) {
    std::memset(cc, 0, m * H * 8);
    return QG_OK;
  }
  const size_t Kt = ceil_div(K, (size_t)bk);
  cudaStream_t s0 = host_pipe().in;
  DevBuf dca(s0), dcb(s0), dcc(s0);
  QG_TRY(dcc.alloc(m * H * 8));
  QG_TRY(dca.alloc(qg_tiled_words(m, k, pl.e, bk) * 8));
  QG_TRY(dcb.alloc(qg_tiled_words(n, k, pl.e, bk) * 8));
  return host_pipeline(
      m, k, n, 128, ceil_div(n, (size_t)128), a, b,
      [&](const uint32_t* db, cudaStream_t s2) {
        return cuda_status(qgk::launch_pack_tiled(true, db, QG_U32, k, n, n, pl.t, pl.e, bk, (double*)dcb.p, s2, pl.p,
                                                  gp->balanced != 0));
      },
      [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s2, PhaseScope& ps, ChunkOut* out) {
        double* ca_chunk = (double*)dca.p + (r0 / 128) * Kt * 128 * bk;
        int st2 = cuda_status(qgk::launch_pack_tiled(false, da, QG_U32, rows, k, k, pl.t, pl.e, bk, ca_chunk, s2, pl.p,
                                                     gp->balanced != 0));
        if (st2) return st2;
        ps.begin(s2);
        if ((st2 = qg_mul_common_repacked_tiled(gp, ca_chunk, (const double*)dcb.p, rows, n, k,
                                                (double*)dcc.p + r0 * H, H, s2)))
          return st2;
        ps.end(s2);
        out->src = (const double*)dcc.p + r0 * H;
        out->dst = cc + r0 * H;
        out->bytes = rows * H * 8;
        return (int)QG_OK;
      });
}

int qg_host_mul_common_repacked(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                size_t n, double* cc) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // compress_rows_reversed's check, gemm.hpp:106
  qg_gpu_plan gp;
  if ((st = qg_gpu_plan_from(plan, k, &gp))) return st;
  return host_common_repacked(&gp, a, b, m, k, n, cc);
}

int qg_host_mul_common_repacked_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m,
                                    size_t k, size_t n, double* cc) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  int st = check_plan(&gplan->plan);
  if (st) return st;
  if (gplan->plan.t * gplan->plan.e > 53 || gplan->plan.t > 31) return QG_PLAN_MISMATCH;
  return host_common_repacked(gplan, a, b, m, k, n, cc);
}

// Multi-process (one rank per GPU) host path, SURVEY.md §8e all-gather form:
// each rank uploads and packs only its own tile-column slot of B, the slots
// are all-gathered by the caller (torch.distributed / NCCL), and the rank's
// row shard of A is streamed against the gathered CB_t.
int qg_host_pack_b_slot_tiled(const qg_gpu_plan* gplan, uint32_t bk, const uint32_t* b, size_t ldb, size_t k,
                              size_t c0, size_t cols, double* cb_slot, void* stream) {
  if (!gplan || (k * cols && !b) || (cols && !cb_slot)) return QG_INVALID_ARGUMENT;
  int st = check_plan(&gplan->plan);
  if (st) return st;
  if (ldb < c0 + cols) return QG_INVALID_ARGUMENT;
  if (k == 0 || cols == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  keep_pool_mapped();
  DevBuf db(s);
  QG_TRY(db.alloc(k * cols * 4));
  QG_TRY(host_pipe().stage.h2d(db.p, cols * 4, b + c0, ldb * 4, cols * 4, k, s));
  return qg_pack_b_tiled(gplan, bk, db.p, QG_U32, k, cols, cols, cb_slot, stream);
}

int qg_host_mul_common_packed_b(const qg_gpu_plan* gplan, const uint32_t* a, size_t m, size_t k, const double* cb_t,
                                size_t n, uint32_t* c, void* ready_event) {
  if (!gplan || (m * k && !a) || (m * n && !c) || (n && !cb_t)) return QG_INVALID_ARGUMENT;
  const qg_plan& pl = gplan->plan;
  int st = check_plan(&pl);
  if (st) return st;
  if (m == 0 || n == 0) return QG_OK;
  const size_t K = ceil_div(k, pl.e);
  if (K == 0) {
    std::memset(c, 0, m * n * 4);
    return QG_OK;
  }
  int bk = 0, kbs = 0;
  if ((st = tiled_geometry(gplan, K, &bk, &kbs))) return st;
  const size_t Kt = ceil_div(K, (size_t)bk);
  cudaStream_t s0 = host_pipe().in;
  DevBuf dca(s0), dc(s0);
  QG_TRY(dc.alloc(m * n * 4));
  QG_TRY(dca.alloc(qg_tiled_words(m, k, pl.e, bk) * 8));
  cudaEvent_t ready = static_cast<cudaEvent_t>(ready_event);
  return host_pipeline(
      m, k, n, 128, ceil_div(n, (size_t)128), a, nullptr,
      [&](const uint32_t*, cudaStream_t s2) {  // B is packed: order the contractions after its producer
        return ready ? cuda_status(cudaStreamWaitEvent(s2, ready, 0)) : (int)QG_OK;
      },
      [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s2, PhaseScope& ps, ChunkOut* out) {
        double* ca_chunk = (double*)dca.p + (r0 / 128) * Kt * 128 * bk;
        int st2 = cuda_status(qgk::launch_pack_tiled(false, da, QG_U32, rows, k, k, pl.t, pl.e, bk, ca_chunk, s2, pl.p,
                                                     gplan->balanced != 0));
        if (st2) return st2;
        ps.begin(s2);
        if ((st2 = qg_mul_common_tiled(gplan, ca_chunk, cb_t, rows, n, k, (int32_t*)dc.p + r0 * n, n, s2))) return st2;
        ps.end(s2);
        out->src = (const int32_t*)dc.p + r0 * n;
        out->dst = c + r0 * n;
        out->bytes = rows * n * 4;
        return (int)QG_OK;
      });
}

int qg_host_mul_common(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                       size_t k, size_t n, uint32_t* c) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // compress_rows_reversed's check, gemm.hpp:106
  qg_gpu_plan gp;
  if ((st = qg_gpu_plan_from(plan, k, &gp))) return st;
  return host_common(&gp, a, b, m, k, n, c);
}

int qg_host_mul_common_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b,
                           size_t m, size_t k, size_t n, uint32_t* c) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  int st = check_plan(&gplan->plan);
  if (st) return st;
  return host_common(gplan, a, b, m, k, n, c);
}

int qg_host_blocked_accumulate(const qg_plan* plan, const uint32_t* a, const uint32_t* b,
                               size_t m, size_t k, size_t n, size_t kpanel, uint32_t* c) {
  int st = check_plan(plan);
  if (st) return st;
  if (kpanel < 1) return QG_INVALID_ARGUMENT;             // gemm.hpp:455
  if (kpanel > plan->kmax) return QG_PLAN_MISMATCH;       // gemm.hpp:456
  cudaStream_t s = nullptr;
  if (m * n == 0) return QG_OK;
  PhaseScope ps;
  // Each panel is packed on its own (gemm.hpp:471-478) into words padded to a
  // whole number of 4-word k-steps, so k-blocks never straddle two panels.
  const size_t pw = ceil_div(kpanel, plan->e);
  const uint64_t exact = qg::max_exact_block(plan->p, plan->t, plan->e);
  size_t pw4 = ceil_div(pw, 4) * 4;
  uint64_t kb = 0;  // words per k-block, a divisor of pw4 in whole k-steps
  for (uint64_t steps = pw4 / 4; steps >= 1; --steps)
    if ((pw4 / 4) % steps == 0 && steps * 4 <= exact) {
      kb = steps * 4;
      break;
    }
  if (kb == 0) pw4 = pw;  // DMMA cannot be exact here: high-part kernel, panel = block
  const size_t npanels = k ? ceil_div(k, kpanel) : 0;
  const size_t W = npanels * pw4;
  DevBuf da(s), db(s), dca(s), dcb(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dca.alloc(m * W * 8));
  QG_TRY(dcb.alloc(W * n * 8));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  if (W == 0) {
    QG_TRY(cudaMemsetAsync(dc.p, 0, m * n * 4, s));
  } else {
    QG_TRY(qgk::launch_pack(qgk::PACK_ROWS_REVERSED, da.p, QG_U32, m, k, k, plan->t, plan->e,
                            (double*)dca.p, W, kpanel, pw4, s));
    QG_TRY(qgk::launch_pack(qgk::PACK_COLS_FORWARD, db.p, QG_U32, k, n, n, plan->t, plan->e,
                            (double*)dcb.p, n, kpanel, pw4, s));
    ps.begin(s);
    if (kb) {
      if ((st = run_common(*plan, kb, (const double*)dca.p, W, (const double*)dcb.p, n, m, n, W,
                           (int32_t*)dc.p, n, s)))
        return st;
    } else {
      qgk::HighArgs h;
      h.ca = (const double*)dca.p;
      h.ldca = W;
      h.cb = (const double*)dcb.p;
      h.ldcb = n;
      if (!dims_ok(m, n, W)) return QG_INVALID_ARGUMENT;
      h.M = (int)m;
      h.N = (int)n;
      h.K = (int)W;
      h.inv_qd = plan->inv_qd;
      h.kb_words = (int)pw4;
      h.qmask = (uint32_t)((1ull << plan->t) - 1);
      h.p = plan->p;
      h.acc = nullptr;
      h.c = (int32_t*)dc.p;
      h.ldc = n;
      if ((st = cuda_status(qgk::launch_dot_highpart(h, s, &g_last_kernel)))) return st;
    }
    ps.end(s);
  }
  QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

// Host-data right / left products on the tiled path. gp's kblock_words
// bounds the in-place REDQ blocks (kblock >= k: the reference's single block).
// The mixed variant with k split into parts (config 4): part p brings its
// rows of B (contiguous) and its columns of A (a 2-D copy) over PCIe, is
// packed, and is contracted over all of m x n with the accumulators starting
// from the previous parts' REDQ'd words (qg_dot.cu, EPI_REDQ accumulate). The
// first contraction starts after 1/P of the transfers instead of after all of
// B, every part's contraction fills the GPU, and the last part runs in row
// chunks whose words stream back while the next chunk computes.
// Unsigned plans (the accumulate mode loads canonical digits).
static bool use_ksplit(double packed_flop, size_t b_bytes, size_t k, size_t block) {
  const char* e = getenv("QG_HOST_KSPLIT");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return k >= 2 * (block ? block : 1);
  const double tc = packed_flop / 30e12, tb = (double)b_bytes / 50e9;
  return tc > tb && tc <= 3.0 * tb && k >= 8 * (block ? block : 512);
}

// rows_a / cols_b: rows of the contraction's A operand and columns of its B
// operand (right: m and ceil(n/e) words; left: ceil(m/e) words and n);
// row_align: A-operand rows per 128-row block of the packed layout.
static int host_redq_ksplit(
    const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n, size_t rows_a,
    size_t cols_b, double* cc,
    const std::function<int(const uint32_t* dap, size_t kp, uint32_t bkp, double* at, cudaStream_t s)>& pack_a,
    const std::function<int(const uint32_t* dbp, size_t kp, uint32_t bkp, double* bt, cudaStream_t s)>& pack_b) {
  HostPipe& hp = host_pipe();
  if (!hp.ok) return QG_CUDA_ERROR;
  PhaseScope ps;
  // parts: whole multiples of the in-place REDQ block (same block structure per part)
  int bk = 0, kbs = 0;
  int st = right_tiled_geometry(gp, k, &bk, &kbs);
  if (st) return st;
  const size_t blk = kbs ? (size_t)kbs * bk : k;
  size_t parts = 8;
  if (const char* e = getenv("QG_HOST_KPARTS")) parts = (size_t)atoi(e);  // experiments
  const size_t nblk = ceil_div(k, blk);
  if (parts > nblk) parts = nblk;
  if (parts < 1) parts = 1;
  const size_t blk_per = ceil_div(nblk, parts);
  parts = ceil_div(nblk, blk_per);
  const size_t kp_max = blk_per * blk;
  // per-part tiled buffers (the stage depth follows each part's own k, as in
  // redq_product), sized for the largest part
  auto part_geo = [&](size_t kp, int* bkp, size_t* ktp) {
    int kbsp = 0;
    const int st2 = right_tiled_geometry(gp, kp, bkp, &kbsp);
    *ktp = ceil_div(kp, (size_t)*bkp);
    return st2;
  };
  size_t wa = 0, wbt = 0;
  for (size_t pi = 0; pi < parts; ++pi) {
    const size_t kp = (k - pi * kp_max) < kp_max ? (k - pi * kp_max) : kp_max;
    int bkp = 0;
    size_t ktp = 0;
    if ((st = part_geo(kp, &bkp, &ktp))) return st;
    const size_t a_w = ceil_div(rows_a, 128) * 128 * ktp * bkp, b_w = ceil_div(cols_b, 128) * 128 * ktp * bkp;
    wa = a_w > wa ? a_w : wa;
    wbt = b_w > wbt ? b_w : wbt;
  }
  cudaStream_t s0 = hp.in;
  DevBuf da(s0), db(s0), dat(s0), dbt(s0), dcc(s0);
  PipeJoin join(hp);  // after the buffers: joins the streams before they are freed
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dat.alloc(2 * wa * 8));  // ping-pong: part p packs while part p-1 contracts
  QG_TRY(dbt.alloc(2 * wbt * 8));
  QG_TRY(dcc.alloc(rows_a * cols_b * 8));
  cudaStream_t cs = hp.comps[0], pk = hp.comps[1];  // contractions; packs (one part ahead)
  size_t ev = 0;
  std::vector<cudaEvent_t> contracted(parts, nullptr);
  for (size_t pi = 0; pi < parts; ++pi) {
    const size_t k0 = pi * kp_max, kp = (k - k0) < kp_max ? (k - k0) : kp_max;
    int bkp = 0;
    size_t ktp = 0;
    if ((st = part_geo(kp, &bkp, &ktp))) return st;
    uint32_t* dap = (uint32_t*)da.p + m * k0;  // m x kp, contiguous (A's columns k0..)
    uint32_t* dbp = (uint32_t*)db.p + k0 * n;  // kp x n, contiguous (B's rows k0..)
    QG_TRY(hp.stage.h2d(dbp, 0, b + k0 * n, 0, kp * n * 4, 1, hp.in));
    QG_TRY(hp.stage.h2d(dap, kp * 4, a + k0, k * 4, kp * 4, m, hp.in));
    cudaEvent_t ready = hp.event(ev++);
    if (!ready) return QG_CUDA_ERROR;
    QG_TRY(cudaEventRecord(ready, hp.in));
    QG_TRY(cudaStreamWaitEvent(pk, ready, 0));
    if (pi >= 2) QG_TRY(cudaStreamWaitEvent(pk, contracted[pi - 2], 0));  // its ping-pong buffers are free
    double* at = (double*)dat.p + (pi % 2) * wa;
    double* bt = (double*)dbt.p + (pi % 2) * wbt;
    if ((st = pack_a(dap, kp, (uint32_t)bkp, at, pk))) return st;
    if ((st = pack_b(dbp, kp, (uint32_t)bkp, bt, pk))) return st;
    cudaEvent_t packed = hp.event(ev++);
    if (!packed) return QG_CUDA_ERROR;
    QG_TRY(cudaEventRecord(packed, pk));
    QG_TRY(cudaStreamWaitEvent(cs, packed, 0));
    const bool last = pi + 1 == parts;
    const size_t rows_per = last ? 1024 : rows_a;  // the last part in row chunks: its words stream back
    for (size_t r0 = 0; r0 < rows_a; r0 += rows_per) {
      const size_t rows = (rows_a - r0) < rows_per ? (rows_a - r0) : rows_per;
      ps.begin(cs);
      if ((st = redq_product(gp, at + (r0 / 128) * ktp * 128 * bkp, bt, rows, kp, cols_b,
                             (double*)dcc.p + r0 * cols_b, cols_b, cs, pi > 0)))
        return st;
      ps.end(cs);
      if (last) {
        cudaEvent_t done_c = hp.event(ev++);
        if (!done_c) return QG_CUDA_ERROR;
        QG_TRY(cudaEventRecord(done_c, cs));
        QG_TRY(cudaStreamWaitEvent(hp.out, done_c, 0));
        QG_TRY(hp.stage.d2h(cc + r0 * cols_b, 0, (double*)dcc.p + r0 * cols_b, 0, rows * cols_b * 8, 1, hp.out));
      }
    }
    contracted[pi] = hp.event(ev++);
    if (!contracted[pi]) return QG_CUDA_ERROR;
    QG_TRY(cudaEventRecord(contracted[pi], cs));
  }
  QG_TRY(cudaStreamWaitEvent(hp.out, contracted[parts - 1], 0));
  QG_TRY(cudaEventRecord(hp.done, hp.out));
  QG_TRY(cudaStreamWaitEvent(hp.in, hp.done, 0));
  QG_TRY(cudaStreamSynchronize(hp.out));
  QG_TRY(hp.stage.finish());
  ps.finish();
  return QG_OK;
}

static int host_right_ksplit(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                             size_t n, double* cc) {
  const qg_plan* plan = &gp->plan;
  return host_redq_ksplit(
      gp, a, b, m, k, n, m, ceil_div(n, (size_t)plan->e), cc,
      [&](const uint32_t* dap, size_t kp, uint32_t bkp, double* at, cudaStream_t s) {
        return qg_pack_residues_tiled(bkp, dap, QG_U32, m, kp, kp, at, s);
      },
      [&](const uint32_t* dbp, size_t kp, uint32_t bkp, double* bt, cudaStream_t s) {
        return qg_pack_outer_cols_tiled(plan, bkp, dbp, QG_U32, kp, n, n, bt, s);
      });
}

static int host_left_ksplit(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                            size_t n, double* cc) {
  const qg_plan* plan = &gp->plan;
  return host_redq_ksplit(
      gp, a, b, m, k, n, ceil_div(m, (size_t)plan->e), n, cc,
      [&](const uint32_t* dap, size_t kp, uint32_t bkp, double* at, cudaStream_t s) {
        return qg_pack_outer_rows_tiled(plan, bkp, dap, QG_U32, m, kp, kp, at, s);
      },
      [&](const uint32_t* dbp, size_t kp, uint32_t bkp, double* bt, cudaStream_t s) {
        return qg_pack_residues_b_tiled(bkp, dbp, QG_U32, kp, n, n, bt, s);
      });
}

static int host_right(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                      double* cc) {
  const qg_plan* plan = &gp->plan;
  int st = check_plan(plan);
  if (st) return st;
  const size_t H = ceil_div(n, (size_t)plan->e);
  if (m * H == 0) return QG_OK;
  int bk = 0, kbs = 0;
  if ((st = right_tiled_geometry(gp, k ? k : 1, &bk, &kbs))) return st;
  if (gp->balanced == 0 && use_ksplit(2.0 * m * H * k, k * n * 4, k, kbs ? (size_t)kbs * bk : 0))
    return host_right_ksplit(gp, a, b, m, k, n, cc);
  const size_t kt = ceil_div(k ? k : 1, (size_t)bk);
  cudaStream_t s0 = host_pipe().in;
  DevBuf dat(s0), dbt(s0), dcc(s0);
  QG_TRY(dat.alloc(ceil_div(m, 128) * 128 * kt * bk * 8));
  QG_TRY(dbt.alloc(ceil_div(H, 128) * 128 * kt * bk * 8));
  QG_TRY(dcc.alloc(m * H * 8));
  const bool bal = gp->balanced != 0;
  const size_t Wt = kt * 128 * bk;  // words per 128-row / 128-word-column block
  const size_t e = (size_t)plan->e;
  if (use_pipeline2d(2.0 * m * H * k, k * n * 4))
    return host_pipeline2d(
        m, k, n, 128, 128 * e, 1, a, b,
        [&](size_t c0, size_t cols, const uint32_t* dbp, cudaStream_t s) {
          if (!k) return (int)QG_OK;
          double* dst = (double*)dbt.p + (c0 / e / 128) * Wt;
          return bal ? qg_pack_outer_cols_tiled_bal(plan, (uint32_t)bk, dbp, QG_U32, k, cols, cols, dst, s)
                     : qg_pack_outer_cols_tiled(plan, (uint32_t)bk, dbp, QG_U32, k, cols, cols, dst, s);
        },
        [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s) {
          if (!k) return (int)QG_OK;
          double* at = (double*)dat.p + (r0 / 128) * Wt;
          return bal ? qg_pack_residues_tiled_bal(plan->p, (uint32_t)bk, da, QG_U32, rows, k, k, at, s)
                     : qg_pack_residues_tiled((uint32_t)bk, da, QG_U32, rows, k, k, at, s);
        },
        [&](size_t r0, size_t rows, size_t c0, size_t cols, cudaStream_t s, PhaseScope& ps, TileOut* out) {
          const size_t h0 = c0 / e, hw = ceil_div(cols, e);
          ps.begin(s);
          int st2 = qg_mul_right_tiled(gp, (const double*)dat.p + (r0 / 128) * Wt,
                                       (const double*)dbt.p + (h0 / 128) * Wt, rows, k, cols,
                                       (double*)dcc.p + r0 * H + h0, H, s);
          if (st2) return st2;
          ps.end(s);
          out->src = (const double*)dcc.p + r0 * H + h0;
          out->dst = cc + r0 * H + h0;
          out->spitch = out->dpitch = H * 8;
          out->width = hw * 8;
          out->height = rows;
          return (int)QG_OK;
        });
  return host_pipeline(
      m, k, n, 128, ceil_div(H, (size_t)128), a, b,
      [&](const uint32_t* db, cudaStream_t s) {
        if (!k) return (int)QG_OK;
        return bal ? qg_pack_outer_cols_tiled_bal(plan, (uint32_t)bk, db, QG_U32, k, n, n, (double*)dbt.p, s)
                   : qg_pack_outer_cols_tiled(plan, (uint32_t)bk, db, QG_U32, k, n, n, (double*)dbt.p, s);
      },
      [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s, PhaseScope& ps, ChunkOut* out) {
        double* at = (double*)dat.p + (r0 / 128) * kt * 128 * bk;
        int st2 = QG_OK;
        if (k)
          st2 = bal ? qg_pack_residues_tiled_bal(plan->p, (uint32_t)bk, da, QG_U32, rows, k, k, at, s)
                    : qg_pack_residues_tiled((uint32_t)bk, da, QG_U32, rows, k, k, at, s);
        if (st2) return st2;
        ps.begin(s);
        if ((st2 = qg_mul_right_tiled(gp, at, (const double*)dbt.p, rows, k, n, (double*)dcc.p + r0 * H, H, s)))
          return st2;
        ps.end(s);
        out->src = (const double*)dcc.p + r0 * H;
        out->dst = cc + r0 * H;
        out->bytes = rows * H * 8;
        return (int)QG_OK;
      });
}

static int host_left(const qg_gpu_plan* gp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                     double* cc) {
  const qg_plan* plan = &gp->plan;
  int st = check_plan(plan);
  if (st) return st;
  const size_t e = plan->e, G = ceil_div(m, e);
  if (G * n == 0) return QG_OK;
  int bk = 0, kbs = 0;
  if ((st = right_tiled_geometry(gp, k ? k : 1, &bk, &kbs))) return st;
  if (gp->balanced == 0 && use_ksplit(2.0 * G * n * k, k * n * 4, k, kbs ? (size_t)kbs * bk : 0))
    return host_left_ksplit(gp, a, b, m, k, n, cc);
  const size_t kt = ceil_div(k ? k : 1, (size_t)bk);
  cudaStream_t s0 = host_pipe().in;
  DevBuf dat(s0), dbt(s0), dcc(s0);
  QG_TRY(dat.alloc(ceil_div(G, 128) * 128 * kt * bk * 8));
  QG_TRY(dbt.alloc(ceil_div(n, 128) * 128 * kt * bk * 8));
  QG_TRY(dcc.alloc(G * n * 8));
  const bool bal = gp->balanced != 0;
  return host_pipeline(
      m, k, n, 128 * e, ceil_div(n, (size_t)128), a, b,  // chunks of whole 128-group blocks of the outer-rows layout
      [&](const uint32_t* db, cudaStream_t s) {
        if (!k) return (int)QG_OK;
        return bal ? qg_pack_residues_b_tiled_bal(plan->p, (uint32_t)bk, db, QG_U32, k, n, n, (double*)dbt.p, s)
                   : qg_pack_residues_b_tiled((uint32_t)bk, db, QG_U32, k, n, n, (double*)dbt.p, s);
      },
      [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s, PhaseScope& ps, ChunkOut* out) {
        const size_t g0 = r0 / e, groups = ceil_div(rows, e);
        double* at = (double*)dat.p + (g0 / 128) * kt * 128 * bk;
        int st2 = QG_OK;
        if (k)
          st2 = bal ? qg_pack_outer_rows_tiled_bal(plan, (uint32_t)bk, da, QG_U32, rows, k, k, at, s)
                    : qg_pack_outer_rows_tiled(plan, (uint32_t)bk, da, QG_U32, rows, k, k, at, s);
        if (st2) return st2;
        ps.begin(s);
        if ((st2 = qg_mul_left_tiled(gp, at, (const double*)dbt.p, rows, k, n, (double*)dcc.p + g0 * n, n, s)))
          return st2;
        ps.end(s);
        out->src = (const double*)dcc.p + g0 * n;
        out->dst = cc + g0 * n;
        out->bytes = groups * n * 8;
        return (int)QG_OK;
      });
}

static qg_gpu_plan single_block(const qg_plan* plan, size_t k) {
  qg_gpu_plan gp;
  std::memset(&gp, 0, sizeof gp);
  gp.plan = *plan;
  gp.kblock_words = k ? k : 1;
  gp.max_exact_words = gp.kblock_words;
  return gp;
}

int qg_host_mul_right(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                      size_t k, size_t n, double* cc) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:295
  // one k-block under the caller's plan: words bit-identical to
  // mul_right_compressed(A, compress_outer_cols(B, plan)), gemm.hpp:320-325
  const qg_gpu_plan gp = single_block(plan, k);
  return host_right(&gp, a, b, m, k, n, cc);
}

int qg_host_mul_right_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                          size_t n, double* cc) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  return host_right(gplan, a, b, m, k, n, cc);
}

int qg_host_mul_left(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                     double* cc) {
  int st = check_plan(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:349 check_common_dim
  const qg_gpu_plan gp = single_block(plan, k);
  return host_left(&gp, a, b, m, k, n, cc);
}

int qg_host_mul_left_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                         size_t n, double* cc) {
  if (!gplan) return QG_INVALID_ARGUMENT;
  return host_left(gplan, a, b, m, k, n, cc);
}

int qg_host_mul_full(const qg_full_plan* fp, uint64_t kblock_words, const uint32_t* a, const uint32_t* b,
                     size_t m, size_t k, size_t n, uint32_t* c) {
  qg_gpu_plan gp;
  int st = full_gpu_plan(fp, kblock_words, k, &gp);
  if (st) return st;
  if (fp->base.beta > 53) return QG_PLAN_MISMATCH;  // gemm.hpp:383 check_backend
  if (!kblock_words && k > fp->base.kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:384
  if (m * n == 0) return QG_OK;
  const size_t qs = fp->dq + 1, ts = fp->dtheta + 1;
  const size_t G = ceil_div(m, qs), H = ceil_div(n, ts);
  int bk = 0, kbs = 0;
  if ((st = right_tiled_geometry(&gp, k ? k : 1, &bk, &kbs))) return st;
  const size_t kt = ceil_div(k ? k : 1, (size_t)bk);
  qg_plan pa = fp->base, pb = fp->base;
  pa.e = (int)qs;
  pa.d = (int)qs - 1;
  pb.t = fp->theta_exponent;
  pb.e = (int)ts;
  pb.d = (int)ts - 1;
  cudaStream_t s0 = host_pipe().in;
  DevBuf dat(s0), dbt(s0), dcc(s0), dc(s0);
  QG_TRY(dat.alloc(ceil_div(G, 128) * 128 * kt * bk * 8));
  QG_TRY(dbt.alloc(ceil_div(H, 128) * 128 * kt * bk * 8));
  QG_TRY(dcc.alloc(G * H * 8));
  QG_TRY(dc.alloc(m * n * 4));
  return host_pipeline(
      m, k, n, 128 * qs, ceil_div(H, (size_t)128), a, b,
      [&](const uint32_t* db, cudaStream_t s) {
        if (!k) return (int)QG_OK;
        return cuda_status(qgk::launch_pack_outer_tiled(db, QG_U32, k, n, n, pb.t, pb.e, bk, (double*)dbt.p, s));
      },
      [&](size_t r0, size_t rows, const uint32_t* da, cudaStream_t s, PhaseScope& ps, ChunkOut* out) {
        const size_t g0 = r0 / qs;
        double* at = (double*)dat.p + (g0 / 128) * kt * 128 * bk;
        int st2 = QG_OK;
        if (k && (st2 = cuda_status(qgk::launch_pack_outer_rows_tiled(da, QG_U32, rows, k, k, pa.t, pa.e, bk, at, s))))
          return st2;
        ps.begin(s);
        if ((st2 = qg_mul_full_tiled(fp, gp.kblock_words, at, (const double*)dbt.p, rows, k, n,
                                     (double*)dcc.p + g0 * H, H, s)))
          return st2;
        ps.end(s);
        if ((st2 = qg_uncompress_full(fp, (const double*)dcc.p + g0 * H, H, rows, n, (int32_t*)dc.p + r0 * n, n, s)))
          return st2;
        out->src = (const int32_t*)dc.p + r0 * n;
        out->dst = c + r0 * n;
        out->bytes = rows * n * 4;
        return (int)QG_OK;
      });
}


// extract_coefficient, pack.hpp:78-100, over a buffer of words (both modes).
int qg_extract_coefficients(const qg_plan* plan, const double* words, size_t count, int32_t* out, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (plan->extraction != 0 && plan->extraction != 1) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_extract_coefficients(words, count, plan->t, plan->d, plan->e, plan->inv_qd,
                                                      plan->extraction, plan->p, out, as_stream(stream)));
}

// reduce_and_compress, pack.hpp:141-155, on every row of a words matrix.
int qg_reduce_and_compress(const qg_plan* plan, const double* words, size_t rows, size_t cols, size_t ldw,
                           double* out, size_t ldo, void* stream) {
  int st = check_plan(plan);
  if (st) return st;
  if (plan->extraction != 0 && plan->extraction != 1) return QG_INVALID_ARGUMENT;
  if (ldw < cols || ldo < ceil_div(cols, (size_t)plan->e)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_reduce_and_compress(words, rows, cols, ldw, plan->t, plan->d, plan->e,
                                                     plan->inv_qd, plan->extraction, plan->p, out, ldo,
                                                     as_stream(stream)));
}

// naive_gemm, gemm.hpp:80-100, on the device.
int qg_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n, int32_t* c,
                  size_t ldc, void* stream) {
  if (p < 2 || !qg::is_prime(p)) return QG_INVALID_MODULUS;
  if (ldc < n) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_naive_gemm(a, b, m, k, n, p, c, ldc, as_stream(stream)));
}

int qg_host_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                       uint32_t* c) {
  if (p < 2 || !qg::is_prime(p)) return QG_INVALID_MODULUS;
  if (m * n == 0) return QG_OK;
  cudaStream_t s = nullptr;
  PhaseScope ps;
  DevBuf da(s), db(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  ps.begin(s);
  int st = qg_naive_gemm(p, (const uint32_t*)da.p, (const uint32_t*)db.p, m, k, n, (int32_t*)dc.p, n, s);
  if (st) return st;
  ps.end(s);
  QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

int qg_host_uncompress(const qg_plan* plan, qg_orientation o, const double* words, size_t stored_rows,
                       size_t stored_cols, size_t logical_rows, size_t logical_cols, uint32_t* out) {
  int st = check_plan(plan);
  if (st) return st;
  cudaStream_t s = nullptr;
  DevBuf dw(s), dout(s);
  QG_TRY(dw.alloc(stored_rows * stored_cols * 8));
  QG_TRY(dout.alloc(logical_rows * logical_cols * 4));
  if (stored_rows * stored_cols)
    QG_TRY(cudaMemcpyAsync(dw.p, words, stored_rows * stored_cols * 8, cudaMemcpyHostToDevice, s));
  if ((st = qg_uncompress(plan, o, (const double*)dw.p, stored_rows, stored_cols, logical_rows, logical_cols,
                          (int32_t*)dout.p, s)))
    return st;
  if (logical_rows * logical_cols)
    QG_TRY(cudaMemcpyAsync(out, dout.p, logical_rows * logical_cols * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  return QG_OK;
}

int qg_host_random_residue_matrix(size_t rows, size_t cols, uint32_t p, uint64_t seed, uint32_t* out) {
  if (rows * cols == 0) return (p < 2 || !qg::is_prime(p)) ? QG_INVALID_MODULUS : QG_OK;
  cudaStream_t s = nullptr;
  DevBuf d(s);
  QG_TRY(d.alloc(rows * cols * 4));
  int st = qg_gen_residues(seed, p, 0, rows, cols, d.p, QG_U32, s);
  if (st) return st;
  QG_TRY(cudaMemcpyAsync(out, d.p, rows * cols * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  return QG_OK;
}

void qg_set_phase_timing(int enable) { g_phase_timing.store(enable ? 1 : 0); }

void qg_last_phase_seconds(double* multiply, double* convert) {
  if (multiply) *multiply = g_phase.multiply;
  if (convert) *convert = g_phase.convert;
}

// ======================================================== Int64Word backend
// word.hpp:36-54: uint64 words, products wrap mod 2^64, beta up to 63. The
// entry points mirror the DoubleWord ones with uint64 word buffers.
static int check_plan_i64(const qg_plan* plan) {
  if (!plan) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !qg::is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->beta > 63) return QG_PLAN_MISMATCH;  // check_backend<Int64Word>, pack.hpp:19-24
  if (plan->t < 1 || plan->e < 1 || plan->d != plan->e - 1 || plan->t * plan->e > 63) return QG_PLAN_MISMATCH;
  return QG_OK;
}

static int pack_u64(int kind, const qg_plan* plan, const void* src, qg_dtype dtype, size_t rows, size_t cols,
                    size_t ld, uint64_t* out, size_t ldo, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  return cuda_status(qgk::launch_pack_u64(kind, src, dtype, rows, cols, ld, plan->t, plan->e, out, ldo, 0, 0,
                                          as_stream(stream)));
}

int qg_compress_rows_reversed_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda,
                                  uint64_t* ca, size_t ldca, void* stream) {
  if (!plan) return QG_INVALID_ARGUMENT;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:106
  if (lda < k || ldca < ceil_div(k, (size_t)plan->e)) return QG_INVALID_ARGUMENT;
  return pack_u64(qgk::PACK_ROWS_REVERSED, plan, a, dtype, m, k, lda, ca, ldca, stream);
}
int qg_compress_cols_forward_u64(const qg_plan* plan, const void* b, qg_dtype dtype, size_t k, size_t n, size_t ldb,
                                 uint64_t* cb, size_t ldcb, void* stream) {
  if (plan && k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:125
  if (ldb < n || ldcb < n) return QG_INVALID_ARGUMENT;
  return pack_u64(qgk::PACK_COLS_FORWARD, plan, b, dtype, k, n, ldb, cb, ldcb, stream);
}
int qg_compress_outer_cols_u64(const qg_plan* plan, const void* b, qg_dtype dtype, size_t rows, size_t cols,
                               size_t ldb, uint64_t* out, size_t ldo, void* stream) {
  if (ldb < cols || ldo < ceil_div(cols, (size_t)(plan ? plan->e : 1))) return QG_INVALID_ARGUMENT;
  return pack_u64(qgk::PACK_OUTER_COLS, plan, b, dtype, rows, cols, ldb, out, ldo, stream);
}
int qg_compress_outer_rows_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t rows, size_t cols,
                               size_t lda, uint64_t* out, size_t ldo, void* stream) {
  if (lda < cols || ldo < cols) return QG_INVALID_ARGUMENT;
  return pack_u64(qgk::PACK_OUTER_ROWS, plan, a, dtype, rows, cols, lda, out, ldo, stream);
}

// packed_common_product<Int64Word>, gemm.hpp:210-244: acc = sum of high parts.
int qg_packed_common_product_u64(const qg_plan* plan, const uint64_t* ca, const uint64_t* cb, size_t m, size_t n,
                                 size_t groups, uint64_t* acc, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  const uint64_t mask = (1ull << plan->t) - 1;
  return cuda_status(qgk::launch_gemm_u64(0, ca, -1, groups, cb, -1, n, m, n, groups, plan->t * plan->d, mask, acc, n,
                                          as_stream(stream)));
}
// reduce_common_entry<Int64Word>, gemm.hpp:247-250
int qg_reduce_common_u64(const qg_plan* plan, const uint64_t* acc, size_t count, int32_t* c, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  return cuda_status(qgk::launch_word_reduce_u64(acc, count, 0, 0, (1ull << plan->t) - 1, plan->p, c, 0,
                                                 as_stream(stream)));
}
// extract_coefficient<Int64Word>, pack.hpp:96-98
int qg_extract_coefficients_u64(const qg_plan* plan, const uint64_t* words, size_t count, int32_t* out, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  return cuda_status(qgk::launch_word_reduce_u64(words, count, 1, plan->t * plan->d, (1ull << plan->t) - 1, plan->p,
                                                 out, 0, as_stream(stream)));
}
int qg_reduce_and_compress_u64(const qg_plan* plan, const uint64_t* words, size_t rows, size_t cols, size_t ldw,
                               uint64_t* out, size_t ldo, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if (ldw < cols || ldo < ceil_div(cols, (size_t)plan->e)) return QG_INVALID_ARGUMENT;
  return cuda_status(qgk::launch_reduce_and_compress_u64(words, rows, cols, ldw, plan->t, plan->d, plan->e, plan->p,
                                                         out, ldo, as_stream(stream)));
}
// redq_in_place<Int64Word>, gemm.hpp:313-316
int qg_redq_u64(const qg_plan* plan, uint64_t* words, size_t count, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  cudaStream_t s = as_stream(stream);
  DeviceFlag flag(s);
  if (!flag.ptr) return QG_CUDA_ERROR;
  if ((st = cuda_status(qgk::launch_redq_u64(words, count, plan->t, plan->e, plan->p, flag.ptr, s)))) return st;
  int over = 0;
  if ((st = flag.read(&over))) return st;
  return over ? QG_DIGIT_OVERFLOW : QG_OK;
}
// uncompress<Int64Word>, gemm.hpp:182-204
int qg_uncompress_u64(const qg_plan* plan, qg_orientation o, const uint64_t* words, size_t stored_rows,
                      size_t stored_cols, size_t logical_rows, size_t logical_cols, int32_t* out, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if (o.slots < 1 || o.slots > plan->e) return QG_INVALID_ARGUMENT;
  cudaStream_t s = as_stream(stream);
  DeviceFlag flag(s);
  if (!flag.ptr) return QG_CUDA_ERROR;
  if ((st = cuda_status(qgk::launch_uncompress_u64(words, stored_rows, stored_cols, logical_rows, logical_cols,
                                                   plan->t, plan->e, o.slots, o.direction == 1, o.axis == 1,
                                                   plan->p, out, flag.ptr, s))))
    return st;
  int over = 0;
  if ((st = flag.read(&over))) return st;
  return over ? QG_DIGIT_OVERFLOW : QG_OK;
}
// packed_right_product<Int64Word> (gemm.hpp:285-310) and + REDQ (:320-325)
int qg_packed_right_product_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t lda, const uint64_t* cbo,
                                size_t m, size_t k, size_t n, uint64_t* cc, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:295
  if (lda < k) return QG_INVALID_ARGUMENT;
  const size_t H = ceil_div(n, (size_t)plan->e);
  if (k == 0) return m * H ? cuda_status(cudaMemsetAsync(cc, 0, m * H * 8, as_stream(stream))) : QG_OK;
  return cuda_status(qgk::launch_gemm_u64(1, a, dtype, lda, cbo, -1, H, m, H, k, 0, 0, cc, H, as_stream(stream)));
}
int qg_mul_right_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t lda, const uint64_t* cbo, size_t m,
                     size_t k, size_t n, uint64_t* cc, void* stream) {
  int st = qg_packed_right_product_u64(plan, a, dtype, lda, cbo, m, k, n, cc, stream);
  if (st) return st;
  return qg_redq_u64(plan, cc, m * ceil_div(n, (size_t)plan->e), stream);
}
// packed_left_product<Int64Word> (gemm.hpp:340-364) and + REDQ (:366-371)
int qg_packed_left_product_u64(const qg_plan* plan, const uint64_t* ca, const void* b, qg_dtype dtype, size_t ldb,
                               size_t m, size_t k, size_t n, uint64_t* cc, void* stream) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if ((st = check_dtype(dtype))) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:349
  if (ldb < n) return QG_INVALID_ARGUMENT;
  const size_t G = ceil_div(m, (size_t)plan->e);
  if (k == 0) return G * n ? cuda_status(cudaMemsetAsync(cc, 0, G * n * 8, as_stream(stream))) : QG_OK;
  return cuda_status(qgk::launch_gemm_u64(1, ca, -1, k, b, dtype, ldb, G, n, k, 0, 0, cc, n, as_stream(stream)));
}
int qg_mul_left_u64(const qg_plan* plan, const uint64_t* ca, const void* b, qg_dtype dtype, size_t ldb, size_t m,
                    size_t k, size_t n, uint64_t* cc, void* stream) {
  int st = qg_packed_left_product_u64(plan, ca, b, dtype, ldb, m, k, n, cc, stream);
  if (st) return st;
  return qg_redq_u64(plan, cc, ceil_div(m, (size_t)plan->e) * n, stream);
}
// mul_full_compressed<Int64Word>, gemm.hpp:377-445, on device residues.
int qg_mul_full_u64(const qg_full_plan* fp, const void* a, qg_dtype adt, const void* b, qg_dtype bdt, size_t m,
                    size_t k, size_t n, int32_t* c, size_t ldc, void* stream) {
  if (!fp) return QG_INVALID_ARGUMENT;
  int st = check_plan_i64(&fp->base);
  if (st) return st;
  if ((st = check_dtype(adt)) || (st = check_dtype(bdt))) return st;
  const int qs = fp->dq + 1, ts = fp->dtheta + 1;
  if (qs < 1 || ts < 1 || fp->base.e != qs * ts || fp->theta_exponent != fp->base.t * qs) return QG_PLAN_MISMATCH;
  if (k > fp->base.kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:384
  if (ldc < n) return QG_INVALID_ARGUMENT;
  if (m * n == 0) return QG_OK;
  cudaStream_t s = as_stream(stream);
  const size_t G = ceil_div(m, (size_t)qs), H = ceil_div(n, (size_t)ts);
  DevBuf ma(s), mb(s), acc(s);
  QG_TRY(ma.alloc(G * k * 8));
  QG_TRY(mb.alloc(k * H * 8));
  QG_TRY(acc.alloc(G * H * 8));
  if (k) {
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_OUTER_ROWS, a, adt, m, k, k, fp->base.t, qs, (uint64_t*)ma.p, k, 0, 0, s));
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_OUTER_COLS, b, bdt, k, n, n, fp->theta_exponent, ts, (uint64_t*)mb.p, H, 0,
                                0, s));
    QG_TRY(qgk::launch_gemm_u64(1, ma.p, -1, k, mb.p, -1, H, G, H, k, 0, 0, (uint64_t*)acc.p, H, s));
  } else {
    QG_TRY(cudaMemsetAsync(acc.p, 0, G * H * 8, s));
  }
  return cuda_status(qgk::launch_uncompress_full_u64((const uint64_t*)acc.p, H, m, n, fp->base.t, qs, ts, fp->base.p,
                                                     c, ldc, s));
}

// ---- host-data entries of the Int64Word backend (value semantics)
int qg_host_mul_common_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                           uint32_t* c) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:106
  if (m * n == 0) return QG_OK;
  cudaStream_t s = nullptr;
  PhaseScope ps;
  const size_t K = ceil_div(k, (size_t)plan->e);
  DevBuf da(s), db(s), dca(s), dcb(s), dacc(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dca.alloc(m * K * 8));
  QG_TRY(dcb.alloc(K * n * 8));
  QG_TRY(dacc.alloc(m * n * 8));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  if (K) {
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_ROWS_REVERSED, da.p, QG_U32, m, k, k, plan->t, plan->e, (uint64_t*)dca.p, K,
                                0, 0, s));
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_COLS_FORWARD, db.p, QG_U32, k, n, n, plan->t, plan->e, (uint64_t*)dcb.p, n,
                                0, 0, s));
  }
  ps.begin(s);
  if (K) {
    if ((st = qg_packed_common_product_u64(plan, (const uint64_t*)dca.p, (const uint64_t*)dcb.p, m, n, K,
                                           (uint64_t*)dacc.p, s)))
      return st;
  } else {
    QG_TRY(cudaMemsetAsync(dacc.p, 0, m * n * 8, s));
  }
  ps.end(s);
  if ((st = qg_reduce_common_u64(plan, (const uint64_t*)dacc.p, m * n, (int32_t*)dc.p, s))) return st;
  QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

int qg_host_blocked_accumulate_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                   size_t n, size_t kpanel, uint32_t* c) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if (kpanel < 1) return QG_INVALID_ARGUMENT;        // gemm.hpp:455
  if (kpanel > plan->kmax) return QG_PLAN_MISMATCH;  // gemm.hpp:456
  if (m * n == 0) return QG_OK;
  cudaStream_t s = nullptr;
  PhaseScope ps;
  const size_t Kp = ceil_div(kpanel, (size_t)plan->e);
  DevBuf da(s), db(s), dca(s), dcb(s), dacc(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dca.alloc(m * Kp * 8));
  QG_TRY(dcb.alloc(Kp * n * 8));
  QG_TRY(dacc.alloc(m * n * 8));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  QG_TRY(cudaMemsetAsync(dc.p, 0, m * n * 4, s));
  // one panel at a time (gemm.hpp:460-487): pack, common product, reduce, add mod p
  for (size_t k0 = 0; k0 < k; k0 += kpanel) {
    const size_t len = k - k0 < kpanel ? k - k0 : kpanel;
    const size_t W = ceil_div(len, (size_t)plan->e);
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_ROWS_REVERSED, (const uint32_t*)da.p + k0, QG_U32, m, len, k, plan->t,
                                plan->e, (uint64_t*)dca.p, W, 0, 0, s));
    QG_TRY(qgk::launch_pack_u64(qgk::PACK_COLS_FORWARD, (const uint32_t*)db.p + k0 * n, QG_U32, len, n, n, plan->t,
                                plan->e, (uint64_t*)dcb.p, n, 0, 0, s));
    ps.begin(s);
    QG_TRY(qgk::launch_gemm_u64(0, dca.p, -1, W, dcb.p, -1, n, m, n, W, plan->t * plan->d, (1ull << plan->t) - 1,
                                (uint64_t*)dacc.p, n, s));
    ps.end(s);
    QG_TRY(qgk::launch_word_reduce_u64((const uint64_t*)dacc.p, m * n, 0, 0, (1ull << plan->t) - 1, plan->p,
                                       (int32_t*)dc.p, 1, s));
  }
  QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

static int host_right_left_i64(bool left, const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                               size_t k, size_t n, uint64_t* cc) {
  int st = check_plan_i64(plan);
  if (st) return st;
  if (k > plan->kmax) return QG_PLAN_MISMATCH;
  const size_t e = plan->e;
  const size_t rows = left ? ceil_div(m, e) : m, cols = left ? n : ceil_div(n, e);
  if (rows * cols == 0) return QG_OK;
  cudaStream_t s = nullptr;
  PhaseScope ps;
  DevBuf da(s), db(s), dw(s), dcc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dw.alloc((left ? ceil_div(m, e) * k : k * ceil_div(n, e)) * 8));
  QG_TRY(dcc.alloc(rows * cols * 8));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  if (left) {
    if (k) QG_TRY(qgk::launch_pack_u64(qgk::PACK_OUTER_ROWS, da.p, QG_U32, m, k, k, plan->t, plan->e,
                                       (uint64_t*)dw.p, k, 0, 0, s));
    ps.begin(s);
    if ((st = qg_packed_left_product_u64(plan, (const uint64_t*)dw.p, db.p, QG_U32, n, m, k, n, (uint64_t*)dcc.p, s)))
      return st;
    ps.end(s);
  } else {
    if (k) QG_TRY(qgk::launch_pack_u64(qgk::PACK_OUTER_COLS, db.p, QG_U32, k, n, n, plan->t, plan->e,
                                       (uint64_t*)dw.p, ceil_div(n, e), 0, 0, s));
    ps.begin(s);
    if ((st = qg_packed_right_product_u64(plan, da.p, QG_U32, k, (const uint64_t*)dw.p, m, k, n, (uint64_t*)dcc.p, s)))
      return st;
    ps.end(s);
  }
  if ((st = qg_redq_u64(plan, (uint64_t*)dcc.p, rows * cols, s))) return st;
  QG_TRY(cudaMemcpyAsync(cc, dcc.p, rows * cols * 8, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

int qg_host_mul_right_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                          uint64_t* cc) {
  return host_right_left_i64(false, plan, a, b, m, k, n, cc);
}
int qg_host_mul_left_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                         uint64_t* cc) {
  return host_right_left_i64(true, plan, a, b, m, k, n, cc);
}

int qg_host_uncompress_u64(const qg_plan* plan, qg_orientation o, const uint64_t* words, size_t stored_rows,
                           size_t stored_cols, size_t logical_rows, size_t logical_cols, uint32_t* out) {
  int st = check_plan_i64(plan);
  if (st) return st;
  cudaStream_t s = nullptr;
  DevBuf dw(s), dout(s);
  QG_TRY(dw.alloc(stored_rows * stored_cols * 8));
  QG_TRY(dout.alloc(logical_rows * logical_cols * 4));
  if (stored_rows * stored_cols)
    QG_TRY(cudaMemcpyAsync(dw.p, words, stored_rows * stored_cols * 8, cudaMemcpyHostToDevice, s));
  if ((st = qg_uncompress_u64(plan, o, (const uint64_t*)dw.p, stored_rows, stored_cols, logical_rows, logical_cols,
                              (int32_t*)dout.p, s)))
    return st;
  if (logical_rows * logical_cols)
    QG_TRY(cudaMemcpyAsync(out, dout.p, logical_rows * logical_cols * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  return QG_OK;
}

int qg_host_mul_full_i64(const qg_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                         uint32_t* c) {
  if (!fp) return QG_INVALID_ARGUMENT;
  int st = check_plan_i64(&fp->base);
  if (st) return st;
  if (k > fp->base.kmax) return QG_PLAN_MISMATCH;
  if (m * n == 0) return QG_OK;
  cudaStream_t s = nullptr;
  PhaseScope ps;
  DevBuf da(s), db(s), dc(s);
  QG_TRY(da.alloc(m * k * 4));
  QG_TRY(db.alloc(k * n * 4));
  QG_TRY(dc.alloc(m * n * 4));
  if (m * k) QG_TRY(cudaMemcpyAsync(da.p, a, m * k * 4, cudaMemcpyHostToDevice, s));
  if (k * n) QG_TRY(cudaMemcpyAsync(db.p, b, k * n * 4, cudaMemcpyHostToDevice, s));
  ps.begin(s);
  if ((st = qg_mul_full_u64(fp, da.p, QG_U32, db.p, QG_U32, m, k, n, (int32_t*)dc.p, n, s))) return st;
  ps.end(s);
  QG_TRY(cudaMemcpyAsync(c, dc.p, m * n * 4, cudaMemcpyDeviceToHost, s));
  QG_TRY(cudaStreamSynchronize(s));
  ps.finish();
  return QG_OK;
}

}  // extern "C"
