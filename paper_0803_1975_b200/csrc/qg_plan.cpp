// qg_plan.cpp — host planners behind the C ABI (include/qgemm_b200.h).
//
// The reference planners (plan.hpp) are restated with identical results:
// tests/test_plan_parity.py checks them against the reference itself.
// The GPU planner is new: the reference keeps every partial sum exact by
// flooring each word product (word.hpp:28-30); a tensor-core contraction
// accumulates full products in FP64 and rounds, so blocks of the common
// dimension are sized by the exactness bound "Eq. G":
//
//   L_max(Kb) + rho * sum_{j=1..Kb} [ulp(x_max) + ulp(j x_max)] < Q^d,
//   ulp(Kb x_max) <= Q^d,
//
// with rho = 1 (faithful rounding, any order, products not fused) — more
// conservative than the measured DMMA behaviour (an RN FMA chain in k order,
// profiles/r01_fp64_probe.log).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>

#include "../../include/qgemm_b200.h"

using u128 = unsigned __int128;

namespace qg {

bool is_prime(uint64_t n) {  // field.hpp:42-48
  if (n < 2) return false;
  if (n % 2 == 0) return n == 2;
  for (uint64_t f = 3; f * f <= n; f += 2)
    if (n % f == 0) return false;
  return true;
}

static uint64_t pm1sq(uint32_t p) { return uint64_t(p - 1) * (p - 1); }

int minimal_radix_exponent(uint32_t p, uint64_t k) {  // plan.hpp:98-104
  const u128 bound = u128(k) * pm1sq(p);
  int t = 1;
  while ((u128(1) << t) <= bound) ++t;
  return t;
}

int word_capacity(int t, int beta) {  // plan.hpp:107-111
  int e = beta / t;
  if (e * t == beta) --e;
  return e;
}

uint64_t largest_common_dim(uint32_t p, int t) {  // plan.hpp:113-115
  return ((uint64_t(1) << t) - 1) / pm1sq(p);
}

static void fill(qg_plan* out, uint32_t p, int t, int e, int beta, double inv_qd) {
  std::memset(out, 0, sizeof *out);
  out->p = p;
  out->t = t;
  out->e = e;
  out->d = e - 1;
  out->beta = beta;
  out->kmax = largest_common_dim(p, t);
  out->inv_qd = inv_qd;
}

static int bitlen(u128 v) {
  int b = 0;
  while (v) {
    ++b;
    v >>= 1;
  }
  return b;
}

static u128 ulp_of(u128 v) {  // spacing of doubles at v (>= 1 for integers)
  const int b = bitlen(v);
  return b > 53 ? (u128(1) << (b - 53)) : u128(1);
}

// Largest rounding error of one FP64 operation whose exact result is the
// integer v: zero while v < 2^53 (integers there are representable).
static u128 round_err(u128 v) { return bitlen(v) > 53 ? ulp_of(v) : u128(0); }

// Largest number of packed words whose full-product FP64 accumulation keeps
// digit d exact (Eq. G). Digits below d are bounded by min(Q-1, Kb n_s (p-1)^2)
// — carry-free whenever a block holds at most kmax real residues, which the
// callers enforce separately (Eq. 3).
uint64_t max_exact_block(uint32_t p, int t, int e) {
  static std::mutex mu;
  static std::map<std::tuple<uint32_t, int, int>, uint64_t> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({p, t, e});
    if (it != cache.end()) return it->second;
  }
  const int d = e - 1;
  const u128 Q = u128(1) << t;
  const u128 Qd = u128(1) << (t * d);
  const u128 pm = pm1sq(p);
  u128 amax = 0;
  for (int i = 0; i < e; ++i) amax += u128(p - 1) << (t * i);
  const u128 xmax = amax * amax;  // < 2^106 for t*e <= 53
  const u128 err_x = round_err(xmax);
  u128 err = 0;
  uint64_t best = 0;
  const uint64_t cap = uint64_t(1) << 20;
  for (uint64_t kb = 1; kb <= cap; ++kb) {
    u128 L = 0;
    for (int s = 0; s < d; ++s) {
      const int ns = (s + 1) < (2 * d + 1 - s) ? (s + 1) : (2 * d + 1 - s);
      u128 ds = u128(kb) * ns * pm;
      if (ds > Q - 1) ds = Q - 1;
      L += ds << (t * s);
    }
    const u128 smax = u128(kb) * xmax;
    if (bitlen(smax) > 120) break;
    err += round_err(smax) + err_x;
    if (ulp_of(smax) > Qd) break;
    if (L + err >= Qd) break;
    // digit extraction adds 2^(td+52) with round-toward-zero: needs H < 2^52
    if ((smax >> (t * d)) >= (u128(1) << 52)) break;
    best = kb;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{p, t, e}] = best;
  return best;
}

// Per-word cost of a stage depth relative to the deepest (calibrated on B200
// with tools/plan_sweep.py, profiles/r01_plan_sweep_*.jsonl: short stages pay
// their fixed barrier/producer overhead over fewer words).
static double stage_cost(int bk) {
  // tiled kernel, profiles/r01_tiled_sweep_*.jsonl: stages of >= 20 words
  // run at the same per-word speed; 12-word stages pay ~5 %, 4-word ~50 %
  switch (bk) {
    case 52: return 1.02;  // two 104 KiB stages in flight only
    case 44: return 1.02;
    case 36: return 1.0;
    case 32: return 1.0;
    case 28: return 1.0;
    case 24: return 1.01;
    case 20: return 1.01;
    case 16: return 1.03;
    case 12: return 1.05;
    case 8: return 1.2;
    default: return 1.5;
  }
}
constexpr double kFlushWords = 3.0;  // per-block flush overhead, in packed words (measured 2.5-3.4)
constexpr double kAnchorFlushWords = 1.0;  // the same for the anchored contraction (K4A; measured 0.8-1.2)

// Eq. G for balanced digits: residues v > p/2 enter as
// v - p, so |v| <= h = floor(p/2), every digit is signed and digit d is read
// by rounding S / Q^d to nearest. Exact while |L| + err < Q^d / 2, with
// L_max = sum_{s<d} min(Q/2 - 1, Kb n_s h^2) Q^s; the anchor of the
// extraction needs |S| < 2^(td+50).
uint64_t max_exact_block_balanced(uint32_t p, int t, int e) {
  static std::mutex mu;
  static std::map<std::tuple<uint32_t, int, int>, uint64_t> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({p, t, e});
    if (it != cache.end()) return it->second;
  }
  const int d = e - 1;
  const u128 Q = u128(1) << t;
  const u128 Qd = u128(1) << (t * d);
  const u128 h = p / 2;
  const u128 h2 = h * h;
  u128 amax = 0;
  for (int i = 0; i < e; ++i) amax += h << (t * i);
  const u128 xmax = amax * amax;
  const u128 err_x = round_err(xmax);
  u128 err = 0;
  uint64_t best = 0;
  const uint64_t cap = uint64_t(1) << 20;
  for (uint64_t kb = 1; kb <= cap && t >= 2; ++kb) {
    u128 L = 0;
    for (int s = 0; s < d; ++s) {
      const int ns = (s + 1) < (2 * d + 1 - s) ? (s + 1) : (2 * d + 1 - s);
      u128 ds = u128(kb) * ns * h2;
      if (ds > Q / 2 - 1) ds = Q / 2 - 1;
      L += ds << (t * s);
    }
    const u128 smax = u128(kb) * xmax;
    if (bitlen(smax) > 120) break;
    err += round_err(smax) + err_x;
    if (ulp_of(smax) > Qd) break;
    if (2 * (L + err) >= Qd) break;
    if ((smax >> (t * d)) >= (u128(1) << 50)) break;
    best = kb;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{p, t, e}] = best;
  return best;
}

// Anchored accumulation (K4A, qg_anchor.cu): the first DMMA of
// a block takes C = A0 = 1.5 2^E + Q^d/2 + Q^(d+1)/2 (+ Q^(d+1) in the odd
// columns) and every partial sum of the block stays in the binade
// [2^E, 2^(E+1)), so every rounding has the same ulp u = 2^(E-52) and digit d
// of the block sits at bits [s, s+t) of the result's low word, s = t d -
// (E - 52). Returns the smallest E that keeps a block of kb words in the
// binade (0 if none is exact):
//   off + kb x_max + err < 2^(E-1)            (range, off = Q^d/2 + Q^(d+1)/2 + Q^(d+1))
//   2 (L_max(kb) + err) < Q^d                 (Eq. G with the fixed ulp)
//   err = kb (u + ulp(x_max))                 (one product and one add rounding
//                                              per word, faithful, any order)
//   1 <= s, s + t <= 32                       (Q^d/2 on the grid; low word)
int anchored_exponent(uint32_t p, int t, int e, uint64_t kb) {
  const int d = e - 1;
  if (t < 2 || d < 1 || kb == 0 || t * e > 53) return 0;
  const u128 Q = u128(1) << t;
  const u128 Qd = u128(1) << (t * d);
  const u128 h = p / 2;
  const u128 h2 = h * h;
  if (h == 0) return 0;
  u128 amax = 0;
  for (int i = 0; i < e; ++i) amax += h << (t * i);
  const u128 xmax = amax * amax;
  if (bitlen(xmax) > 100) return 0;
  const u128 err_x = round_err(xmax);
  const u128 off = Qd / 2 + (Qd << t) / 2 + (Qd << t);  // rounding half, Q/2 bias, the odd columns' Q^(d+1)
  u128 L = 0;
  for (int s = 0; s < d; ++s) {
    const int ns = (s + 1) < (2 * d + 1 - s) ? (s + 1) : (2 * d + 1 - s);
    u128 ds = u128(kb) * ns * h2;
    if (ds > Q / 2 - 1) ds = Q / 2 - 1;
    L += ds << (t * s);
  }
  for (int E = bitlen(u128(kb) * xmax) + 1; E <= t * d + 51; ++E) {
    if (E < 53) continue;
    const u128 u = u128(1) << (E - 52);
    const u128 err = u128(kb) * (u + err_x);
    if (off + u128(kb) * xmax + err >= (u128(1) << (E - 1))) continue;  // leaves the binade: try the next one
    const int s = t * d - (E - 52);
    if (s + t > 32) continue;           // digit field above the low word: a coarser grid lowers it
    if (s < 1) return 0;
    if (2 * (L + err) >= Qd) return 0;  // a larger E only adds error
    return E;
  }
  return 0;
}

uint64_t max_exact_block_anchored(uint32_t p, int t, int e) {
  static std::mutex mu;
  static std::map<std::tuple<uint32_t, int, int>, uint64_t> cache;
  {
    std::lock_guard<std::mutex> lk(mu);
    auto it = cache.find({p, t, e});
    if (it != cache.end()) return it->second;
  }
  uint64_t best = 0;
  // not monotone at binade steps (a block may need the next E and fail where a slightly longer
  // one fails too): scan and keep the largest
  for (uint64_t kb = 1; kb <= 4096; ++kb) {
    if (anchored_exponent(p, t, e, kb)) best = kb;
    else if (kb > 2 * best + 8) break;
  }
  std::lock_guard<std::mutex> lk(mu);
  cache[{p, t, e}] = best;
  return best;
}

// K4A has kernels for blocks of an odd multiple of 4 words (conflict-free fragment loads) up to 52;
// the tiled layout of an anchored plan has stage depth = block.
int anchored_stage(uint64_t kb) { return (kb >= 12 && kb <= 52 && kb % 8 == 4) ? int(kb) : 0; }

// Eq. 3 for balanced digits: a block may hold at most this many residues.
uint64_t largest_common_dim_balanced(uint32_t p, int t) {
  const uint64_t h = p / 2;
  if (t < 2 || h == 0) return 0;
  return ((uint64_t(1) << (t - 1)) - 1) / (h * h);
}

// The contraction kernels flush k-blocks at pipeline-stage boundaries. The
// tiled kernel (the main path) has stages of BK in {36, 28, 20, 12, 4} words,
// the row-layout kernels of BK in {32, 28, 24, 16, 8, 4}. Picks the stage
// depth (and the block BK * j <= limit) with the least predicted per-word
// cost; returns the block length, *bk the stage depth.
static uint64_t stage_block_set(uint64_t limit, int* bk, const int* set, int nset) {
  uint64_t best = 0;
  int best_bk = 0;
  double best_cost = 1e300;
  for (int i = 0; i < nset; ++i) {
    const int b = set[i];
    if (uint64_t(b) > limit) continue;
    const uint64_t blk = limit / b * b;
    const double cost = stage_cost(b) + kFlushWords / double(blk);
    if (cost < best_cost - 1e-12) {
      best_cost = cost;
      best = blk;
      best_bk = b;
    }
  }
  if (bk) *bk = best_bk;
  return best;
}

uint64_t stage_block(uint64_t limit, int* bk) {
  static const int kSet[] = {32, 28, 24, 16, 8, 4};
  return stage_block_set(limit, bk, kSet, 6);
}

uint64_t stage_block_tiled(uint64_t limit, int* bk) {
  static const int kSet[] = {52, 44, 36, 28, 20, 12, 4};
  return stage_block_set(limit, bk, kSet, 7);
}

// Stage depths the REDQ-epilogue (right / left / full) kernels are built for.
uint64_t stage_block_redq(uint64_t limit, int* bk) {
  static const int kSet[] = {36, 28, 20, 12, 4};
  return stage_block_set(limit, bk, kSet, 5);
}

// Stage depth for a single-block contraction of K words: least padded work
// ceil(K/BK) BK x stage cost (config 3, K = 52: BK = 52, no padding; long K:
// 28/36-word stages, which keep 3-4 stages in flight).
int stage_single(uint64_t K) {
  static const int kSet[] = {52, 44, 36, 28, 20, 12, 4};
  int best = 28;
  double best_cost = 1e300;
  for (int b : kSet) {
    const double cost = double((K + b - 1) / b * b) * stage_cost(b);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      best = b;
    }
  }
  return best;
}

// Predicted relative cost of a blocked plan, in packed-word units: words
// rounded up to the stage depth times the stage's per-word overhead, plus a
// per-block flush cost.
double blocked_cost(uint64_t k, int e, uint64_t kb_words, double flush_words) {
  const uint64_t K = (k + e - 1) / e;
  if (kb_words >= K) {  // single block
    const int b = stage_single(K);
    return double((K + b - 1) / b * b) * stage_cost(b);
  }
  int bk = 4;
  const uint64_t blk = stage_block_tiled(kb_words, &bk);
  if (blk == 0) return 1e300;
  const uint64_t Kpad = (K + bk - 1) / bk * bk;
  const uint64_t nblocks = (K + blk - 1) / blk;
  return double(Kpad) * stage_cost(bk) + flush_words * double(nblocks);
}

}  // namespace qg

using namespace qg;

extern "C" {

int qg_abi_version(void) { return QG_ABI_VERSION; }

const char* qg_status_string(int s) {
  switch (s) {
    case QG_OK: return "ok";
    case QG_INVALID_MODULUS: return "InvalidModulus";
    case QG_NO_COMPRESSION: return "NoCompression";
    case QG_SLOT_OVERFLOW: return "SlotOverflow";
    case QG_DIGIT_OVERFLOW: return "DigitOverflow";
    case QG_DIMENSION_MISMATCH: return "DimensionMismatch";
    case QG_PLAN_MISMATCH: return "PlanMismatch";
    case QG_UNSUPPORTED_ALGORITHM: return "UnsupportedAlgorithm";
    case QG_PARSE_ERROR: return "ParseError";
    case QG_INVALID_ARGUMENT: return "InvalidArgument";
    case QG_CUDA_ERROR: return "CudaError";
    case QG_NCCL_ERROR: return "NcclError";
    case QG_NOT_EXACT: return "NotExact";
  }
  return "unknown";
}

int qg_plan_compression(uint32_t p, uint64_t k, int beta, int mode, qg_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;  // field.hpp:19-21
  if (k < 1 || beta < 2) return QG_INVALID_ARGUMENT;     // plan.hpp:128-129
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QG_NO_COMPRESSION;  // plan.hpp:132-135
  const int e_raw = word_capacity(t, beta);
  const int e = int(uint64_t(e_raw) < k ? uint64_t(e_raw) : k);
  if (e < 2) return QG_NO_COMPRESSION;  // plan.hpp:138-140
  fill(out, p, t, e, beta, std::ldexp(1.0, -t * (e - 1)));
  out->extraction = mode;
  if (mode == QG_EXTRACT_ADD_HIGH_BITS) {  // plan.hpp:150-157
    const long double limit = std::exp2l(static_cast<long double>(t) - 1.0L / e);
    uint64_t km = out->kmax;
    while (km > 0 && static_cast<long double>(km) * pm1sq(p) >= limit) --km;
    out->kmax = km;
  }
  return QG_OK;
}

int qg_uncompressed_plan(uint32_t p, uint64_t k, int beta, qg_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1) return QG_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QG_NO_COMPRESSION;
  fill(out, p, t, 1, beta, 1.0);
  return QG_OK;
}

int qg_plan_packed_axis(uint32_t p, uint64_t k, uint64_t axis_len, int beta, qg_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1 || axis_len < 1) return QG_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  if (t >= beta) return QG_NO_COMPRESSION;
  const uint64_t cap = uint64_t(word_capacity(t, beta));
  const int e = int(cap < axis_len ? cap : axis_len);
  fill(out, p, t, e, beta, std::ldexp(1.0, -t * (e - 1)));
  return QG_OK;
}

int qg_choose_panel(uint32_t p, uint64_t k, int beta, uint64_t* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1 || beta < 2) return QG_INVALID_ARGUMENT;
  int direct_e = 1;
  qg_plan pl;
  if (qg_plan_compression(p, k, beta, 0, &pl) == QG_OK) direct_e = pl.e;
  for (int t = 1; t < beta; ++t) {  // plan.hpp:215-222
    const uint64_t km = largest_common_dim(p, t);
    if (km == 0) continue;
    const uint64_t panel = km < k ? km : k;
    const uint64_t cap = uint64_t(word_capacity(t, beta));
    const int e = int(cap < panel ? cap : panel);
    if (e > direct_e) {
      *out = panel;
      return QG_OK;
    }
  }
  *out = 0;
  return QG_OK;
}

int qg_max_exact_block(const qg_plan* plan, uint64_t* words) {
  if (!plan || !words) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->e < 1 || plan->t < 1 || plan->t * plan->e > 53) return QG_PLAN_MISMATCH;
  *words = max_exact_block(plan->p, plan->t, plan->e);
  return QG_OK;
}

// Mixed (right) variant, gemm.hpp:285-335, on the tensor-core path: every
// partial sum A x CBo is an exact integer below Q^e <= 2^53, so no rounding
// bound applies; k is blocked only to keep digits below Q: the kernel
// REDQs the accumulators in place between blocks (digits drop below p), so a
// block may add kb residues with (p-1) + kb (p-1)^2 < Q. Picks (t, e, kb)
// minimising words x (1 + flush cost / kb); e <= n as plan_packed_axis does.
int qg_plan_right_gpu(uint32_t p, uint64_t k, uint64_t n, qg_gpu_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1 || n < 1) return QG_INVALID_ARGUMENT;
  double best_cost = 1e300;
  bool found = false;
  qg_gpu_plan best;
  std::memset(&best, 0, sizeof best);
  // unsigned digits: a block may add kb residues with (p-1) + kb (p-1)^2 < Q;
  // balanced digits (|v| <= p/2): h + kb h^2 < Q/2 with h = p/2 — 2x longer
  // blocks for odd p (qg_dot.cu, redq_words_inplace_bal)
  for (int bal = 0; bal <= 1; ++bal) {
    const uint64_t h = bal ? p / 2 : p - 1;
    const uint64_t pm = h * h ? h * h : 1;
    for (int e = 1; e <= 26; ++e) {
      if (uint64_t(e) > n && e > 1) break;
      const int t = 52 / e;  // largest t with t e <= 52: words stay below 2^52
      if (t < 2 || t > 52 || (bal && t > 31)) continue;
      const uint64_t Q = uint64_t(1) << t, lim = bal ? Q / 2 : Q;
      const uint64_t km = (lim - 1) / pm;  // one block: k h^2 < lim
      if (km == 0) continue;
      uint64_t kb;
      if (k <= km && (bal || k <= largest_common_dim(p, t))) kb = k;  // one block (gemm.hpp:295 for unsigned)
      else {
        if (lim <= h + 1) continue;
        kb = (lim - 1 - h) / pm;
        if (kb < 4) continue;
        kb = stage_block_redq(kb, nullptr);
        if (kb == 0) continue;
      }
      // cost in residue-steps of the contraction per output word: stage-padded
      // k at the stage's cost, plus a calibrated in-place REDQ per block
      // (config 4 on B200: ~5.5 e unsigned, ~11 e balanced; profiles/r01_notes.md)
      int bk = 28;
      if (kb < k) stage_block_redq(kb, &bk);
      const double H = double((n + e - 1) / e);
      const double nflush = kb >= k ? 0.0 : double((k + kb - 1) / kb);
      const double cost = H * (double((k + bk - 1) / bk * bk) * stage_cost(bk) + (bal ? 11.0 : 5.5) * e * nflush);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        found = true;
        fill(&best.plan, p, t, e, 53, std::ldexp(1.0, -t * (e - 1)));
        best.kblock_words = kb;  // residues of k per block
        best.max_exact_words = kb;
        best.balanced = bal;
      }
    }
  }
  if (!found) return QG_NO_COMPRESSION;
  *out = best;
  return QG_OK;
}

// plan_full, plan.hpp:229-252: the word capacity at the minimal radix for k,
// split into dq+1 = floor(sqrt(E)) base-Q slots and dtheta+1 = E/(dq+1)
// base-Theta slots, Theta = Q^(dq+1).
static void fill_full(qg_full_plan* out, uint32_t p, int t, int qs, int ts, int beta, uint64_t kmax) {
  std::memset(out, 0, sizeof *out);
  fill(&out->base, p, t, qs * ts, beta, std::ldexp(1.0, -t * (qs * ts - 1)));
  out->base.kmax = kmax;
  out->dq = qs - 1;
  out->dtheta = ts - 1;
  out->theta_exponent = t * qs;
}

static int isqrt_int(int v) {
  int r = int(std::sqrt(double(v)));
  while (r * r > v) --r;
  while ((r + 1) * (r + 1) <= v) ++r;
  return r;
}

int qg_plan_full(uint32_t p, uint64_t k, int beta, qg_full_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1 || beta < 2) return QG_INVALID_ARGUMENT;
  const int t = minimal_radix_exponent(p, k);
  const int capacity = t < beta ? word_capacity(t, beta) : 0;
  if (capacity < 4) return QG_NO_COMPRESSION;  // plan.hpp:235-237
  const int qs = isqrt_int(capacity);
  fill_full(out, p, t, qs, capacity / qs, beta, largest_common_dim(p, t));
  return QG_OK;
}

// GPU planner for the full variant: the same slot split as plan_full, but t
// and the k-block are free. A block of kb residues keeps every digit exact
// after the in-place REDQ while (p-1) + kb (p-1)^2 < Q; cost is packed-word
// products (k / ((dq+1)(dtheta+1)) per output cell) plus a per-flush REDQ of
// e digits, as in qg_plan_right_gpu.
int qg_plan_full_gpu(uint32_t p, uint64_t k, qg_full_plan* out, uint64_t* kblock_words) {
  if (!out || !kblock_words) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1) return QG_INVALID_ARGUMENT;
  const uint64_t pm = pm1sq(p);
  double best_cost = 1e300;
  bool found = false;
  for (int t = 1; t <= 52; ++t) {
    const int cap = word_capacity(t, 53);
    if (cap < 1) continue;
    const int qs = isqrt_int(cap), ts = cap / qs, e = qs * ts;
    const uint64_t Q = uint64_t(1) << t;
    const uint64_t km = largest_common_dim(p, t);
    if (km == 0) continue;
    uint64_t kb;
    if (k <= km) kb = k;
    else {
      if (Q <= p) continue;
      kb = (Q - p) / (pm ? pm : 1);
      if (kb < 4) continue;
      kb = stage_block_redq(kb, nullptr);
      if (kb == 0) continue;
    }
    int bk = 28;
    if (kb < k) stage_block_redq(kb, &bk);
    const double nflush = kb >= k ? 0.0 : double((k + kb - 1) / kb);
    // as qg_plan_right_gpu: stage-padded k at the stage's cost + calibrated REDQ flushes
    const double cost = (double((k + bk - 1) / bk * bk) * stage_cost(bk) + 5.5 * e * nflush) / double(e);
    if (cost < best_cost - 1e-9) {
      best_cost = cost;
      found = true;
      fill_full(out, p, t, qs, ts, 53, km);
      *kblock_words = kb;
    }
  }
  return found ? QG_OK : QG_NO_COMPRESSION;
}

int qg_max_exact_block_balanced(const qg_plan* plan, uint64_t* words) {
  if (!plan || !words) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->e < 1 || plan->t < 1 || plan->t * plan->e > 53) return QG_PLAN_MISMATCH;
  *words = max_exact_block_balanced(plan->p, plan->t, plan->e);
  return QG_OK;
}

int qg_max_exact_block_anchored(const qg_plan* plan, uint64_t* words, int* exponent) {
  if (!plan || !words) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->e < 1 || plan->t < 1 || plan->t * plan->e > 53) return QG_PLAN_MISMATCH;
  *words = max_exact_block_anchored(plan->p, plan->t, plan->e);
  if (exponent) *exponent = *words ? anchored_exponent(plan->p, plan->t, plan->e, *words) : 0;
  return QG_OK;
}

int qg_gpu_plan_from(const qg_plan* plan, uint64_t k, qg_gpu_plan* out) {
  if (!plan || !out) return QG_INVALID_ARGUMENT;
  if (plan->p < 2 || !is_prime(plan->p)) return QG_INVALID_MODULUS;
  if (plan->e < 1 || plan->t < 1 || plan->t * plan->e > 53 || plan->beta > 53)
    return QG_PLAN_MISMATCH;
  std::memset(out, 0, sizeof *out);
  out->plan = *plan;
  const uint64_t exact = max_exact_block(plan->p, plan->t, plan->e);
  out->max_exact_words = exact;
  const uint64_t K = (k + plan->e - 1) / plan->e;
  uint64_t kb = exact;
  // Eq. 3 per block: a block may hold at most kmax real residues. When the
  // whole common dimension already satisfies it, any blocking does.
  if (k > plan->kmax) {
    const uint64_t lim = plan->kmax / uint64_t(plan->e);
    if (lim < kb) kb = lim;
  }
  if (kb >= K) kb = K;  // single block
  out->kblock_words = kb;
  return QG_OK;
}

int qg_plan_gpu(uint32_t p, uint64_t k, qg_gpu_plan* out) { return qg_plan_gpu_ex(p, k, 0, out); }

int qg_plan_gpu_ex(uint32_t p, uint64_t k, int flags, qg_gpu_plan* out) {
  if (!out) return QG_INVALID_ARGUMENT;
  if (p < 2 || !is_prime(p)) return QG_INVALID_MODULUS;
  if (k < 1) return QG_INVALID_ARGUMENT;
  const double flush_words = kFlushWords;
  double best_cost = 1e300, anch_cost = 1e300;
  bool found = false;
  qg_gpu_plan best, anch;
  std::memset(&best, 0, sizeof best);
  std::memset(&anch, 0, sizeof anch);
  const int max_bal = (flags & QG_PLAN_UNSIGNED_ONLY) ? 0 : 1;
  for (int bal = 0; bal <= max_bal; ++bal)
  for (int t = 1; t < 53; ++t) {
    const uint64_t km = bal ? largest_common_dim_balanced(p, t) : largest_common_dim(p, t);
    if (km == 0) continue;
    const int cap = word_capacity(t, 53);
    for (int e = 1; e <= cap; ++e) {
      if (uint64_t(e) > k && e > 1) break;
      const uint64_t exact = bal ? max_exact_block_balanced(p, t, e) : max_exact_block(p, t, e);
      uint64_t kb = exact;
      if (k > km) {
        const uint64_t lim = km / uint64_t(e);
        if (lim < kb) kb = lim;
      }
      const uint64_t K = (k + e - 1) / e;
      if (kb >= K) kb = K;
      else kb = stage_block_tiled(kb, nullptr);  // multi-block plans flush at stage ends
      if (kb == 0 || (kb < 4 && kb < K)) continue;
      const uint64_t nblocks = (K + kb - 1) / kb;
      // digit sums of all blocks must fit the kernel's uint32 accumulator
      if (u128(nblocks + 1) * ((u128(1) << t) - 1) + p >= (u128(1) << 32)) continue;
      const double cost = blocked_cost(k, e, kb, flush_words);
      if (cost < best_cost - 1e-9) {
        best_cost = cost;
        found = true;
        fill(&best.plan, p, t, e, 53, std::ldexp(1.0, -t * (e - 1)));
        best.kblock_words = kb;
        best.max_exact_words = exact;
        best.balanced = bal;
        best.anchored = 0;
      }
      // the same (t, e) with anchored accumulation (K4A): shorter blocks (an odd multiple of 4
      // words <= 52), but the block flush is integer-pipe only: ~1 word per block instead of ~3
      // (config 5: 12-word blocks 92.9 % vs 20-word blocks 86.7 % of the DMMA peak)
      if (bal && !(flags & QG_PLAN_NO_ANCHOR) && e >= 2) {
        uint64_t ka = max_exact_block_anchored(p, t, e);
        if (k > km && km / uint64_t(e) < ka) ka = km / uint64_t(e);
        if (ka > 52) ka = 52;
        while (ka >= 12 && !(ka % 8 == 4 && anchored_exponent(p, t, e, ka))) --ka;
        if (ka >= 12 && 16 * ka <= K) {  // long products only: short ones run the small-product kernel (K9)
          const uint64_t nb = (K + ka - 1) / ka;
          const int E = anchored_exponent(p, t, e, ka);
          const int sh = t * (e - 1) - (E - 52);
          if ((u128(nb + 3) * ((u128(1) << t) - 1) << sh) + 2 * p < (u128(1) << 32)) {
            const double acost = double(nb * ka) + kAnchorFlushWords * double(nb);
            if (acost < anch_cost - 1e-9) {
              anch_cost = acost;
              fill(&anch.plan, p, t, e, 53, std::ldexp(1.0, -t * (e - 1)));
              anch.kblock_words = ka;
              anch.max_exact_words = exact;
              anch.balanced = 1;
              anch.anchored = 1;
            }
          }
        }
      }
    }
  }
  if (!found) return QG_NO_COMPRESSION;
  // the anchored plan is taken only when clearly ahead (3 %): other entries (the small-product
  // and the repacking kernels) run an anchored plan's shorter blocks with the FP64 flush
  *out = anch_cost < 0.97 * best_cost ? anch : best;
  return QG_OK;
}

}  // extern "C"
