// qg_dot.cu — the packed contractions on the FP64 tensor cores of sm_100a.
//
// sm_100a has no FP64 kind for tcgen05.mma (ptxas rejects .kind::f64), so the
// FP64 tensor path is the warp-level mma.sync.m8n8k4.f64, which ptxas lowers
// to SASS DMMA.8x8x4 (37.1 TFLOP/s measured on B200, profiles/r01_*). The
// operands are staged global -> shared by cp.async (LDGSTS, zero-filling
// the ragged edges) in a multi-stage ring and fed to DMMA from shared memory.
// CTA tile 128x128, 8 warps, each owning a 64x32 tile: 64 FP64 accumulators
// and 32 DMMAs per 4-word k-step per warp, 12 fragment loads per k-step.
//
// K4 (common / dot-product variant, gemm.hpp:210-271 + 450-489): the FP64
// accumulators hold sum_g CA[i][g] CB[g][j] over one k-block. Blocks end on
// pipeline-stage boundaries (stage depth BK is a template parameter chosen
// by the host so that blocks align with stages; no branch sits inside the
// unrolled DMMA sequence). At a block end every accumulator is added with
// round-toward-zero to the anchor 2^(td+52): the sum's ulp is then exactly
// Q^d, so its low mantissa bits ARE floor(acc / Q^d) — one DADD.RZ and one
// LOP3 per accumulator give digit d, which is added to a uint32 digit sum in
// registers. The epilogue reduces mod p and stores int32 C. Exactness of
// digit d per block is the planner's Eq. G (qg_plan.cpp); the k-block flush
// replaces the reference's per-product floor (word.hpp:28-30).
//
// K5 (mixed / right variant, gemm.hpp:285-325): plain exact DGEMM of residues
// by forward-packed words (every partial sum < Q^e < 2^53) with a fused REDQ
// epilogue (pack.hpp:124-137).
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <mutex>

#include "qg_kernels.h"
#include "qg_device.cuh"

namespace qgk {

constexpr int BM = 128, BN = 128;  // CTA tile
constexpr int WM = 64, WN = 32;    // warp tile
constexpr int WARPS_N = BN / WN;
constexpr int NT = (BM / WM) * (BN / WN) * 32;  // 256 threads
constexpr int MI = WM / 8, NI = WN / 8;
constexpr int B_ST = BN + 4;  // 132 words = 1056 B = 32 mod 128: conflict-free B fragments
constexpr int SMEM_BUDGET = 220 * 1024;
constexpr bool kDynamicDefault = false;  // tiled kernels: dynamic tile schedule by default

// Stage geometry for a stage depth of BK words. The A row stride is the
// smallest s >= BK with s = 4 or 12 (mod 16) words: rows g = 0..3 of a
// fragment then start 32 bytes apart modulo 128, so the A-fragment loads are
// conflict-free (BK = 28 and 4 need no padding at all).
template <int BK>
struct Geo {
  static constexpr int A_ST = (BK % 16 == 4 || BK % 16 == 12) ? BK : (BK % 16 < 4 ? BK - BK % 16 + 4 : (BK % 16 < 12 ? BK - BK % 16 + 12 : BK - BK % 16 + 20));
  static constexpr int A_TILE = BM * A_ST;
  static constexpr int B_TILE = BK * B_ST;
  static constexpr int STAGE = A_TILE + B_TILE;  // doubles
  static constexpr int STAGES_RAW = SMEM_BUDGET / (STAGE * 8);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
};

// Tiled-layout geometry (k_gemm_tiled): a stage is one dense 128 x BK block
// of A and one of B^T, each a single contiguous chunk in HBM. Fragment loads
// are conflict-free when BK = 4 or 12 (mod 16); BK in {4, 12, 20, 28, 36}.
template <int BK, int RESERVE = 0>
struct GeoT {
  static constexpr int A_TILE = BM * BK;
  static constexpr int STAGE = 2 * BM * BK;  // doubles
  static constexpr int BUDGET = 232448 - 1024 - RESERVE;  // RESERVE: epilogue staging (EPI_REPACK)
  static constexpr int STAGES_RAW = BUDGET / (STAGE * 8);
  static constexpr int STAGES = STAGES_RAW > 8 ? 8 : (STAGES_RAW < 2 ? 2 : STAGES_RAW);
  static constexpr size_t SMEM = size_t(STAGES) * STAGE * sizeof(double);
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// D = A * B (C = 0): the first k-step of a new k-block.
__device__ __forceinline__ void dmma_zc(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%4};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(0.0));
}

// One pipeline stage: A rows [m0, m0+BM) x words [k0, k0+BK), B words
// [k0, k0+BK) x cols [n0, n0+BN). Out-of-range elements are zero-filled by
// cp.async's src-size operand, so partial tiles contribute nothing.
template <int BK, int VEC>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* __restrict__ A,
                                           size_t lda, const double* __restrict__ B, size_t ldb,
                                           int m0, int n0, int k0, int M, int N, int K, int tid) {
  using G = Geo<BK>;
  constexpr int A_CPR = BK / VEC;
  constexpr int A_CH = BM * A_CPR;
#pragma unroll
  for (int c = tid; c < A_CH; c += NT) {
    const int r = c / A_CPR, kc = (c % A_CPR) * VEC;
    const int gm = m0 + r, gk = k0 + kc;
    int bytes = 0;
    if (gm < M) {
      const int rem = K - gk;
      bytes = rem >= VEC ? VEC * 8 : (rem > 0 ? rem * 8 : 0);
    }
    const double* src = bytes ? A + (size_t)gm * lda + gk : A;
    if (VEC == 2) cp_async16(sA + r * G::A_ST + kc, src, bytes);
    else cp_async8(sA + r * G::A_ST + kc, src, bytes);
  }
  constexpr int B_CPR = BN / VEC;
  constexpr int B_CH = BK * B_CPR;
#pragma unroll
  for (int c = tid; c < B_CH; c += NT) {
    const int r = c / B_CPR, nc = (c % B_CPR) * VEC;
    const int gk = k0 + r, gn = n0 + nc;
    int bytes = 0;
    if (gk < K) {
      const int rem = N - gn;
      bytes = rem >= VEC ? VEC * 8 : (rem > 0 ? rem * 8 : 0);
    }
    const double* src = bytes ? B + (size_t)gk * ldb + gn : B;
    if (VEC == 2) cp_async16(sB + r * B_ST + nc, src, bytes);
    else cp_async8(sB + r * B_ST + nc, src, bytes);
  }
}

// digit d of an accumulator: floor(acc / Q^d) mod Q. acc + 2^(td+52) rounded
// toward zero has ulp exactly Q^d (the planner keeps acc < 2^(td+52)), so
// its low mantissa bits hold floor(acc / Q^d) with no rounding.
// The flush's DADD as a volatile asm statement: ptxas keeps volatile asm in
// source order, so the DADDs of a flushing row group stay behind the other
// row groups' DMMAs of the same k-step (issued after them in the source)
// instead of being hoisted right behind the group's own DMMAs, where the warp
// would stall on their latency with DMMAs still to issue.
__device__ __forceinline__ double dadd_rz_ordered(double a, double b) {
  double r;
  asm volatile("add.rz.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}
__device__ __forceinline__ double dadd_rn_ordered(double a, double b) {
  double r;
  asm volatile("add.rn.f64 %0, %1, %2;" : "=d"(r) : "d"(a), "d"(b));
  return r;
}

__device__ __forceinline__ uint32_t block_digit(double acc, double anchor, uint32_t qmask) {
#ifdef QG_INT_DIGIT
  // integer-pipe variant: floor(acc / 2^td) from the IEEE fields; anchor's
  // exponent field is 1023 + td + 52, so its high word gives the shift base
  const int sh_base = (int)((unsigned)__double2hiint(anchor) >> 20) - 52 - 1023 + 1075;
  return digit_at(acc, sh_base, qmask);
#elif defined(QG_ORDERED_FLUSH)
  return (uint32_t)__double2loint(dadd_rz_ordered(acc, anchor)) & qmask;
#else
  return (uint32_t)__double2loint(__dadd_rz(acc, anchor)) & qmask;
#endif
}

// Balanced digits: S = sum D_s Q^s with |D_s| < Q/2, digit d
// = round(S / Q^d) mod Q (centered). anchor = 1.5*2^(td+52) + 2^(td+t-1):
// the round-to-nearest sum has ulp Q^d, its low mantissa bits are
// round(S/Q^d) + Q/2, so the result is D_d + Q/2 in [0, Q); the Q/2 biases
// are removed mod p in the epilogue (args.corr).
template <bool BAL>
__device__ __forceinline__ uint32_t block_digit_t(double acc, double anchor, uint32_t qmask) {
#ifdef QG_ORDERED_FLUSH
  if (BAL) return (uint32_t)__double2loint(dadd_rn_ordered(acc, anchor)) & qmask;
#else
  if (BAL) return (uint32_t)__double2loint(__dadd_rn(acc, anchor)) & qmask;
#endif
  return block_digit(acc, anchor, qmask);
}


// EPI_DIGIT: K4 epilogue (int32 C = digit sums mod p). EPI_REDQ: K5 fused
// REDQ of exact packed sums (pack.hpp:124-137). EPI_RAW: plain words.
// EPI_REPACK: K4 with ReduceAndCompress fused (pack.hpp:141-155): the residues
// of C go through a per-warp shared-memory tile and leave as forward-packed
// words of e adjacent columns (mul_common_repacked, gemm.hpp:275-280).
enum { EPI_DIGIT = 0, EPI_REDQ = 1, EPI_RAW = 2, EPI_REPACK = 3 };
// EPI_REPACK staging: one byte per residue (p < 256), one 64 x 32 tile per warp
constexpr int REPACK_SMEM = BM * BN;
template <int EPI>
constexpr int epi_reserve() { return EPI == EPI_REPACK ? REPACK_SMEM : 0; }

// ReduceAndCompress of one warp's residue tile: repack_warp_segment (qg_device.cuh).
__device__ __forceinline__ void repack_segment(const uint8_t* st, const GemmArgs& a, int r0, int c0, int lane) {
  static_assert(WM == 64 && WN == 32, "repack_warp_segment's tile");
  repack_warp_segment(st, a.cc, a.ldcc, a.M, a.N, a.e, a.t, r0, c0, lane);
}

// redq, pack.hpp:124-137, on an exact integer-valued word w < 2^53: every
// base-Q digit replaced by itself mod p.
__device__ __forceinline__ double redq_word(double w, int t, int e, const ModP& modp) {
  const uint64_t bits = __double2ull_rz(w);
  const uint64_t mask = (1ull << t) - 1;
  uint64_t r = 0;
  for (int s = 0; s < t * e; s += t) {
    const uint64_t digit = (bits >> s) & mask;
    // digits wider than 32 bits (one-digit words of large p) need the 64-bit reduction
    r |= (t > 31 ? digit % modp.p : (uint64_t)modp((uint32_t)digit)) << s;
  }
  return __ull2double_rn(r);
}

// In-place REDQ of a whole warp tile of exact words 0 <= w < 2^52 (t <= 31,
// t e <= 52). Each word lives as the raw bits of w + 2^52 (low 52 bits = w);
// for every digit offset o the digit x = (u >> o) mod Q leaves u as
// u -= (x - x mod p) << o, which replaces the digit by its residue without a
// borrow. The digit loop is outermost (uniform trip count) and the words are
// unrolled inside it, so the 2 MI NI independent chains interleave instead of
// running one latency-bound word at a time.
template <int NW>
__device__ __forceinline__ void redq_words_inplace(double* w, int t, int e, const ModP& modp) {
  const uint32_t qmask = (1u << t) - 1;
  uint64_t u[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) u[i] = (uint64_t)__double_as_longlong(w[i] + 4503599627370496.0);
  const int total = t * e;
  for (int o = 0; o < total; o += t) {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint32_t x = (uint32_t)(u[i] >> o) & qmask;
      const uint32_t q = __umulhi(x, modp.magic);
      const uint32_t r0 = x - q * modp.p;  // x mod p or x mod p + p
      const uint32_t r = min(r0, r0 - modp.p);
      u[i] -= (uint64_t)(x - r) << o;
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i) w[i] = __longlong_as_double((long long)u[i]) - 4503599627370496.0;
}

// The same in-place REDQ on balanced (signed) digits: w = sum_s D_s Q^s with
// |D_s| < Q/2. Adding OFF = sum_s (Q/2) Q^s makes every digit D_s + Q/2 an
// unsigned base-Q digit (no borrows), so the digits can be read as above;
// x + ybias is >= 0 and = D_s (mod p). Between k-blocks a digit becomes its
// centred residue (|r| <= p/2) offset by Q/2 and w = u - OFF - 2^52 keeps the
// signed form; FINAL replaces it by the canonical residue in [0, p) and drops
// the offset, giving exactly the unsigned REDQ words (pack.hpp:124-137).
template <int NW, bool FINAL>
__device__ __forceinline__ void redq_words_inplace_bal(double* w, int t, int e, const ModP& modp, double off2,
                                                       uint32_t ybias) {
  const uint32_t qmask = (1u << t) - 1, half = 1u << (t - 1), h = modp.p >> 1;
  uint64_t u[NW];
#pragma unroll
  for (int i = 0; i < NW; ++i) u[i] = (uint64_t)__double_as_longlong(w[i] + off2);
  const int total = t * e;
  for (int o = 0; o < total; o += t) {
#pragma unroll
    for (int i = 0; i < NW; ++i) {
      const uint32_t x = (uint32_t)(u[i] >> o) & qmask;
      const uint32_t y = x + ybias;
      const uint32_t r1 = y - __umulhi(y, modp.magic) * modp.p;
      const uint32_t r0 = min(r1, r1 - modp.p);  // D mod p in [0, p)
      const uint32_t nd = FINAL ? r0 : (r0 > h ? r0 - modp.p : r0) + half;
      u[i] -= (uint64_t)((long long)x - (long long)nd) << o;
    }
  }
#pragma unroll
  for (int i = 0; i < NW; ++i)
    w[i] = __longlong_as_double((long long)u[i]) - (FINAL ? 4503599627370496.0 : off2);
}

template <int BK, int VEC, int EPI, bool MULTI>
__global__ void __launch_bounds__(NT, 1) k_gemm_dmma(GemmArgs args) {
  using G = Geo<BK>;
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;

  double acc[MI][NI][2];
  uint32_t dsum[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        acc[mi][ni][h] = 0.0;
        dsum[mi][ni][h] = 0u;
      }

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < G::STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<BK, VEC>(smem + s * G::STAGE, smem + s * G::STAGE + G::A_TILE, args.a, args.lda,
                          args.b, args.ldb, m0, n0, s * BK, M, N, K, tid);
    cp_async_commit();
  }

  int kst = 0;
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<G::STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + G::STAGES - 1;
      if (nk < ktiles) {
        const int slot = nk % G::STAGES;
        load_stage<BK, VEC>(smem + slot * G::STAGE, smem + slot * G::STAGE + G::A_TILE, args.a,
                            args.lda, args.b, args.ldb, m0, n0, nk * BK, M, N, K, tid);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % G::STAGES) * G::STAGE;
    const double* sB = sA + G::A_TILE;
    const double* a_base = sA + (warp_m * WM + g) * G::A_ST + t;
    const double* b_base = sB + t * B_ST + warp_n * WN + g;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[MI], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = a_base[mi * 8 * G::A_ST + kk * 4];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = b_base[kk * 4 * B_ST + ni * 8];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    if (MULTI) {
      if (++kst == args.kb_stages) {  // end of a k-block: digit d out, accumulators reset
        kst = 0;
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              dsum[mi][ni][h] += block_digit(acc[mi][ni][h], args.anchor, args.qmask);
              acc[mi][ni][h] = 0.0;
            }
      }
    }
  }
  cp_async_wait<0>();

  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int row = m0 + warp_m * WM + mi * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int col = n0 + warp_n * WN + ni * 8 + 2 * t;
      if (EPI == EPI_DIGIT) {
        int32_t* dst = args.c + (size_t)row * args.ldc + col;
        uint32_t r[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          uint32_t v = block_digit(acc[mi][ni][h], args.anchor, args.qmask) + dsum[mi][ni][h];
          if (args.accumulate && col + h < N) v += (uint32_t)dst[h];
          r[h] = modp(v);
        }
        if (col + 1 < N && ((((uintptr_t)dst) & 7) == 0)) {
          *reinterpret_cast<int2*>(dst) = make_int2((int)r[0], (int)r[1]);
        } else {
          if (col < N) dst[0] = (int32_t)r[0];
          if (col + 1 < N) dst[1] = (int32_t)r[1];
        }
      } else {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          if (col + h >= N) continue;
          double w = acc[mi][ni][h];
          if (EPI == EPI_REDQ) w = redq_word(w, args.t, args.e, modp);  // redq, pack.hpp:124-137
          args.cc[(size_t)row * args.ldcc + col + h] = w;
        }
      }
    }
  }
}

// ------------------------------------------------------------------ v3
// Persistent, barrier-free variant of the same contraction. Shared-memory
// stages are filled by cp.async.bulk (the TMA engine's bulk-copy path, SASS
// UBLKCP): every warp issues ~BM/8 + BK/8 row copies of its share of each
// stage from single lanes and arms the stage's `full` mbarrier with the bytes
// it expects; consumers wait on `full`, compute, and arrive on `empty`. No
// __syncthreads in the main loop, no per-thread address arithmetic for the
// loads, and the next tile's first stages stream in during the current
// tile's epilogue. Tiles are walked in groups of 8 row panels so the CTAs
// resident at one time share their CA/CB panels in L2. Requires 16-byte row
// alignment (even leading dimensions, even K and N); the v2 kernel above
// covers every other shape.

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n QG_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra QG_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// Tile raster: groups of `group` tile rows, walked column by column, so the
// CTAs resident at one time share their A and B panels in L2.
__device__ __forceinline__ void tile_coords(int tile, int tiles_m, int tiles_n, int group, int& tm, int& tn) {
  const int GROUP = group > 0 ? group : 8;
  const int per_group = GROUP * tiles_n;
  const int gid = tile / per_group;
  const int first_m = gid * GROUP;
  const int gsz = (tiles_m - first_m) < GROUP ? (tiles_m - first_m) : GROUP;
  const int r = tile - gid * per_group;
  tm = first_m + r % gsz;
  tn = r / gsz;
}

// Per-output digit sums of finished k-blocks. PACK: two outputs share one
// register as 16-bit lanes (t <= 16); the caller reduces both lanes mod p
// every args.pack_period flushes, before a lane could reach 2^16. Saves the
// 32 registers the fused flush needs.
template <bool PACK>
struct DigitSums {
  uint32_t v[MI][NI][2];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) v[i][j][0] = v[i][j][1] = 0u;
  }
  __device__ __forceinline__ void add(int i, int j, uint32_t d0, uint32_t d1) {
    v[i][j][0] += d0;
    v[i][j][1] += d1;
  }
  __device__ __forceinline__ uint32_t get(int i, int j, int h) const { return v[i][j][h]; }
  __device__ __forceinline__ void reduce(const ModP&) {}
};
template <>
struct DigitSums<true> {
  uint32_t v[MI][NI];
  __device__ __forceinline__ void reset() {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) v[i][j] = 0u;
  }
  __device__ __forceinline__ void add(int i, int j, uint32_t d0, uint32_t d1) { v[i][j] += d0 + (d1 << 16); }
  __device__ __forceinline__ uint32_t get(int i, int j, int h) const { return h ? (v[i][j] >> 16) : (v[i][j] & 0xFFFFu); }
  __device__ __forceinline__ void reduce(const ModP& modp) {
#pragma unroll
    for (int i = 0; i < MI; ++i)
#pragma unroll
      for (int j = 0; j < NI; ++j) v[i][j] = modp(v[i][j] & 0xFFFFu) | (modp(v[i][j] >> 16) << 16);
  }
};

// Split flush (kb_stages == 1): the warp tile's MI accumulator rows form
// SG groups (row mi in group mi % SG); group q ends its k-blocks after k-step
// split_step(q) of every stage, group SG-1 at the stage end. Every row's blocks
// are then one stage long (shifted windows; any partition of k into pieces of
// <= the exact block is exact), the flush bursts are SG times smaller, and in
// the k-step where a group flushes its DMMAs issue first: its DADDs wait only
// for them while the other rows' DMMAs queue behind and keep the pipe busy.
template <int BK>
struct SplitFlush {
  static constexpr int KS = BK / 4;  // k-steps per stage
#ifndef QG_SPLIT_GROUPS
#define QG_SPLIT_GROUPS 4
#endif
  static constexpr int SG = KS < QG_SPLIT_GROUPS ? KS : QG_SPLIT_GROUPS;
  __host__ __device__ static constexpr int step(int q) { return ((q + 1) * KS) / SG - 1; }
  // group flushing after k-step kk, or -1
  __host__ __device__ static constexpr int group_at(int kk) {
    for (int q = 0; q < SG; ++q)
      if (step(q) == kk) return q;
    return -1;
  }
  // issue order of the rows in k-step kk: the flushing group's rows first
  __host__ __device__ static constexpr int row(int kk, int i) {
    const int q = group_at(kk);
    if (q < 0) return i;
    const int c = (MI - q + SG - 1) / SG;  // rows of group q
    if (i < c) return q + i * SG;
    int j = i - c;
    for (int mi = 0; mi < MI; ++mi)
      if (mi % SG != q && j-- == 0) return mi;
    return i;
  }
};

// Consumer side of k_gemm_bulk (TILED = false: padded row layout) and
// k_gemm_tiled (TILED = true: dense A and B^T blocks). MID = 0: k-blocks end
// on stage boundaries (every kb_stages stages). MID > 0 (kb_stages == 1 only):
// blocks end after k-step MID-1 of every stage, i.e. they straddle stages.
// MID < 0 (kb_stages == 1 only): blocks are stages and the flush is fused
// into the first k-step of the next stage.
template <int BK, int EPI, bool MULTI, int MID, bool TILED, bool PACK = false, bool SPLIT = false, bool BAL = false>
__device__ __forceinline__ void consume(const GemmArgs& args, double* smem, uint64_t* full, uint64_t* empty,
                                        int tiles_m, int tiles_n, int my_tiles, int ktiles, bool nomem,
                                        uint8_t* repack = nullptr, const volatile int* tile_of = nullptr) {
  using G = Geo<BK>;
  using GT = GeoT<BK, epi_reserve<EPI>()>;
  constexpr int S = TILED ? GT::STAGES : G::STAGES;
  constexpr int STAGE = TILED ? GT::STAGE : G::STAGE;
  constexpr int A_TILE = TILED ? GT::A_TILE : G::A_TILE;
  constexpr int AST = TILED ? BK : G::A_ST;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = args.M, N = args.N;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  double acc[MI][NI][2];
  DigitSums<PACK> ds;
  ds.reset();
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
  uint32_t slot = 0, phase = 0;
  int nflush = 0;
  if (warp >= 4 && args.skew_ns > 0) start_skew(args.skew_ns);  // desynchronise SMSP warp pairs
  // dynamic schedule (tile_of != nullptr): the producer claims tiles from a
  // global counter and posts each tile's index beside its first stage; a
  // negative index ends the loop
  const bool dyn = TILED && tile_of != nullptr && !nomem;
  for (int ts = 0;; ++ts) {
    int tile;
    if (dyn) {
      mbar_wait(full + slot, phase);  // the tile's first stage (and its index) has landed
      tile = tile_of[slot];
      if (tile < 0) break;
    } else {
      if (ts >= my_tiles) break;
      tile = blockIdx.x + ts * gridDim.x;
    }
    int tm, tn;
    tile_coords(tile, tiles_m, tiles_n, args.group, tm, tn);
    const int m0 = tm * BM, n0 = tn * BN;
    if (EPI != EPI_DIGIT && args.accumulate) {
      // continue from the words already in CC (a k-split host product: the
      // previous part's REDQ left every digit below p, so the in-place REDQ
      // block bound is the same as between blocks)
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int row = m0 + warp_m * WM + mi * 8 + g, col = n0 + warp_n * WN + ni * 8 + 2 * t + h;
            acc[mi][ni][h] = (row < M && col < N) ? args.cc[(size_t)row * args.ldcc + col] : 0.0;
          }
    }
    int kst = 0;
    for (int kt = 0; kt < ktiles; ++kt) {
      if (!nomem && !(dyn && kt == 0)) mbar_wait(full + slot, phase);
      const double* sA = smem + slot * STAGE;
      const double* sB = sA + A_TILE;
      const double* a_base = sA + (warp_m * WM + g) * AST + t;
      // B^T block (tiled): element (n, k) at n*BK + k; row block: (k, n) at k*B_ST + n
      const double* b_base = TILED ? sB + (warp_n * WN + g) * BK + t : sB + t * B_ST + warp_n * WN + g;
      if (!(args.debug & 2)) {  // debug bit 1: data delivery alone (no DMMA)
#pragma unroll
        for (int kk = 0; kk < BK / 4; ++kk) {
          double af[MI], bf[NI];
#pragma unroll
          for (int mi = 0; mi < MI; ++mi) af[mi] = a_base[mi * 8 * AST + kk * 4];
#pragma unroll
          for (int ni = 0; ni < NI; ++ni) bf[ni] = TILED ? b_base[ni * 8 * BK + kk * 4] : b_base[kk * 4 * B_ST + ni * 8];
#pragma unroll
          for (int mi0 = 0; mi0 < MI; ++mi0)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              const int mi = SPLIT ? SplitFlush<BK>::row(kk, mi0) : mi0;  // flushing rows first
              if (MULTI && MID < 0 && kk == 0) {
                // fused flush (one stage per block): the finished block's digit
                // d leaves each accumulator right before that accumulator's
                // first DMMA of the new block (C = 0), so the integer work of
                // the flush interleaves with DMMAs that keep the pipe busy
                ds.add(mi, ni, block_digit_t<BAL>(acc[mi][ni][0], args.anchor, args.qmask),
                       block_digit_t<BAL>(acc[mi][ni][1], args.anchor, args.qmask));
                dmma_zc(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
              } else {
                dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
              }
            }
          if (MULTI && SPLIT) {  // groups ending their blocks mid-stage (compile-time positions)
            const int q = SplitFlush<BK>::group_at(kk);
            if (q >= 0 && q < SplitFlush<BK>::SG - 1) {
              asm volatile("" ::: "memory");  // keep the next fragment loads below the flush (register pressure)
#pragma unroll
              for (int mi = 0; mi < MI; ++mi)
                if (mi % SplitFlush<BK>::SG == q)
#pragma unroll
                  for (int ni = 0; ni < NI; ++ni) {
                    ds.add(mi, ni, block_digit_t<BAL>(acc[mi][ni][0], args.anchor, args.qmask),
                           block_digit_t<BAL>(acc[mi][ni][1], args.anchor, args.qmask));
                    acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
                  }
            }
          } else if (MULTI && MID > 0 && kk == MID - 1) {  // compile-time position: no branch in the DMMA stream
            asm volatile("" ::: "memory");  // keep the next fragment loads below the flush (register pressure)
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < NI; ++ni) {
                ds.add(mi, ni, block_digit_t<BAL>(acc[mi][ni][0], args.anchor, args.qmask),
                       block_digit_t<BAL>(acc[mi][ni][1], args.anchor, args.qmask));
                acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
              }
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == S) {
        slot = 0;
        phase ^= 1;
      }
      if (MULTI && EPI == EPI_REDQ) {  // mixed variant: in-place REDQ between k-blocks
        if (++kst == args.kb_stages) {
          kst = 0;
          if (args.debug & 8) {
            // debug bit 3: timing without the in-place REDQ (wrong results)
          } else if (BAL) {
            redq_words_inplace_bal<MI * NI * 2, false>(&acc[0][0][0], args.t, args.e, modp, args.redq_off2,
                                                       args.redq_ybias);
          } else if (args.t <= 31 && args.t * args.e <= 52) {
            redq_words_inplace<MI * NI * 2>(&acc[0][0][0], args.t, args.e, modp);
          } else {
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < NI; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) acc[mi][ni][h] = redq_word(acc[mi][ni][h], args.t, args.e, modp);
          }
        }
      } else if (MULTI && (MID == 0 || SPLIT)) {  // (MID != 0 flushes inside the unrolled k-steps)
        if (SPLIT || ++kst == args.kb_stages) {  // SPLIT (kb_stages == 1): the last row group ends here
          kst = 0;
          ++nflush;
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
            if (!SPLIT || mi % SplitFlush<BK>::SG == SplitFlush<BK>::SG - 1)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
              ds.add(mi, ni, block_digit_t<BAL>(acc[mi][ni][0], args.anchor, args.qmask),
                     block_digit_t<BAL>(acc[mi][ni][1], args.anchor, args.qmask));
              acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
            }
        }
      } else if (MULTI) {
        ++nflush;
      }
      (void)kst;
      if (PACK && nflush >= args.pack_period) {  // keep both 16-bit lanes below 2^16
        ds.reduce(modp);
        nflush = 0;
      }
    }
    // epilogue of this tile (the producer is already filling the next tile's stages)
    if (EPI == EPI_REDQ) {  // redq, pack.hpp:124-137, on the whole warp tile
      if (BAL) {
        redq_words_inplace_bal<MI * NI * 2, true>(&acc[0][0][0], args.t, args.e, modp, args.redq_off2,
                                                  args.redq_ybias);
      } else if (args.t <= 31 && args.t * args.e <= 52) {
        redq_words_inplace<MI * NI * 2>(&acc[0][0][0], args.t, args.e, modp);
      } else {
#pragma unroll
        for (int mi = 0; mi < MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < NI; ++ni)
#pragma unroll
            for (int h = 0; h < 2; ++h) acc[mi][ni][h] = redq_word(acc[mi][ni][h], args.t, args.e, modp);
      }
    }
    if (EPI == EPI_REPACK) {  // residues -> this warp's byte tile -> packed words
      uint8_t* st = repack + warp * (WM * WN);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t x = block_digit_t<BAL>(acc[mi][ni][h], args.anchor, args.qmask) + ds.get(mi, ni, h) +
                               (BAL ? args.corr : 0u);
            const uint32_t r0 = x - __umulhi(x, modp.magic) * modp.p;
            r[h] = min(r0, r0 - modp.p);
          }
          *reinterpret_cast<uint16_t*>(st + (mi * 8 + g) * WN + ni * 8 + 2 * t) = (uint16_t)(r[0] | (r[1] << 8));
          acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
      __syncwarp();
      repack_segment(st, args, m0 + warp_m * WM, n0 + warp_n * WN, lane);
      __syncwarp();  // the next tile overwrites the staging tile
    }
    // interior tiles without accumulation (nearly all of them): no per-element
    // bounds or accumulate checks, one int2 store per accumulator pair
    const bool fast = EPI == EPI_DIGIT && !args.accumulate && m0 + BM <= M && n0 + BN <= N;
    if (EPI == EPI_DIGIT && fast) {
      int32_t* cbase = args.c + (size_t)(m0 + warp_m * WM + g) * args.ldc + n0 + warp_n * WN + 2 * t;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        int32_t* crow = cbase + (size_t)(mi * 8) * args.ldc;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t x = block_digit_t<BAL>(acc[mi][ni][h], args.anchor, args.qmask) + ds.get(mi, ni, h) +
                               (BAL ? args.corr : 0u);
            const uint32_t r0 = x - __umulhi(x, modp.magic) * modp.p;
            r[h] = min(r0, r0 - modp.p);
          }
          *reinterpret_cast<int2*>(crow + ni * 8) = make_int2((int)r[0], (int)r[1]);
          acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
        }
      }
    }
#pragma unroll
    for (int mi = 0; mi < MI && !(EPI == EPI_DIGIT && fast) && EPI != EPI_REPACK; ++mi) {
      const int row = m0 + warp_m * WM + mi * 8 + g;
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        const int col = n0 + warp_n * WN + ni * 8 + 2 * t;
        if (EPI == EPI_DIGIT) {
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h)
            r[h] = block_digit_t<BAL>(acc[mi][ni][h], args.anchor, args.qmask) + ds.get(mi, ni, h) + (BAL ? args.corr : 0u);
          if (row < M && col < N) {  // N even: col < N implies col + 1 < N
            int32_t* dst = args.c + (size_t)row * args.ldc + col;
            if (args.accumulate) {
              const int2 old = *reinterpret_cast<const int2*>(dst);
              r[0] += (uint32_t)old.x;
              r[1] += (uint32_t)old.y;
            }
            *reinterpret_cast<int2*>(dst) = make_int2((int)modp(r[0]), (int)modp(r[1]));
          }
        } else if (row < M) {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            if (col + h >= N) continue;
            args.cc[(size_t)row * args.ldcc + col + h] = acc[mi][ni][h];
          }
        }
        acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
      }
    }
    ds.reset();
    nflush = 0;
  }
}

template <int BK, int EPI, bool MULTI>
__global__ void __launch_bounds__(NT + 128, 1) k_gemm_bulk(GemmArgs args, int tiles_m, int tiles_n) {
  using G = Geo<BK>;
  constexpr int S = G::STAGES;
  constexpr int NWARPS = NT / 32;  // consumer warps 0..7; warpgroup 2 (warps 8..11) produces
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * G::STAGE);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int M = args.M, N = args.N, K = args.K;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  const int ktiles = (K + BK - 1) / BK;
  const int total_tiles = tiles_m * tiles_n;
  const int my_tiles = blockIdx.x < total_tiles ? (total_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool nomem = args.debug & 1;  // timing experiment: compute on stale smem

  if (warp >= NWARPS) {
    // ---------------- producer warpgroup: gives its registers to the consumers
    // (setmaxnreg); warp 8 fills stage after stage, ahead of the consumers.
    // Ragged edges: A rows >= M are skipped (they only feed output rows that are
    // never stored); words >= K are zero-filled.
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (nomem || warp != NWARPS) return;
    uint32_t slot = 0, phase = 0;
    for (int ts = 0; ts < my_tiles; ++ts) {
      int tm, tn;
      tile_coords(blockIdx.x + ts * gridDim.x, tiles_m, tiles_n, args.group, tm, tn);
      const int m0 = tm * BM, n0 = tn * BN;
      const int mrows = (M - m0) < BM ? (M - m0) : BM;
      const int ncols = (N - n0) < BN ? (N - n0) : BN;
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(empty + slot, phase ^ 1);
        const int k0 = kt * BK;
        const int kval = (K - k0) < BK ? (K - k0) : BK;
        double* sA = smem + slot * G::STAGE;
        double* sB = sA + G::A_TILE;
        if (kval < BK) {  // zero the k tail (generic stores, ordered before the async copies)
          for (int i = lane; i < BM * (BK - kval); i += 32) {
            const int r = i / (BK - kval), c = kval + i % (BK - kval);
            sA[r * G::A_ST + c] = 0.0;
          }
          for (int i = lane; i < (BK - kval) * BN; i += 32) sB[(kval + i / BN) * B_ST + i % BN] = 0.0;
          asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        }
        __syncwarp();
        if (lane == 0) mbar_arrive_expect_tx(full + slot, (uint32_t)(mrows * kval + kval * ncols) * 8u);
        __syncwarp();
        for (int r = lane; r < mrows; r += 32)
          bulk_g2s(sA + r * G::A_ST, args.a + (size_t)(m0 + r) * args.lda + k0, (uint32_t)kval * 8u, full + slot);
        for (int r = lane; r < kval; r += 32)
          bulk_g2s(sB + r * B_ST, args.b + (size_t)(k0 + r) * args.ldb + n0, (uint32_t)ncols * 8u, full + slot);
        if (++slot == S) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---------------- consumer warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  // With one stage per k-block every warp would flush at the same stage end and
  // the DMMA pipe would idle meanwhile; warps 4..7 (the second warp of every
  // SMSP) therefore cut their blocks in the middle of each stage instead. Any
  // partition of k into blocks of <= kb words is exact, so both are correct.
  if (MULTI && args.kb_stages == 1 && (warp >= 4) && BK / 8 >= 1)
    consume<BK, EPI, MULTI, (BK / 8 >= 1 ? BK / 8 : 1), false>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem);
  else
    consume<BK, EPI, MULTI, 0, false>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem);
}

// ------------------------------------------------------------------ v4 (tiled)
// The contraction on the tiled packed layout written by qg_pack_*_tiled:
//   CA_t[tm][kt] = rows 128*tm.. x words BK*kt.. of CA      (128 x BK, dense)
//   CB_t[tn][kt] = cols 128*tn.. x words BK*kt.. of CB^T    (128 x BK, dense)
// zero padded at pack time, so a stage is exactly two cp.async.bulk copies of
// 128*BK*8 bytes (28 KiB at BK = 28) and there is no ragged-edge handling
// left in the kernel. Same warpgroup split and consumers as k_gemm_bulk.
template <int BK, int EPI, bool MULTI, int FLUSH, bool BAL>
__global__ void __launch_bounds__(NT + 128, 1) k_gemm_tiled(GemmArgs args, int tiles_m, int tiles_n) {
  using GT = GeoT<BK, epi_reserve<EPI>()>;
  constexpr int S = GT::STAGES;
  constexpr int NWARPS = NT / 32;
  constexpr uint32_t CHUNK = BM * BK * 8;  // bytes of one operand block
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * GT::STAGE);
  uint64_t* empty = full + S;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, NWARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  const int ktiles = (args.K + BK - 1) / BK;
  const int total_tiles = tiles_m * tiles_n;
  const int my_tiles = blockIdx.x < total_tiles ? (total_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  const bool nomem = args.debug & 1;

  // dynamic tile schedule (args.tile_counter): index of the tile whose first
  // stage sits in each ring slot, written by the producer before it arms the
  // slot's `full` barrier (whose completion orders it for the consumers)
  volatile int* tile_of = reinterpret_cast<volatile int*>(empty + S);
  const bool dyn = args.tile_counter != nullptr && !nomem;
  uint8_t* repack = reinterpret_cast<uint8_t*>(empty + S + 4);  // EPI_REPACK staging (after barriers + tile_of)

  if (warp >= NWARPS) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 40;\n" ::: "memory");
    if (nomem || warp != NWARPS || lane != 0) return;
    uint32_t slot = 0, phase = 0;
    for (int ts = 0;; ++ts) {
      // static: every gridDim.x-th tile; dynamic: claimed from the counter, so
      // a CTA that starts late (SMs held by another kernel, e.g. an NCCL
      // all-gather) simply takes fewer tiles
      const int tile = dyn ? atomicAdd(args.tile_counter, 1) : blockIdx.x + ts * gridDim.x;
      if (tile >= total_tiles) {
        if (dyn) {  // post the end marker in the next slot
          mbar_wait(empty + slot, phase ^ 1);
          tile_of[slot] = -1;
          mbar_arrive(full + slot);
        }
        break;
      }
      int tm, tn;
      tile_coords(tile, tiles_m, tiles_n, args.group, tm, tn);
      const double* ablk = args.a + (size_t)tm * ktiles * BM * BK;
      const double* bblk = args.b + (size_t)tn * ktiles * BM * BK;
      for (int kt = 0; kt < ktiles; ++kt) {
        mbar_wait(empty + slot, phase ^ 1);
        double* sA = smem + slot * GT::STAGE;
        if (dyn && kt == 0) tile_of[slot] = tile;
        mbar_arrive_expect_tx(full + slot, 2 * CHUNK);
        bulk_g2s(sA, ablk + (size_t)kt * BM * BK, CHUNK, full + slot);
        bulk_g2s(sA + GT::A_TILE, bblk + (size_t)kt * BM * BK, CHUNK, full + slot);
        if (++slot == S) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }
  asm volatile("setmaxnreg.inc.sync.aligned.u32 232;\n" ::: "memory");
  // FLUSH (multi-block): 0 = at stage ends; for kb_stages == 1 also
  // 1 = staggered (warps 4..7 cut mid-stage; two inlined consumer bodies, so
  // instantiated separately) and 2 = fused into the next stage's first k-step.
  if (FLUSH == 3)  // split phases: odd accumulator rows flush mid-stage, even rows at stage ends
    consume<BK, EPI, MULTI, (BK / 8 >= 1 ? BK / 8 : 1), true, false, true, BAL>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem, repack, dyn ? tile_of : nullptr);
  else if (FLUSH == 2)  // fused flush with packed digit sums (t <= 16)
    consume<BK, EPI, MULTI, -1, true, true, false, BAL>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem, repack, dyn ? tile_of : nullptr);
  else if (FLUSH == 1 && warp >= 4)
    consume<BK, EPI, MULTI, (BK / 8 >= 1 ? BK / 8 : 1), true, true, false, BAL>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem, repack, dyn ? tile_of : nullptr);
  else if (FLUSH == 1)
    consume<BK, EPI, MULTI, 0, true, true, false, BAL>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem, repack, dyn ? tile_of : nullptr);
  else
    consume<BK, EPI, MULTI, 0, true, false, false, BAL>(args, smem, full, empty, tiles_m, tiles_n, my_tiles, ktiles, nomem, repack, dyn ? tile_of : nullptr);
}

// Reference-semantics contraction (DoubleWord::high_part, word.hpp:28-30):
// acc[i][j] = sum_g trunc((CA[i][g] 2^-td) CB[g][j]) — the scale is a power
// of two, so this rounds exactly like the reference's (a*b)*inv_qd. FP64
// vector pipe (3 ops per term). Optional k-blocking with per-block digit
// extraction for plans whose blocks the DMMA path cannot make exact.
constexpr int HB = 64, HBK = 16, HT = 256;
__global__ void __launch_bounds__(HT) k_dot_highpart(HighArgs args) {
  __shared__ double sA[HB][HBK + 1];
  __shared__ double sB[HBK][HB + 2];
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  const int m0 = blockIdx.y * HB, n0 = blockIdx.x * HB;
  double acc[4][4];
  uint32_t ds[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      acc[i][j] = 0.0;
      ds[i][j] = 0u;
    }
  int cnt = args.kb_words;
  for (int k0 = 0; k0 < args.K; k0 += HBK) {
    for (int q = tid; q < HB * HBK; q += HT) {
      const int r = q / HBK, c = q % HBK;
      const int gm = m0 + r, gk = k0 + c;
      sA[r][c] = (gm < args.M && gk < args.K) ? args.ca[(size_t)gm * args.ldca + gk] * args.inv_qd : 0.0;
    }
    for (int q = tid; q < HB * HBK; q += HT) {
      const int r = q / HB, c = q % HB;
      const int gk = k0 + r, gn = n0 + c;
      sB[r][c] = (gk < args.K && gn < args.N) ? args.cb[(size_t)gk * args.ldcb + gn] : 0.0;
    }
    __syncthreads();
    const int kend = (args.K - k0) < HBK ? (args.K - k0) : HBK;
    for (int kk = 0; kk < kend; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = sA[ty + 16 * i][kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = sB[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] += trunc(__dmul_rn(a[i], b[j]));
      if (args.kb_words > 0 && --cnt == 0) {
        cnt = args.kb_words;
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            ds[i][j] += (uint32_t)(__double2ull_rz(acc[i][j]) & args.qmask);
            acc[i][j] = 0.0;
          }
      }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int row = m0 + ty + 16 * i;
    if (row >= args.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int col = n0 + tx + 16 * j;
      if (col >= args.N) continue;
      if (args.acc) args.acc[(size_t)row * args.N + col] = acc[i][j];
      if (args.c) {
        const uint32_t v = ds[i][j] + (uint32_t)(__double2ull_rz(acc[i][j]) & args.qmask);
        args.c[(size_t)row * args.ldc + col] = (int32_t)(v % args.p);
      }
    }
  }
}

// ---------------------------------------------------------------- launchers
// QG_FORCE_CPASYNC=1 forces the v2 (cp.async + __syncthreads) kernels.
static bool getenv_flag() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("QG_FORCE_CPASYNC");
    v = (e && e[0] == '1') ? 1 : 0;
  }
  return v == 1;
}

template <int BK, int VEC, int EPI, bool MULTI>
static cudaError_t launch_one(const GemmArgs& a, cudaStream_t s) {
  using G = Geo<BK>;
  auto k = k_gemm_dmma<BK, VEC, EPI, MULTI>;
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)G::SMEM);
  if (err) return err;
  const dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  k<<<grid, NT, G::SMEM, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <int VEC>
static cudaError_t launch_digit(const GemmArgs& a, int bk, cudaStream_t s) {
  if (a.kb_stages == 0) return launch_one<32, VEC, EPI_DIGIT, false>(a, s);
  switch (bk) {
    case 32: return launch_one<32, VEC, EPI_DIGIT, true>(a, s);
    case 28: return launch_one<28, VEC, EPI_DIGIT, true>(a, s);
    case 24: return launch_one<24, VEC, EPI_DIGIT, true>(a, s);
    case 16: return launch_one<16, VEC, EPI_DIGIT, true>(a, s);
    case 8: return launch_one<8, VEC, EPI_DIGIT, true>(a, s);
    case 4: return launch_one<4, VEC, EPI_DIGIT, true>(a, s);
  }
  return cudaErrorInvalidValue;
}

static int num_sms() {
  static int n = 0;
  if (n == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) n = 148;
  }
  return n;
}

template <int BK, int EPI, bool MULTI>
static cudaError_t launch_bulk(const GemmArgs& a, cudaStream_t s) {
  using G = Geo<BK>;
  auto k = k_gemm_bulk<BK, EPI, MULTI>;
  const size_t smem = G::SMEM + 2 * G::STAGES * sizeof(uint64_t);
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int tiles = tiles_m * tiles_n;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  GemmArgs a2 = a;
  const char* dbg = getenv("QG_DEBUG_MODE");
  a2.debug = dbg ? atoi(dbg) : 0;
  // warps 4..7 start 3 us late (a clock spin) so the two warps of an SMSP do not flush their
  // k-blocks at the same moment (+3% on config 2, profiles/r01_notes.md)
  const char* skew = getenv("QG_SKEW_NS");
  a2.skew_ns = skew ? (unsigned)atoi(skew) : (a.kb_stages ? 4000u : 0u);
  k<<<grid, NT + 128, smem, s>>>(a2, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

static cudaError_t launch_digit_bulk(const GemmArgs& a, int bk, cudaStream_t s) {
  if (a.kb_stages == 0) {
    const char* e = getenv("QG_SINGLE_BK");  // experiments: stage depth of single-block runs
    if (e && atoi(e) == 16) return launch_bulk<16, EPI_DIGIT, false>(a, s);
    return launch_bulk<32, EPI_DIGIT, false>(a, s);
  }
  switch (bk) {
    case 32: return launch_bulk<32, EPI_DIGIT, true>(a, s);
    case 28: return launch_bulk<28, EPI_DIGIT, true>(a, s);
    case 24: return launch_bulk<24, EPI_DIGIT, true>(a, s);
    case 16: return launch_bulk<16, EPI_DIGIT, true>(a, s);
    case 8: return launch_bulk<8, EPI_DIGIT, true>(a, s);
    case 4: return launch_bulk<4, EPI_DIGIT, true>(a, s);
  }
  return cudaErrorInvalidValue;
}

static int num_sms();
// A zeroed tile counter for one launch of the dynamically scheduled tiled
// kernel: a slot of a per-device pool (4096 launches in flight at most),
// cleared by a memset on the launch's stream (a graph node when captured).
static int* tile_counter(cudaStream_t s) {
  static std::mutex mu;
  static std::map<int, int*> pools;
  static std::atomic<unsigned> next{0};
  constexpr unsigned kSlots = 4096;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  int* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(mu);
    int*& p = pools[dev];
    if (!p && cudaMalloc(&p, kSlots * sizeof(int)) != cudaSuccess) p = nullptr;
    base = p;
  }
  if (!base) return nullptr;
  int* c = base + (next.fetch_add(1) % kSlots);
  return cudaMemsetAsync(c, 0, sizeof(int), s) == cudaSuccess ? c : nullptr;
}

// Dynamic tile schedule for the tiled kernels: QG_DYN=0/1 (experiments),
// default from qg_set_dynamic_tiles.
static std::atomic<int> g_dynamic_tiles{-1};
void set_dynamic_tiles(int enable) { g_dynamic_tiles.store(enable ? 1 : 0); }
static bool dynamic_tiles() {
  if (const char* e = getenv("QG_DYN")) return e[0] != '0';
  const int v = g_dynamic_tiles.load();
  return v < 0 ? kDynamicDefault : v != 0;
}

template <int BK, int EPI, bool MULTI, int FLUSH, bool BAL>
static cudaError_t launch_tiled_one(const GemmArgs& a, cudaStream_t s) {
  using GT = GeoT<BK, epi_reserve<EPI>()>;
  auto k = k_gemm_tiled<BK, EPI, MULTI, FLUSH, BAL>;
  const size_t smem = GT::SMEM + (2 * GT::STAGES + 4) * sizeof(uint64_t) + epi_reserve<EPI>();
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int tiles = tiles_m * tiles_n;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  GemmArgs a2 = a;
  const char* dbg = getenv("QG_DEBUG_MODE");
  a2.debug = dbg ? atoi(dbg) : 0;
  // warps 4..7 start 3 us late (a clock spin) so the two warps of an SMSP do not flush their
  // k-blocks (or run their tile epilogues) at the same moment: config 2
  // +3 %, config 3 75.6 -> 78.9 % (profiles/r01_notes.md)
  const char* skew = getenv("QG_SKEW_NS");
  a2.skew_ns = skew ? (unsigned)atoi(skew) : 3000u;
  if (const char* sl = getenv("QG_SKEW_SLEEP"))
    if (sl[0] == '1' && a2.skew_ns) a2.skew_ns |= 0x80000000u;  // experiments: nanosleep instead of the clock spin
  const char* grp = getenv("QG_GROUP");  // experiments: tile-row group of the raster
  a2.group = grp ? atoi(grp) : 8;
  a2.tile_counter = nullptr;
  if (dynamic_tiles() && !(a2.debug & 1)) {
    a2.tile_counter = tile_counter(s);
    if (!a2.tile_counter) return cudaErrorMemoryAllocation;
  }
  if (BAL) {  // remove the Q/2 bias of every digit extraction (mod p)
    const unsigned long long ktiles = (unsigned long long)((a.K + BK - 1) / BK);
    const unsigned long long nb = !MULTI ? 1ull : (FLUSH == 0 ? ktiles / a.kb_stages + 1 : ktiles + 1);
    const unsigned long long halfq = ((unsigned long long)a.qmask + 1) / 2;
    a2.corr = (uint32_t)((a.p - (nb % a.p) * (halfq % a.p) % a.p) % a.p);
  }
  k<<<grid, NT + 128, smem, s>>>(a2, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

template <int BK, bool BAL>
static cudaError_t launch_tiled_bk(const GemmArgs& a, int flush, cudaStream_t s) {
  const char* dbg = getenv("QG_DEBUG_MODE");  // bit 2: time without flushes (wrong digits)
  if (a.kb_stages == 0 || (dbg && (atoi(dbg) & 4))) return launch_tiled_one<BK, EPI_DIGIT, false, 0, BAL>(a, s);
  if (a.kb_stages == 1 && flush == 3 && BK >= 8) return launch_tiled_one<BK, EPI_DIGIT, true, (BK >= 8 ? 3 : 0), BAL>(a, s);
  if (!BAL && a.kb_stages == 1 && flush == 2 && a.pack_period >= 1) return launch_tiled_one<BK, EPI_DIGIT, true, 2, false>(a, s);
  if (!BAL && a.kb_stages == 1 && flush == 1 && BK >= 8 && a.pack_period >= 1)
    return launch_tiled_one<BK, EPI_DIGIT, true, (BK >= 8 ? 1 : 0), false>(a, s);
  return launch_tiled_one<BK, EPI_DIGIT, true, 0, BAL>(a, s);
}

template <int BK>
static cudaError_t launch_tiled_b(const GemmArgs& a, int flush, cudaStream_t s) {
  return a.balanced ? launch_tiled_bk<BK, true>(a, flush, s) : launch_tiled_bk<BK, false>(a, flush, s);
}

cudaError_t launch_dot_tiled(const GemmArgs& a, int bk, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (a.anchored_kb > 0) {  // K4A (qg_anchor.cu)
    int* counter = nullptr;
    if (dynamic_tiles()) {
      counter = tile_counter(s);
      if (!counter) return cudaErrorMemoryAllocation;
    }
    return launch_dot_anchor(a, a.anchored_kb, counter, s, variant);
  }
  static thread_local char name[80];
  // k-block flush placement for one-stage blocks: 3 = split phases (default:
  // odd accumulator rows mid-stage, even rows at stage ends), 0 = stage ends,
  // 1 = staggered warps, 2 = fused into the next stage's first k-step
  const char* e = getenv("QG_FLUSH");
  const int flush = e ? atoi(e) : 3;
  static const char* kFlush[] = {"", "_stagger", "_fused", "_split"};
  const bool named = a.kb_stages == 1 && flush >= 1 && flush <= 3 && (flush == 3 || !a.balanced);
  snprintf(name, sizeof name, "dot_tiled_bk%d_%s%s%s", bk, a.kb_stages ? "multiblock" : "singleblock",
           named ? kFlush[flush] : "", a.balanced ? "_balanced" : "");
  *variant = name;
  switch (bk) {
    case 52: return launch_tiled_b<52>(a, flush, s);
    case 44: return launch_tiled_b<44>(a, flush, s);
    case 36: return launch_tiled_b<36>(a, flush, s);
    case 28: return launch_tiled_b<28>(a, flush, s);
    case 20: return launch_tiled_b<20>(a, flush, s);
    case 12: return launch_tiled_b<12>(a, flush, s);
    case 4: return launch_tiled_b<4>(a, flush, s);
  }
  return cudaErrorInvalidValue;
}

// K4 with the fused ReduceAndCompress epilogue (EPI_REPACK): CC = m x ceil(n/e)
// words in a.cc (a.ldcc), a.t / a.e the packing of the output rows.
template <int BK, bool BAL>
static cudaError_t launch_tiled_repack_bk(const GemmArgs& a, int flush, cudaStream_t s) {
  if (a.kb_stages == 0) return launch_tiled_one<BK, EPI_REPACK, false, 0, BAL>(a, s);
  if (a.kb_stages == 1 && flush == 3 && BK >= 8) return launch_tiled_one<BK, EPI_REPACK, true, (BK >= 8 ? 3 : 0), BAL>(a, s);
  return launch_tiled_one<BK, EPI_REPACK, true, 0, BAL>(a, s);
}

template <int BK>
static cudaError_t launch_tiled_repack_b(const GemmArgs& a, int flush, cudaStream_t s) {
  return a.balanced ? launch_tiled_repack_bk<BK, true>(a, flush, s) : launch_tiled_repack_bk<BK, false>(a, flush, s);
}

cudaError_t launch_dot_tiled_repack(const GemmArgs& a, int bk, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (a.anchored_kb > 0) {  // K4A with the ReduceAndCompress epilogue (qg_anchor.cu)
    int* counter = nullptr;
    if (dynamic_tiles()) {
      counter = tile_counter(s);
      if (!counter) return cudaErrorMemoryAllocation;
    }
    return launch_dot_anchor(a, a.anchored_kb, counter, s, variant, true);
  }
  static thread_local char name[80];
  const char* e = getenv("QG_FLUSH");
  const int flush = e ? (atoi(e) == 3 ? 3 : 0) : 3;
  snprintf(name, sizeof name, "dot_tiled_repack_bk%d_%s%s%s", bk, a.kb_stages ? "multiblock" : "singleblock",
           a.kb_stages == 1 && flush == 3 ? "_split" : "", a.balanced ? "_balanced" : "");
  *variant = name;
  switch (bk) {
    case 52: return launch_tiled_repack_b<52>(a, flush, s);
    case 44: return launch_tiled_repack_b<44>(a, flush, s);
    case 36: return launch_tiled_repack_b<36>(a, flush, s);
    case 28: return launch_tiled_repack_b<28>(a, flush, s);
    case 20: return launch_tiled_repack_b<20>(a, flush, s);
    case 12: return launch_tiled_repack_b<12>(a, flush, s);
    case 4: return launch_tiled_repack_b<4>(a, flush, s);
  }
  return cudaErrorInvalidValue;
}

template <int BK>
static cudaError_t launch_right_tiled_bk(const GemmArgs& a, bool redq, cudaStream_t s) {
  if (!redq) return launch_tiled_one<BK, EPI_RAW, false, 0, false>(a, s);
  if (a.balanced)
    return a.kb_stages ? launch_tiled_one<BK, EPI_REDQ, true, 0, true>(a, s)
                       : launch_tiled_one<BK, EPI_REDQ, false, 0, true>(a, s);
  if (a.kb_stages) return launch_tiled_one<BK, EPI_REDQ, true, 0, false>(a, s);
  return launch_tiled_one<BK, EPI_REDQ, false, 0, false>(a, s);
}

cudaError_t launch_right_tiled(const GemmArgs& a, int bk, bool redq, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  static thread_local char name[64];
  snprintf(name, sizeof name, "right_tiled_bk%d_%s%s%s", bk, redq ? "redq" : "raw", a.kb_stages ? "_blocked" : "",
           a.balanced ? "_balanced" : "");
  *variant = name;
  switch (bk) {
    case 36: return launch_right_tiled_bk<36>(a, redq, s);
    case 28: return launch_right_tiled_bk<28>(a, redq, s);
    case 20: return launch_right_tiled_bk<20>(a, redq, s);
    case 12: return launch_right_tiled_bk<12>(a, redq, s);
    case 4: return launch_right_tiled_bk<4>(a, redq, s);
  }
  return cudaErrorInvalidValue;
}

static bool vec2_ok(const GemmArgs& a) {
  return (a.lda % 2 == 0) && (a.ldb % 2 == 0) && ((((uintptr_t)a.a) & 15) == 0) &&
         ((((uintptr_t)a.b) & 15) == 0);
}

// The bulk-copy kernel moves whole 16-byte multiples: rows must start
// 16-byte aligned and every partial row (K tail, N tail) must be even.
static bool bulk_ok(const GemmArgs& a, bool digit_out) {
  return vec2_ok(a) && (a.K % 2 == 0) && (a.N % 2 == 0) &&
         (!digit_out || ((a.ldc % 2 == 0) && ((((uintptr_t)a.c) & 7) == 0))) && !getenv_flag();
}

cudaError_t launch_dot_dmma(const GemmArgs& a, int bk, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  static thread_local char name[64];
  const bool v2 = vec2_ok(a);
  const bool bulk = bulk_ok(a, true);
  snprintf(name, sizeof name, "dot_%s_bk%d_%s", bulk ? "bulk" : (v2 ? "cpasync16" : "cpasync8"),
           a.kb_stages ? bk : 32, a.kb_stages ? "multiblock" : "singleblock");
  *variant = name;
  if (bulk) return launch_digit_bulk(a, bk, s);
  return v2 ? launch_digit<2>(a, bk, s) : launch_digit<1>(a, bk, s);
}

cudaError_t launch_right_dmma(const GemmArgs& a, bool redq, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  const bool v2 = vec2_ok(a);
  const bool bulk = bulk_ok(a, false);
  if (bulk) {
    *variant = redq ? "right_bulk_redq" : "right_bulk_raw";
    return redq ? launch_bulk<32, EPI_REDQ, false>(a, s) : launch_bulk<32, EPI_RAW, false>(a, s);
  }
  *variant = redq ? (v2 ? "right_cpasync16_redq" : "right_cpasync8_redq") : (v2 ? "right_cpasync16_raw" : "right_cpasync8_raw");
  if (redq) return v2 ? launch_one<32, 2, EPI_REDQ, false>(a, s) : launch_one<32, 1, EPI_REDQ, false>(a, s);
  return v2 ? launch_one<32, 2, EPI_RAW, false>(a, s) : launch_one<32, 1, EPI_RAW, false>(a, s);
}

cudaError_t launch_dot_highpart(const HighArgs& a, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  const dim3 grid((a.N + HB - 1) / HB, (a.M + HB - 1) / HB);
  k_dot_highpart<<<grid, HT, 0, s>>>(a);
  *variant = "dot_highpart";
  count_launch();
  return cudaGetLastError();
}

}  // namespace qgk
