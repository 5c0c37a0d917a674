// qg_dot.cu — the packed contractions on the FP64 tensor cores of sm_100a.
//
// sm_100a has no FP64 kind for tcgen05.mma (ptxas rejects .kind::f64), so the
// FP64 tensor path is the warp-level mma.sync.m8n8k4.f64, which ptxas lowers
// to SASS DMMA.8x8x4 (37.1 TFLOP/s measured on B200, profiles/r01_*). The
// operands are staged global -> shared by cp.async (LDGSTS) in a 4-stage
// ring and fed to DMMA from shared memory; each warp owns a 32x32 tile of
// the 128x128 CTA tile (16 DMMAs per 4-word k-step).
//
// K4 (common / dot-product variant, gemm.hpp:210-271 + 450-489): the FP64
// accumulator holds sum_g CA[i][g] CB[g][j] over one k-block; at the end of
// every block its base-Q digit d is read straight from the IEEE bits
// (digit_at) and added to an integer digit sum kept in shared memory; the
// epilogue reduces mod p and stores int32 C. Exactness of digit d per block
// is the planner's Eq. G (qg_plan.cpp); the k-block flush replaces the
// reference's per-product floor (word.hpp:28-30).
//
// K5 (mixed / right variant, gemm.hpp:285-325): plain exact DGEMM of residues
// by forward-packed words (every partial sum < Q^e < 2^53) with a fused REDQ
// epilogue (pack.hpp:124-137).
#include "qg_kernels.h"
#include "qg_device.cuh"

namespace qgk {

constexpr int BM = 128, BN = 128, BK = 16;  // CTA tile; BK in words
constexpr int WM = 32, WN = 32;             // warp tile
constexpr int WARPS_N = BN / WN;
constexpr int NWARPS = (BM / WM) * (BN / WN);
constexpr int NT = NWARPS * 32;  // 512 threads
constexpr int MI = WM / 8, NI = WN / 8;
constexpr int NACC = MI * NI * 2;  // accumulators per thread
constexpr int A_ST = BK + 4;       // padded smem row strides (conflict-free fragments)
constexpr int B_ST = BN + 4;
constexpr int A_TILE = BM * A_ST;
constexpr int B_TILE = BK * B_ST;
constexpr int STAGE_DBL = A_TILE + B_TILE;
constexpr int STAGES = 4;
constexpr size_t SMEM_PIPE = size_t(STAGES) * STAGE_DBL * sizeof(double);
constexpr size_t SMEM_DIGITS = size_t(NACC) * NT * sizeof(uint32_t);

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

// One pipeline stage: A rows [m0, m0+BM) x words [k0, k0+BK), B words
// [k0, k0+BK) x cols [n0, n0+BN). Out-of-range elements are zero-filled by
// cp.async's src-size operand, so partial tiles contribute nothing.
template <int VEC>
__device__ __forceinline__ void load_stage(double* sA, double* sB, const double* __restrict__ A,
                                           size_t lda, const double* __restrict__ B, size_t ldb,
                                           int m0, int n0, int k0, int M, int N, int K, int tid) {
  constexpr int A_CPR = BK / VEC;  // chunks per A row
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
    if (VEC == 2) cp_async16(sA + r * A_ST + kc, src, bytes);
    else cp_async8(sA + r * A_ST + kc, src, bytes);
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

// Common variant, K4. MULTI: more than one k-block (digit sums in smem).
template <int VEC, bool MULTI>
__global__ void __launch_bounds__(NT, 1) k_dot_dmma(DotArgs args) {
  extern __shared__ __align__(128) double smem[];
  uint32_t* dsum = reinterpret_cast<uint32_t*>(smem + STAGES * STAGE_DBL);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;

  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;
  if (MULTI) {
#pragma unroll
    for (int q = 0; q < NACC; ++q) dsum[q * NT + tid] = 0u;
  }
  int cnt = args.kb_steps;

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<VEC>(smem + s * STAGE_DBL, smem + s * STAGE_DBL + A_TILE, args.ca, args.ldca,
                      args.cb, args.ldcb, m0, n0, s * BK, M, N, K, tid);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        const int slot = nk % STAGES;
        load_stage<VEC>(smem + slot * STAGE_DBL, smem + slot * STAGE_DBL + A_TILE, args.ca,
                        args.ldca, args.cb, args.ldcb, m0, n0, nk * BK, M, N, K, tid);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % STAGES) * STAGE_DBL;
    const double* sB = sA + A_TILE;
    const double* a_base = sA + (warp_m * WM + g) * A_ST + t;
    const double* b_base = sB + t * B_ST + warp_n * WN + g;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[MI], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = a_base[mi * 8 * A_ST + kk * 4];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = b_base[kk * 4 * B_ST + ni * 8];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
      if (MULTI) {
        if (--cnt == 0) {  // end of a k-block: digit d out, accumulator reset
          cnt = args.kb_steps;
#pragma unroll
          for (int mi = 0; mi < MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < NI; ++ni)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int q = (mi * NI + ni) * 2 + h;
                uint32_t v = dsum[q * NT + tid] + digit_at(acc[mi][ni][h], args.sh_base, args.qmask);
                if (args.reduce_each) v %= args.p;
                dsum[q * NT + tid] = v;
                acc[mi][ni][h] = 0.0;
              }
        }
      }
    }
  }
  cp_async_wait<0>();

  // Epilogue: last (partial) block's digit + earlier blocks' digits, mod p.
  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int row = m0 + warp_m * WM + mi * 8 + g;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int col = n0 + warp_n * WN + ni * 8 + 2 * t;
      uint32_t r[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t v = digit_at(acc[mi][ni][h], args.sh_base, args.qmask);
        if (MULTI) {
          const int q = (mi * NI + ni) * 2 + h;
          v += args.reduce_each ? modp(dsum[q * NT + tid]) : dsum[q * NT + tid];
        }
        r[h] = modp(v);
      }
      if (row < M) {
        int32_t* dst = args.c + (size_t)row * args.ldc + col;
        if (col + 1 < N && ((((uintptr_t)dst) & 7) == 0)) {
          *reinterpret_cast<int2*>(dst) = make_int2((int)r[0], (int)r[1]);
        } else {
          if (col < N) dst[0] = (int32_t)r[0];
          if (col + 1 < N) dst[1] = (int32_t)r[1];
        }
      }
    }
  }
}

// Mixed variant, K5: exact DGEMM + fused REDQ (or raw words).
template <int VEC>
__global__ void __launch_bounds__(NT, 1) k_right_dmma(RightArgs args) {
  extern __shared__ __align__(128) double smem[];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int M = args.M, N = args.N, K = args.K;

  double acc[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

  const int ktiles = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles)
      load_stage<VEC>(smem + s * STAGE_DBL, smem + s * STAGE_DBL + A_TILE, args.a, args.lda,
                      args.cb, args.ldcb, m0, n0, s * BK, M, N, K, tid);
    cp_async_commit();
  }
  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      if (nk < ktiles) {
        const int slot = nk % STAGES;
        load_stage<VEC>(smem + slot * STAGE_DBL, smem + slot * STAGE_DBL + A_TILE, args.a,
                        args.lda, args.cb, args.ldcb, m0, n0, nk * BK, M, N, K, tid);
      }
      cp_async_commit();
    }
    const double* sA = smem + (kt % STAGES) * STAGE_DBL;
    const double* sB = sA + A_TILE;
    const double* a_base = sA + (warp_m * WM + g) * A_ST + t;
    const double* b_base = sB + t * B_ST + warp_n * WN + g;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[MI], bf[NI];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) af[mi] = a_base[mi * 8 * A_ST + kk * 4];
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) bf[ni] = b_base[kk * 4 * B_ST + ni * 8];
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
  }
  cp_async_wait<0>();

  const int tb = args.t * args.e;
  const uint64_t mask = (1ull << args.t) - 1;
  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
#pragma unroll
  for (int mi = 0; mi < MI; ++mi) {
    const int row = m0 + warp_m * WM + mi * 8 + g;
    if (row >= M) continue;
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      const int col = n0 + warp_n * WN + ni * 8 + 2 * t;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        if (col + h >= N) continue;
        double w = acc[mi][ni][h];
        if (args.redq) {  // redq, pack.hpp:124-137 (every partial sum exact, < Q^e)
          const uint64_t bits = __double2ull_rz(w);
          uint64_t r = 0;
          for (int s = 0; s < tb; s += args.t) r |= (uint64_t)modp((uint32_t)((bits >> s) & mask)) << s;
          w = __ull2double_rn(r);
        }
        args.cc[(size_t)row * args.ldcc + col + h] = w;
      }
    }
  }
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
template <typename Kern>
static cudaError_t prep(Kern k, size_t smem) {
  return cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

cudaError_t launch_dot_dmma(const DotArgs& a, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  const bool vec2 = (a.ldca % 2 == 0) && (a.ldcb % 2 == 0) && ((((uintptr_t)a.ca) & 15) == 0) &&
                    ((((uintptr_t)a.cb) & 15) == 0);
  const bool multi = a.kb_steps > 0;
  const dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  const size_t smem = SMEM_PIPE + (multi ? SMEM_DIGITS : 0);
  cudaError_t err;
  if (vec2 && multi) {
    err = prep(k_dot_dmma<2, true>, smem);
    if (err) return err;
    k_dot_dmma<2, true><<<grid, NT, smem, s>>>(a);
    *variant = "dot_dmma_v2_multiblock";
  } else if (vec2) {
    err = prep(k_dot_dmma<2, false>, smem);
    if (err) return err;
    k_dot_dmma<2, false><<<grid, NT, smem, s>>>(a);
    *variant = "dot_dmma_v2_singleblock";
  } else if (multi) {
    err = prep(k_dot_dmma<1, true>, smem);
    if (err) return err;
    k_dot_dmma<1, true><<<grid, NT, smem, s>>>(a);
    *variant = "dot_dmma_v1_multiblock";
  } else {
    err = prep(k_dot_dmma<1, false>, smem);
    if (err) return err;
    k_dot_dmma<1, false><<<grid, NT, smem, s>>>(a);
    *variant = "dot_dmma_v1_singleblock";
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_right_dmma(const RightArgs& a, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  const bool vec2 = (a.lda % 2 == 0) && (a.ldcb % 2 == 0) && ((((uintptr_t)a.a) & 15) == 0) &&
                    ((((uintptr_t)a.cb) & 15) == 0);
  const dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM);
  cudaError_t err;
  if (vec2) {
    err = prep(k_right_dmma<2>, SMEM_PIPE);
    if (err) return err;
    k_right_dmma<2><<<grid, NT, SMEM_PIPE, s>>>(a);
    *variant = "right_dmma_v2";
  } else {
    err = prep(k_right_dmma<1>, SMEM_PIPE);
    if (err) return err;
    k_right_dmma<1><<<grid, NT, SMEM_PIPE, s>>>(a);
    *variant = "right_dmma_v1";
  }
  count_launch();
  return cudaGetLastError();
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
