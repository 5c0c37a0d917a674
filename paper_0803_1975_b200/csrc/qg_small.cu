// qg_small.cu — the dot-product contraction for products too small to fill
// the 148 SMs with the main kernel's 128x128 tiles (BASELINE config 1: 512^3
// gives 16 such tiles, 11 % of the SMs).
//
// Same tiled packed operands as k_gemm_tiled (qg_pack.cu: CA_t / CB_t, dense
// 128 x BK blocks per stage), same exactness argument (Eq. G per k-block,
// DESIGN.md §3), but 64x64 output tiles — a 64-row half of a 128-row block is
// one contiguous 64 x BK chunk, so a stage is still two cp.async.bulk copies —
// and the k stages split over a thread-block cluster of S CTAs along grid z
// (any partition of k into pieces of <= the exact block is exact). Every CTA
// extracts digit d of its own k-blocks (one DADD per accumulator at a block
// end, qg_dot.cu); the cluster's leader sums the S partial digit sums through
// distributed shared memory, reduces mod p and stores int32 C
// (reduce_common_entry, gemm.hpp:247-250; blocked_accumulate's mod-p sum of
// k-blocks, gemm.hpp:484-486). No workspace, no atomics, one launch; config 1
// runs as 8 x 8 tiles x 2 splits = 128 CTAs.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstdlib>

#include "qg_device.cuh"
#include "qg_kernels.h"

namespace cg = cooperative_groups;

namespace qgk {

namespace {

constexpr int SM_BM = 64, SM_BN = 64;  // CTA tile
constexpr int SM_WM = 32, SM_WN = 16;  // warp tile (8 warps: 2 x 4)
constexpr int SM_MI = SM_WM / 8, SM_NI = SM_WN / 8;
constexpr int SM_NT = 256;

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void bar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void bar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("{\n .reg .b64 st;\n mbarrier.arrive.expect_tx.shared::cta.b64 st, [%0], %1;\n}\n" ::"r"(su32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n QG_SWAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra QG_SWAIT_%=;\n}\n" ::"r"(su32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   su32(dst)),
               "l"(src), "r"(bytes), "r"(su32(bar))
               : "memory");
}

__device__ __forceinline__ void dmma_s(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool BAL>
__device__ __forceinline__ uint32_t digit_of(double acc, double anchor, uint32_t qmask) {
  // Eq. G: the sum with the anchor has ulp Q^d, so its low mantissa bits are
  // floor(S / Q^d) (unsigned, round toward zero) or round(S / Q^d) + Q/2
  // (balanced, round to nearest)
  return (uint32_t)__double2loint(BAL ? __dadd_rn(acc, anchor) : __dadd_rz(acc, anchor)) & qmask;
}

template <int BK, bool BAL>
__global__ void __launch_bounds__(SM_NT, 2) k_small_tiled(SmallArgs args) {
  constexpr uint32_t CHUNK = SM_BM * BK * 8;  // bytes of one 64 x BK operand chunk
  extern __shared__ __align__(128) double smem[];
  const int NS = args.nstages;               // ring depth
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + (size_t)NS * 2 * SM_BM * BK);
  uint32_t* red = reinterpret_cast<uint32_t*>(smem);  // [64][64] partial digit sums (after the k loop)

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, tq = lane & 3;
  const int warp_m = warp >> 2, warp_n = warp & 3;
  const int m0 = blockIdx.y * SM_BM, n0 = blockIdx.x * SM_BN;
  const int s_begin = blockIdx.z * args.split_stages;
  const int s_end = min(args.Kt, s_begin + args.split_stages);
  const int nst = s_end - s_begin;
  // the 64-row half of 128-row block (m0 / 128) that holds rows m0.., at stage 0
  const double* a_src = args.a + ((size_t)(m0 >> 7) * args.Kt * 128 + (m0 & 64)) * BK;
  const double* b_src = args.b + ((size_t)(n0 >> 7) * args.Kt * 128 + (n0 & 64)) * BK;

  if (tid == 0) {
    for (int i = 0; i < NS; ++i) bar_init(full + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  auto issue = [&](int i) {  // stage i of this split into ring slot i % NS (thread 0)
    if (i < nst) {
      const int sl = i % NS;
      double* sA = smem + (size_t)sl * 2 * SM_BM * BK;
      const size_t off = (size_t)(s_begin + i) * 128 * BK;
      bar_expect_tx(full + sl, 2 * CHUNK);
      bulk_copy(sA, a_src + off, CHUNK, full + sl);
      bulk_copy(sA + SM_BM * BK, b_src + off, CHUNK, full + sl);
    }
  };
  if (tid == 0)
    for (int i = 0; i < NS - 1; ++i) issue(i);

  double acc[SM_MI][SM_NI][2];
  uint32_t ds[SM_MI][SM_NI][2];
#pragma unroll
  for (int i = 0; i < SM_MI; ++i)
#pragma unroll
    for (int j = 0; j < SM_NI; ++j) {
      acc[i][j][0] = acc[i][j][1] = 0.0;
      ds[i][j][0] = ds[i][j][1] = 0u;
    }

  int kst = 0;
  for (int i = 0; i < nst; ++i) {
    if (tid == 0) issue(i + NS - 1);  // its slot was released by the barrier ending stage i - 1
    const int sl = i % NS;
    bar_wait(full + sl, (uint32_t)((i / NS) & 1));
    const double* sA = smem + (size_t)sl * 2 * SM_BM * BK;
    const double* sB = sA + SM_BM * BK;
    // A chunk [64][BK] row-major, B^T chunk [64 cols][BK]: BK = 4 or 12 (mod 16)
    // makes both fragment loads conflict-free
    const double* a_base = sA + (warp_m * SM_WM + g) * BK + tq;
    const double* b_base = sB + (warp_n * SM_WN + g) * BK + tq;
#pragma unroll
    for (int kk = 0; kk < BK / 4; ++kk) {
      double af[SM_MI], bf[SM_NI];
#pragma unroll
      for (int mi = 0; mi < SM_MI; ++mi) af[mi] = a_base[mi * 8 * BK + kk * 4];
#pragma unroll
      for (int ni = 0; ni < SM_NI; ++ni) bf[ni] = b_base[ni * 8 * BK + kk * 4];
#pragma unroll
      for (int mi = 0; mi < SM_MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < SM_NI; ++ni) dmma_s(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
    }
    // k-block end (never at the split's last stage: that digit leaves below)
    if (args.kb_stages && ++kst == args.kb_stages && i + 1 < nst) {
      kst = 0;
#pragma unroll
      for (int mi = 0; mi < SM_MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < SM_NI; ++ni)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            ds[mi][ni][h] += digit_of<BAL>(acc[mi][ni][h], args.anchor, args.qmask);
            acc[mi][ni][h] = 0.0;
          }
    }
    __syncthreads();  // every warp is done with slot sl: it may be refilled
  }
#pragma unroll
  for (int mi = 0; mi < SM_MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < SM_NI; ++ni)
#pragma unroll
      for (int h = 0; h < 2; ++h) ds[mi][ni][h] += digit_of<BAL>(acc[mi][ni][h], args.anchor, args.qmask);

  // ---- cluster reduction of the split partial sums over distributed shared memory
  const int lr0 = warp_m * SM_WM + g, lc0 = warp_n * SM_WN + 2 * tq;
  if (gridDim.z > 1) {
    cg::cluster_group cluster = cg::this_cluster();
    const unsigned rank = cluster.block_rank();
    if (rank != 0) {
#pragma unroll
      for (int mi = 0; mi < SM_MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < SM_NI; ++ni)
          *reinterpret_cast<uint2*>(red + (lr0 + mi * 8) * SM_BN + lc0 + ni * 8) = make_uint2(ds[mi][ni][0], ds[mi][ni][1]);
    }
    cluster.sync();
    if (rank == 0) {
      for (unsigned r = 1; r < cluster.num_blocks(); ++r) {
        const uint32_t* peer = cluster.map_shared_rank(red, r);
#pragma unroll
        for (int mi = 0; mi < SM_MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < SM_NI; ++ni) {
            const uint2 v = *reinterpret_cast<const uint2*>(peer + (lr0 + mi * 8) * SM_BN + lc0 + ni * 8);
            ds[mi][ni][0] += v.x;
            ds[mi][ni][1] += v.y;
          }
      }
    }
    cluster.sync();  // peers stay resident until the leader has read their sums
    if (rank != 0) return;
  }
  // ---- epilogue: mod p (+ the balanced Q/2 bias correction), int32 C
  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
  const bool pairs = (args.ldc % 2 == 0) && ((reinterpret_cast<uintptr_t>(args.c) & 7) == 0);
#pragma unroll
  for (int mi = 0; mi < SM_MI; ++mi) {
    const int row = m0 + lr0 + mi * 8;
    if (row >= args.M) continue;
#pragma unroll
    for (int ni = 0; ni < SM_NI; ++ni) {
      const int col = n0 + lc0 + ni * 8;
      int32_t* dst = args.c + (size_t)row * args.ldc + col;
      const int32_t r0 = (int32_t)modp(ds[mi][ni][0] + args.corr), r1 = (int32_t)modp(ds[mi][ni][1] + args.corr);
      if (pairs && col + 1 < args.N) {
        *reinterpret_cast<int2*>(dst) = make_int2(r0, r1);
      } else {
        if (col < args.N) dst[0] = r0;
        if (col + 1 < args.N) dst[1] = r1;
      }
    }
  }
}

template <int BK, bool BAL>
cudaError_t launch_small_t(const SmallArgs& a0, int splits, cudaStream_t s) {
  auto k = k_small_tiled<BK, BAL>;
  SmallArgs a = a0;
  // ring depth: 2..4 stages within ~110 KB, so two CTAs fit on an SM
  const size_t stage = (size_t)2 * SM_BM * BK * sizeof(double);
  int ns = (int)((110 * 1024) / stage);
  ns = ns > 4 ? 4 : (ns < 2 ? 2 : ns);
  a.nstages = ns;
  size_t smem = ns * stage;
  const size_t redb = (size_t)SM_BM * SM_BN * sizeof(uint32_t);
  if (smem < redb) smem = redb;
  smem += 8 * sizeof(uint64_t);
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)((a.N + SM_BN - 1) / SM_BN), (unsigned)((a.M + SM_BM - 1) / SM_BM), (unsigned)splits);
  cfg.blockDim = dim3(SM_NT);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = 1;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = (unsigned)splits;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  err = cudaLaunchKernelEx(&cfg, k, a);
  count_launch();
  return err ? err : cudaGetLastError();
}

template <bool BAL>
cudaError_t launch_small_b(const SmallArgs& a, int bk, int splits, cudaStream_t s) {
  switch (bk) {
    case 52: return launch_small_t<52, BAL>(a, splits, s);
    case 44: return launch_small_t<44, BAL>(a, splits, s);
    case 36: return launch_small_t<36, BAL>(a, splits, s);
    case 28: return launch_small_t<28, BAL>(a, splits, s);
    case 20: return launch_small_t<20, BAL>(a, splits, s);
    case 12: return launch_small_t<12, BAL>(a, splits, s);
    case 4: return launch_small_t<4, BAL>(a, splits, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace

cudaError_t launch_small_tiled(const SmallArgs& a, int bk, int splits, cudaStream_t s, const char** variant) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  if (splits < 1 || splits > 8) return cudaErrorInvalidValue;
  static thread_local char name[80];
  snprintf(name, sizeof name, "small_tiled_bk%d_s%d%s", bk, splits, a.balanced ? "_balanced" : "");
  if (variant) *variant = name;
  return a.balanced ? launch_small_b<true>(a, bk, splits, s) : launch_small_b<false>(a, bk, splits, s);
}

}  // namespace qgk
