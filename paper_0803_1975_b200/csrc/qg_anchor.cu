// qg_anchor.cu — K4A: the common (dot-product) contraction with ANCHORED
// accumulators (packed_common_product + reduce_common_entry + blocked_accumulate,
// gemm.hpp:210-271, 450-489), balanced digits, tiled layout.
//
// K4 (qg_dot.cu) ends every k-block with one DADD per accumulator (acc +
// anchor, rounded), whose low mantissa bits are the block's digit d. DADD and
// DMMA share the FP64 datapath: with 20-word blocks (config 5) the 64 DADDs
// per warp per block take 1/21 of the pipe and, with their drain, cost ~10
// points of the DMMA peak (no-flush timing 97.4 % vs 86.8 %).
//
// Here the anchor is folded into the accumulation instead: the first DMMA of
// every block takes C = anchor = 1.5*2^E + Q^d/2 + Q^d*Q/2 (a uniform register
// quad {anchor, anchor + Q^(d+1)} — two distinct values, or ptxas rebuilds the
// pair with four MOVs before every such DMMA; the difference is invisible to
// the digit field; D overwrites the accumulator, so nothing is zeroed), every
// partial sum
// of the block stays inside the binade [2^E, 2^(E+1)) (planner:
// qg::max_exact_block_anchored), so its ulp is u = 2^(E-52) throughout and the
// block's digit d sits at FIXED bits [s, s+t) of the accumulator's low word,
// s = t d - (E - 52): the flush is one LOP3 and one IADD per accumulator on
// the integer pipe, issued right before that accumulator's first DMMA of the
// next block — no FP64-pipe work, no drain. The digit sums stay scaled by 2^s
// until the epilogue.
//
// Exactness: every operation rounds onto the grid u Z, which
// contains Q^d/2 Z; with at most one rounding of the product (unfused, err <=
// ulp(x_max)) and one of the add (err <= u) per word, in any order,
// |S^ - S| <= Kb (u + ulp(x_max)), and digit d of the block is
// floor((S^ + Q^d/2) / Q^d) mod Q (biased by Q/2) whenever
// 2 (L_max(Kb) + Kb (u + ulp(x_max))) < Q^d — Eq. G with the fixed ulp u.
#include <atomic>
#include <cstdio>
#include <cstdlib>

#include "qg_kernels.h"
#include "qg_device.cuh"

namespace qgk {
namespace {

constexpr int BM = 128, BN = 128;
constexpr int WM = 64, WN = 32;
constexpr int WARPS_N = BN / WN;
constexpr int NT = (BM / WM) * (BN / WN) * 32;  // 256 consumer threads
constexpr int MI = WM / 8, NI = WN / 8;

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
      "{\n .reg .pred p;\n QGA_WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra QGA_WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

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

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}
// D = A * B + c (both C elements the same uniform constant): the first k-step of a k-block.
__device__ __forceinline__ void dmma_c(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%4,%5};\n"
               : "=d"(d0), "=d"(d1)
               : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

// One k-block (BK words = KBS k-steps) of the warp tile from the operand blocks at a_blk / b_blk
// (dense 128 x BK, B transposed). Split flush: accumulator row mi ends its blocks after k-step
// (mi % KBS) - 1 of every block (shifted windows of exactly KBS k-steps — any partition of k into
// pieces of <= the exact block is exact), so every k-step carries 1/KBS of the integer flush work.
// Measured (profiles/r02_notes.md): 92.9-93.4 % of the DMMA peak on config 5 (12-word blocks); the
// same loop without restarts 98.8 %. At a block boundary the finished block's digit leaves the accumulator's low word (LOP3 + IADD) and
// the DMMA restarts the accumulator from the anchor pair {c0, c1}.
template <int BK>
__device__ __forceinline__ void anchored_block(double (&acc)[MI][NI][2], uint32_t (&ds)[MI][NI][2],
                                               const double* a_blk, const double* b_blk, uint32_t amask,
                                               double c0, double c1) {
  constexpr int KBS = BK / 4;
#pragma unroll
  for (int kk = 0; kk < KBS; ++kk) {
    double af[MI], bf[NI];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi) af[mi] = a_blk[mi * 8 * BK + kk * 4];
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) bf[ni] = b_blk[ni * 8 * BK + kk * 4];
#pragma unroll
    for (int mi = 0; mi < MI; ++mi)
#pragma unroll
      for (int ni = 0; ni < NI; ++ni) {
        if (kk == mi % KBS) {
          ds[mi][ni][0] += (uint32_t)__double2loint(acc[mi][ni][0]) & amask;
          ds[mi][ni][1] += (uint32_t)__double2loint(acc[mi][ni][1]) & amask;
          dmma_c(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni], c0, c1);
        } else {
          dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
      }
  }
}

// Zero operand blocks for the slots that reach past the end of K (SS > 1): (SS - 1) blocks at most.
__device__ __align__(128) double g_zero_blocks[2 * BM * 20];  // >= 2 * 128 * 12 (BK 12, SS 3) and 1 * 128 * 20 (BK 20, SS 2)

// BK: words per k-block = stage depth of the tiled layout (an odd multiple of 4, conflict-free
// fragment loads). SS: blocks per pipeline slot ("super-stage"): consecutive blocks of one row panel
// are contiguous in CA_t / CB_t, so a slot is still two bulk copies (SS * 128 * BK * 8 bytes each) and
// one full/empty barrier round; short blocks (BK = 12) then pay their barrier and producer overhead
// once per SS blocks. A tile's last slot is filled up with zero blocks (exact no-ops that only add
// extractions of the bias, counted in corr), so the consumers have no tail code.
constexpr int REPACK_SMEM = BM * BN;  // REPACK: one byte per residue (p < 256), one 64 x 32 tile per warp

template <int BK, int SS, bool REPACK>
__global__ void __launch_bounds__(NT + 128, 1) k_gemm_anchor(GemmArgs args, int tiles_m, int tiles_n) {
  constexpr int SLOT = 2 * SS * BM * BK;  // doubles per slot: SS blocks of A, then SS blocks of B
  constexpr int BUDGET = 232448 - 1024 - (REPACK ? REPACK_SMEM : 0);
  constexpr int S_RAW = BUDGET / (SLOT * 8);
  constexpr int S = S_RAW > 8 ? 8 : S_RAW;
  static_assert(S >= 2, "at least two slots");
  constexpr int NWARPS = NT / 32;
  constexpr uint32_t CHUNK = BM * BK * 8;  // bytes of one operand block
  extern __shared__ __align__(128) double smem[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * SLOT);
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
  const int kblocks = (args.K + BK - 1) / BK;  // blocks of the layout
  const int nslots = (kblocks + SS - 1) / SS;  // pipeline slots per tile (the last one zero-filled past K)
  const int total_tiles = tiles_m * tiles_n;
  const int my_tiles = blockIdx.x < total_tiles ? (total_tiles - 1 - blockIdx.x) / gridDim.x + 1 : 0;
  volatile int* tile_of = reinterpret_cast<volatile int*>(empty + S);
  uint8_t* repack = reinterpret_cast<uint8_t*>(empty + S + 4);  // REPACK staging (after barriers + tile_of)
  const bool dyn = args.tile_counter != nullptr;

  if (warp >= NWARPS) {
    // ---- producer warpgroup: one lane streams the tiles' slots (two bulk copies each)
    asm volatile("setmaxnreg.dec.sync.aligned.u32 24;\n" ::: "memory");
    if (warp != NWARPS || lane != 0) return;
    uint32_t slot = 0, phase = 0;
    for (int ts = 0;; ++ts) {
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
      const double* ablk = args.a + (size_t)tm * kblocks * BM * BK;
      const double* bblk = args.b + (size_t)tn * kblocks * BM * BK;
      for (int st = 0; st < nslots; ++st) {
        const int nb = (kblocks - st * SS) < SS ? (kblocks - st * SS) : SS;  // real blocks in this slot
        const size_t off = (size_t)st * SS * BM * BK;
        mbar_wait(empty + slot, phase ^ 1);
        double* sA = smem + slot * SLOT;
        if (dyn && st == 0) tile_of[slot] = tile;
        mbar_arrive_expect_tx(full + slot, 2 * SS * CHUNK);
        bulk_g2s(sA, ablk + off, nb * CHUNK, full + slot);
        bulk_g2s(sA + SS * BM * BK, bblk + off, nb * CHUNK, full + slot);
        if (SS > 1 && nb < SS) {  // the last slot of a tile: zero blocks past the end of K (they add nothing)
          bulk_g2s(sA + nb * BM * BK, g_zero_blocks, (SS - nb) * CHUNK, full + slot);
          bulk_g2s(sA + (SS + nb) * BM * BK, g_zero_blocks, (SS - nb) * CHUNK, full + slot);
        }
        if (++slot == S) {
          slot = 0;
          phase ^= 1;
        }
      }
    }
    return;
  }

  // ---- consumer warps
  asm volatile("setmaxnreg.inc.sync.aligned.u32 240;\n" ::: "memory");
  const int M = args.M, N = args.N;
  const int g = lane >> 2, t = lane & 3;
  const int warp_m = warp / WARPS_N, warp_n = warp % WARPS_N;
  // C operand of a block's first DMMA: the register quad {anchor, anchor + delta}. delta = Q^(d+1) is
  // invisible to the digit field; two DISTINCT values keep ptxas from rebuilding the pair in the
  // accumulator's registers (4 MOVs) before every such DMMA.
  const double anchor = args.anchor;
  const double anchor1 = args.anchor1;
  const uint32_t amask = args.qmask << args.anch_shift;
  const int sh = args.anch_shift;
  double acc[MI][NI][2];
  uint32_t ds[MI][NI][2];
#pragma unroll
  for (int mi = 0; mi < MI; ++mi)
#pragma unroll
    for (int ni = 0; ni < NI; ++ni) {
      acc[mi][ni][0] = anchor;
      acc[mi][ni][1] = anchor1;
      ds[mi][ni][0] = ds[mi][ni][1] = 0u;
    }
  const ModP modp{args.p, (uint32_t)(0x100000000ull / args.p)};
  uint32_t slot = 0, phase = 0;
  if (warp >= 4 && args.skew_ns > 0) start_skew(args.skew_ns);  // desynchronise the SMSP's two warps
  const int a_off = (warp_m * WM + g) * BK + t;                // fragment bases inside an operand block
  const int b_off = SS * BM * BK + (warp_n * WN + g) * BK + t;
  for (int ts = 0;; ++ts) {
    int tile;
    if (dyn) {
      mbar_wait(full + slot, phase);  // the tile's first slot (and its index) has landed
      tile = tile_of[slot];
      if (tile < 0) break;
    } else {
      if (ts >= my_tiles) break;
      tile = blockIdx.x + ts * gridDim.x;
    }
    int tm, tn;
    tile_coords(tile, tiles_m, tiles_n, args.group, tm, tn);
    const int m0 = tm * BM, n0 = tn * BN;
    for (int st = 0; st < nslots; ++st) {
      if (!(dyn && st == 0)) mbar_wait(full + slot, phase);
      const double* sA = smem + slot * SLOT;
#pragma unroll
      for (int j = 0; j < SS; ++j)
        anchored_block<BK>(acc, ds, sA + a_off + j * BM * BK, sA + b_off + j * BM * BK, amask, anchor, anchor1);
      __syncwarp();
      if (lane == 0) mbar_arrive(empty + slot);
      if (++slot == S) {
        slot = 0;
        phase ^= 1;
      }
    }
    // epilogue: last block's digit + digit sums (scaled by 2^sh), biases removed mod p
    if (REPACK) {  // mul_common_repacked: residues -> this warp's byte tile -> forward-packed words
      uint8_t* st = repack + warp * (WM * WN);
#pragma unroll
      for (int mi = 0; mi < MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t x =
                ((((uint32_t)__double2loint(acc[mi][ni][h]) & amask) + ds[mi][ni][h]) >> sh) + args.corr;
            const uint32_t r0 = x - __umulhi(x, modp.magic) * modp.p;
            r[h] = min(r0, r0 - modp.p);
            acc[mi][ni][h] = h ? anchor1 : anchor;
            ds[mi][ni][h] = 0u;
          }
          *reinterpret_cast<uint16_t*>(st + (mi * 8 + g) * WN + ni * 8 + 2 * t) = (uint16_t)(r[0] | (r[1] << 8));
        }
      __syncwarp();
      repack_warp_segment(st, args.cc, args.ldcc, M, N, args.e, args.t, m0 + warp_m * WM, n0 + warp_n * WN, lane);
      __syncwarp();  // the next tile overwrites the staging tile
      continue;
    }
    const bool fast = !args.accumulate && m0 + BM <= M && n0 + BN <= N;
    if (fast) {
      int32_t* cbase = args.c + (size_t)(m0 + warp_m * WM + g) * args.ldc + n0 + warp_n * WN + 2 * t;
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        int32_t* crow = cbase + (size_t)(mi * 8) * args.ldc;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint32_t x =
                ((((uint32_t)__double2loint(acc[mi][ni][h]) & amask) + ds[mi][ni][h]) >> sh) + args.corr;
            const uint32_t r0 = x - __umulhi(x, modp.magic) * modp.p;
            r[h] = min(r0, r0 - modp.p);
            acc[mi][ni][h] = h ? anchor1 : anchor;
            ds[mi][ni][h] = 0u;
          }
          *reinterpret_cast<int2*>(crow + ni * 8) = make_int2((int)r[0], (int)r[1]);
        }
      }
    } else {
#pragma unroll
      for (int mi = 0; mi < MI; ++mi) {
        const int row = m0 + warp_m * WM + mi * 8 + g;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
          const int col = n0 + warp_n * WN + ni * 8 + 2 * t;
          uint32_t r[2];
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            r[h] = ((((uint32_t)__double2loint(acc[mi][ni][h]) & amask) + ds[mi][ni][h]) >> sh) + args.corr;
            acc[mi][ni][h] = h ? anchor1 : anchor;
            ds[mi][ni][h] = 0u;
          }
          if (row < M && col < N) {  // N even: col < N implies col + 1 < N
            int32_t* dst = args.c + (size_t)row * args.ldc + col;
            if (args.accumulate) {
              const int2 old = *reinterpret_cast<const int2*>(dst);
              r[0] += (uint32_t)old.x;
              r[1] += (uint32_t)old.y;
            }
            *reinterpret_cast<int2*>(dst) = make_int2((int)modp(r[0]), (int)modp(r[1]));
          }
        }
      }
    }
  }
}

int num_sms_a() {
  static std::atomic<int> cached[64];
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  int v = cached[dev].load();
  if (v > 0) return v;
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (sms <= 0) sms = 148;
  cached[dev].store(sms);
  return sms;
}

template <int BK, int SS, bool REPACK>
cudaError_t launch_anchor_one(const GemmArgs& a, int* tile_counter, cudaStream_t s) {
  auto k = k_gemm_anchor<BK, SS, REPACK>;
  constexpr int SLOT = 2 * SS * BM * BK;
  constexpr int S_RAW = (232448 - 1024 - (REPACK ? REPACK_SMEM : 0)) / (SLOT * 8);
  constexpr int S = S_RAW > 8 ? 8 : S_RAW;
  const size_t smem = size_t(S) * SLOT * sizeof(double) + (2 * S + 4) * sizeof(uint64_t) + (REPACK ? REPACK_SMEM : 0);
  cudaError_t err = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (err) return err;
  const int tiles_m = (a.M + BM - 1) / BM, tiles_n = (a.N + BN - 1) / BN;
  const int tiles = tiles_m * tiles_n;
  const int grid = tiles < num_sms_a() ? tiles : num_sms_a();
  GemmArgs a2 = a;
  const char* skew = getenv("QG_SKEW_NS");
  a2.skew_ns = skew ? (unsigned)atoi(skew) : 3000u;
  if (const char* sl = getenv("QG_SKEW_SLEEP"))
    if (sl[0] == '1' && a2.skew_ns) a2.skew_ns |= 0x80000000u;  // experiments: nanosleep instead of the clock spin
  const char* grp = getenv("QG_GROUP");
  a2.group = grp ? atoi(grp) : 8;
  a2.tile_counter = tile_counter;
  // one extraction per block start (the first reads the bare anchor; zero blocks included) + the final one
  const unsigned long long kblocks = (unsigned long long)((a.K + BK - 1) / BK);
  const unsigned long long nb = (kblocks + SS - 1) / SS * SS + 1;
  const unsigned long long halfq = ((unsigned long long)a.qmask + 1) / 2;
  a2.corr = (uint32_t)((a.p - (nb % a.p) * (halfq % a.p) % a.p) % a.p);
  k<<<grid, NT + 128, smem, s>>>(a2, tiles_m, tiles_n);
  count_launch();
  return cudaGetLastError();
}

// kb_words: the block length = the stage depth of the tiled layout (a.K words per row, blocks of
// kb_words). Extractions per output, for the caller's uint32 digit-sum check: <= ceil(K / kb_words) + 3.
template <int BK, int SS>
cudaError_t launch_anchor_bk(const GemmArgs& a, int* tile_counter, cudaStream_t s, bool repack) {
  return repack ? launch_anchor_one<BK, SS, true>(a, tile_counter, s) : launch_anchor_one<BK, SS, false>(a, tile_counter, s);
}

}  // namespace

cudaError_t launch_dot_anchor(const GemmArgs& a, int kb_words, int* tile_counter, cudaStream_t s,
                              const char** variant, bool repack) {
  if (a.M == 0 || a.N == 0) return cudaSuccess;
  static thread_local char name[80];
  snprintf(name, sizeof name, "dot_tiled_%sanchor_kb%d_balanced", repack ? "repack_" : "", kb_words);
  *variant = name;
  switch (kb_words) {
    case 12: return launch_anchor_bk<12, 3>(a, tile_counter, s, repack);
    case 20: return launch_anchor_bk<20, 2>(a, tile_counter, s, repack);
    case 28: return launch_anchor_bk<28, 1>(a, tile_counter, s, repack);
    case 36: return launch_anchor_bk<36, 1>(a, tile_counter, s, repack);
    case 44: return launch_anchor_bk<44, 1>(a, tile_counter, s, repack);
    case 52: return launch_anchor_bk<52, 1>(a, tile_counter, s, repack);
  }
  return cudaErrorInvalidValue;
}

}  // namespace qgk
