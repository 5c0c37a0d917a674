// qg_device.cuh — device helpers shared by the sm_100a kernels.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace qgk {

// Residue element -> integer. Residues on the device are exact small
// integers held as double (BASELINE "stored as double") or as uint32/int32
// (ResidueMatrix::data, matrix.hpp:14-26).
__device__ __forceinline__ uint64_t residue_bits(double v) { return (uint64_t)__double2ull_rz(v); }
__device__ __forceinline__ uint64_t residue_bits(uint32_t v) { return v; }
__device__ __forceinline__ uint64_t residue_bits(int32_t v) { return (uint64_t)(uint32_t)v; }

__device__ __forceinline__ void store_residue(double* p, uint32_t v) { *p = (double)v; }
__device__ __forceinline__ void store_residue(uint32_t* p, uint32_t v) { *p = v; }

// floor(s / 2^(t d)) & mask for an integer-valued double s >= 0, read from the
// IEEE bits (no FP64-pipe work, no extra rounding): s = M * 2^(E - 1075), so
// the high part is M >> (1075 + t d - E). sh_base = 1075 + t d. The exactness
// planner guarantees ulp(s) <= Q^d, i.e. the shift is never negative.
__device__ __forceinline__ uint32_t digit_at(double s, int sh_base, uint32_t mask) {
  const unsigned long long bits = (unsigned long long)__double_as_longlong(s);
  const int E = (int)(bits >> 52);
  const unsigned long long M = (bits & 0xFFFFFFFFFFFFFull) | 0x10000000000000ull;
  int sh = sh_base - E;
  sh = sh < 0 ? 0 : (sh > 63 ? 63 : sh);
  return (uint32_t)(M >> sh) & mask;
}

// SplitMix64::next at counter position `index` (prng.hpp:16-21): the state
// after index+1 calls is seed + (index+1) * golden gamma.
__device__ __forceinline__ uint64_t splitmix64_at(uint64_t seed, uint64_t index) {
  uint64_t z = seed + (index + 1ull) * 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}

// x mod p for x < 2^32, p >= 2, with a precomputed magic = floor(2^32 / p):
// q underestimates floor(x/p) by at most 1, so one correction suffices.
struct ModP {
  uint32_t p;
  uint32_t magic;
  __device__ __forceinline__ uint32_t operator()(uint32_t x) const {
    uint32_t q = __umulhi(x, magic);
    uint32_t r = x - q * p;
    return r >= p ? r - p : r;
  }
};

// Start delay of the second warp of every SMSP (warps 4..7), so that the two warps sharing a DMMA
// pipe run their k-block flushes / tile epilogues half a phase apart. A clock spin: __nanosleep(t)
// sleeps anywhere in [0, 2t], which made the one-stage-per-tile products (config 3) bimodal across
// runs. Bit 31 of skew_ns (QG_SKEW_SLEEP=1, experiments) selects the old nanosleep.
__device__ __forceinline__ void start_skew(unsigned skew_ns) {
  if (skew_ns & 0x80000000u) {
    __nanosleep(skew_ns & 0x7fffffffu);
    return;
  }
  const long long t0 = clock64();
  const long long cycles = 2ll * skew_ns;  // ~2 SM cycles per ns (1.965 GHz)
  while (clock64() - t0 < cycles) {
  }
}

// ReduceAndCompress of one warp's 64 x 32 residue tile (st, row-major, 32
// bytes per row; rows r0.., columns c0.. of the M x N product): word h of a
// row packs columns h e .. h e + e - 1 forward in base Q = 2^t
// (compress_forward, pack.hpp:47-54; reduce_and_compress, pack.hpp:141-155).
// Words whose columns all lie in this segment are stored; a word cut by the
// segment's edge gets its part added atomically (the parts occupy disjoint
// bits, so the float64 sums are exact integers < 2^53 in any order; the
// launcher zeroes CC first whenever a word can straddle segments).
__device__ __forceinline__ void repack_warp_segment(const uint8_t* st, double* cc, size_t ldcc, int M, int N, int e,
                                                    int tb, int r0, int c0, int lane) {
  constexpr int SEG_ROWS = 64, SEG_COLS = 32;
  if (c0 >= N) return;
  const int cend = min(c0 + SEG_COLS, N);
  const int h_lo = c0 / e, h_hi = (cend - 1) / e, W = h_hi - h_lo + 1;
  const int rows = min(SEG_ROWS, M - r0);
  for (int idx = lane; idx < rows * W; idx += 32) {
    const int row = idx / W, hw = h_lo + (idx - row * W);
    const int wc0 = hw * e;
    const int lo = max(wc0, c0), hi = min(wc0 + e, cend);
    uint64_t word = 0;
    for (int c = lo; c < hi; ++c) word |= (uint64_t)st[row * SEG_COLS + (c - c0)] << (tb * (c - wc0));
    double* dst = cc + (size_t)(r0 + row) * ldcc + hw;
    const double wd = __ull2double_rn(word);  // exact: word < Q^e <= 2^53
    if (wc0 >= c0 && min(wc0 + e, N) <= cend) *dst = wd;
    else atomicAdd(dst, wd);
  }
}

}  // namespace qgk
