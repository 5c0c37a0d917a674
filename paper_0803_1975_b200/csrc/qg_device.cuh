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

}  // namespace qgk
