// qg_word64.cu — the Int64Word backend (word.hpp:36-54) on the device: packed
// words are uint64, word products wrap modulo 2^64, and the common product
// adds Int64Word::high_part = ((a b) >> t d) & (Q - 1) per term. Plans may use
// up to beta = 63 bits (t e <= 62). Integer work on the CUDA cores: the
// backend exists for bit-exact parity with the reference's Int64Word results,
// not as a fast path (the FP64 tensor-core path covers every DoubleWord plan).
#include "qg_kernels.h"
#include "qg_device.cuh"

namespace qgk {

template <typename T>
__device__ __forceinline__ uint64_t as_u64(T v) {
  return (uint64_t)residue_bits(v);
}
template <>
__device__ __forceinline__ uint64_t as_u64<uint64_t>(uint64_t v) {
  return v;
}

// D[i][j] = sum_l term(A[i][l], B[l][j]) mod 2^64, term = a b (HIGH = false)
// or ((a b) >> sh) & mask (HIGH = true, Int64Word::high_part). 64 x 64 output
// tiles, 256 threads x (4 x 4) outputs, 16-deep k slices through shared memory.
template <bool HIGH, typename TA, typename TB>
__global__ void __launch_bounds__(256) k_gemm_u64(const TA* __restrict__ a, size_t lda, const TB* __restrict__ b,
                                                  size_t ldb, size_t M, size_t N, size_t K, int sh, uint64_t mask,
                                                  uint64_t* __restrict__ d, size_t ldd) {
  __shared__ uint64_t sa[16][64 + 1], sb[16][64 + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const size_t m0 = (size_t)blockIdx.y * 64, n0 = (size_t)blockIdx.x * 64;
  uint64_t acc[4][4] = {};
  for (size_t k0 = 0; k0 < K; k0 += 16) {
    for (int i = threadIdx.x; i < 64 * 16; i += 256) {
      const int r = i >> 4, c = i & 15;  // A tile: 64 rows x 16 k
      const size_t gr = m0 + r, gk = k0 + c;
      sa[c][r] = (gr < M && gk < K) ? as_u64(a[gr * lda + gk]) : 0ull;
      const int kr = i >> 6, nc = i & 63;  // B tile: 16 k x 64 cols
      const size_t bk = k0 + kr, bn = n0 + nc;
      sb[kr][nc] = (bk < K && bn < N) ? as_u64(b[bk * ldb + bn]) : 0ull;
    }
    __syncthreads();
#pragma unroll 4
    for (int l = 0; l < 16; ++l) {
      uint64_t av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = sa[l][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = sb[l][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint64_t prod = av[i] * bv[j];
          acc[i][j] += HIGH ? ((prod >> sh) & mask) : prod;
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const size_t r = m0 + ty + 16 * i, c = n0 + tx + 16 * j;
      if (r < M && c < N) d[r * ldd + c] = acc[i][j];
    }
}

template <bool HIGH, typename TA, typename TB>
static cudaError_t gemm_u64(const TA* a, size_t lda, const TB* b, size_t ldb, size_t M, size_t N, size_t K, int sh,
                            uint64_t mask, uint64_t* d, size_t ldd, cudaStream_t s) {
  if (M == 0 || N == 0) return cudaSuccess;
  if ((M + 63) / 64 > 65535) return cudaErrorInvalidValue;
  const dim3 grid((unsigned)((N + 63) / 64), (unsigned)((M + 63) / 64));
  k_gemm_u64<HIGH, TA, TB><<<grid, 256, 0, s>>>(a, lda, b, ldb, M, N, K, sh, mask, d, ldd);
  count_launch();
  return cudaGetLastError();
}

// residue operand of a mixed product: dtype 0 double, 1 uint32, 2 int32
template <bool HIGH>
static cudaError_t gemm_res_a(const void* a, int dtype, size_t lda, const uint64_t* b, size_t ldb, size_t M, size_t N,
                              size_t K, int sh, uint64_t mask, uint64_t* d, size_t ldd, cudaStream_t s) {
  switch (dtype) {
    case 0: return gemm_u64<HIGH>((const double*)a, lda, b, ldb, M, N, K, sh, mask, d, ldd, s);
    case 1: return gemm_u64<HIGH>((const uint32_t*)a, lda, b, ldb, M, N, K, sh, mask, d, ldd, s);
    default: return gemm_u64<HIGH>((const int32_t*)a, lda, b, ldb, M, N, K, sh, mask, d, ldd, s);
  }
}
template <bool HIGH>
static cudaError_t gemm_res_b(const uint64_t* a, size_t lda, const void* b, int dtype, size_t ldb, size_t M, size_t N,
                              size_t K, int sh, uint64_t mask, uint64_t* d, size_t ldd, cudaStream_t s) {
  switch (dtype) {
    case 0: return gemm_u64<HIGH>(a, lda, (const double*)b, ldb, M, N, K, sh, mask, d, ldd, s);
    case 1: return gemm_u64<HIGH>(a, lda, (const uint32_t*)b, ldb, M, N, K, sh, mask, d, ldd, s);
    default: return gemm_u64<HIGH>(a, lda, (const int32_t*)b, ldb, M, N, K, sh, mask, d, ldd, s);
  }
}

cudaError_t launch_gemm_u64(int mode, const void* a, int a_dtype, size_t lda, const void* b, int b_dtype, size_t ldb,
                            size_t M, size_t N, size_t K, int sh, uint64_t mask, uint64_t* d, size_t ldd,
                            cudaStream_t s) {
  // a_dtype / b_dtype: -1 = uint64 words, else a residue dtype
  const bool high = mode == 0;
  if (a_dtype < 0 && b_dtype < 0)
    return high ? gemm_u64<true>((const uint64_t*)a, lda, (const uint64_t*)b, ldb, M, N, K, sh, mask, d, ldd, s)
                : gemm_u64<false>((const uint64_t*)a, lda, (const uint64_t*)b, ldb, M, N, K, sh, mask, d, ldd, s);
  if (a_dtype >= 0 && b_dtype < 0)
    return high ? gemm_res_a<true>(a, a_dtype, lda, (const uint64_t*)b, ldb, M, N, K, sh, mask, d, ldd, s)
                : gemm_res_a<false>(a, a_dtype, lda, (const uint64_t*)b, ldb, M, N, K, sh, mask, d, ldd, s);
  if (a_dtype < 0 && b_dtype >= 0)
    return high ? gemm_res_b<true>((const uint64_t*)a, lda, b, b_dtype, ldb, M, N, K, sh, mask, d, ldd, s)
                : gemm_res_b<false>((const uint64_t*)a, lda, b, b_dtype, ldb, M, N, K, sh, mask, d, ldd, s);
  return cudaErrorInvalidValue;
}

static unsigned blocks_for(size_t work) {
  size_t b = (work + 255) / 256;
  if (b > 148 * 16) b = 148 * 16;
  return (unsigned)(b ? b : 1);
}

__device__ __forceinline__ uint32_t mod_u64(uint64_t x, uint32_t p) { return (uint32_t)(x % p); }

// Elementwise word routines of the Int64Word backend:
//   op 0 reduce_common_entry (gemm.hpp:247-250): out = (w & mask) mod p
//   op 1 extract_coefficient (pack.hpp:96-98): out = ((w >> t d) & mask) mod p
__global__ void k_word_reduce_u64(const uint64_t* __restrict__ w, size_t count, int op, int shift, uint64_t mask,
                                  uint32_t p, int32_t* __restrict__ out, int accumulate) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t x = op == 0 ? (w[i] & mask) : ((w[i] >> shift) & mask);
    uint32_t r = mod_u64(x, p);
    if (accumulate) r = (uint32_t)(((uint64_t)(uint32_t)out[i] + r) % p);  // blocked_accumulate, gemm.hpp:484-486
    out[i] = (int32_t)r;
  }
}

// redq (pack.hpp:124-137) on uint64 words; words >= 2^(t e) raise DigitOverflow.
__global__ void k_redq_u64(uint64_t* __restrict__ w, size_t count, int t, int e, uint32_t p,
                           int* __restrict__ overflow) {
  const int total = t * e;
  const uint64_t mask = (1ull << t) - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t bits = w[i];
    if (total < 64 && bits >= (1ull << total)) {
      atomicExch(overflow, 1);
      continue;
    }
    uint64_t r = 0;
    for (int s = 0; s < total; s += t) r |= (uint64_t)mod_u64((bits >> s) & mask, p) << s;
    w[i] = r;
  }
}

// uncompress (gemm.hpp:182-204 + extract_all pack.hpp:104-119) of uint64 words.
__global__ void k_uncompress_u64(const uint64_t* __restrict__ w, size_t srows, size_t scols, size_t lrows, size_t lcols,
                                 int t, int e, int slots, int reversed, int column_axis, uint32_t p,
                                 int32_t* __restrict__ out, int* __restrict__ overflow) {
  const int total = t * e;
  const uint64_t mask = (1ull << t) - 1;
  for (size_t si = blockIdx.y; si < srows; si += gridDim.y)
    for (size_t sj = blockIdx.x * (size_t)blockDim.x + threadIdx.x; sj < scols; sj += (size_t)gridDim.x * blockDim.x) {
      const uint64_t bits = w[si * scols + sj];
      if (total < 64 && bits >= (1ull << total)) {
        atomicExch(overflow, 1);
        continue;
      }
      for (int s = 0; s < slots; ++s) {
        const int di = reversed ? slots - 1 - s : s;
        const uint64_t digit = di < e ? (bits >> (t * di)) & mask : 0;
        size_t i = si, j = sj;
        if (column_axis) j = sj * slots + s;
        else i = si * slots + s;
        if (i < lrows && j < lcols) out[i * lcols + j] = (int32_t)mod_u64(digit, p);
      }
    }
}

// reduce_and_compress (pack.hpp:141-155) with Int64Word words in and out.
__global__ void k_reduce_and_compress_u64(const uint64_t* __restrict__ w, size_t rows, size_t cols, size_t ldw, int t,
                                          int d, int e, uint32_t p, uint64_t* __restrict__ out, size_t ldo) {
  const uint64_t mask = (1ull << t) - 1;
  const size_t groups = (cols + e - 1) / e, count = rows * groups;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / groups, g = i % groups, c0 = g * e;
    const int len = (int)((cols - c0) < (size_t)e ? (cols - c0) : (size_t)e);
    uint64_t word = 0;
    for (int s = len - 1; s >= 0; --s) word = (word << t) | mod_u64((w[r * ldw + c0 + s] >> (t * d)) & mask, p);
    out[r * ldo + g] = word;
  }
}

// the unpack of mul_full_compressed (gemm.hpp:427-443) over uint64 words
__global__ void k_uncompress_full_u64(const uint64_t* __restrict__ cc, size_t ldcc, size_t m, size_t n, int t, int qs,
                                      int ts, uint32_t p, int32_t* __restrict__ c, size_t ldc) {
  const uint64_t mask = (1ull << t) - 1;
  for (size_t row = blockIdx.y; row < m; row += gridDim.y)
    for (size_t col = blockIdx.x * (size_t)blockDim.x + threadIdx.x; col < n; col += (size_t)gridDim.x * blockDim.x) {
      const uint64_t bits = cc[(row / qs) * ldcc + col / ts];
      const int pos = (int)(row % qs) + (int)(col % ts) * qs;
      c[row * ldc + col] = (int32_t)mod_u64((bits >> (t * pos)) & mask, p);
    }
}

static dim3 grid_rows(size_t inner, size_t rows) {
  size_t bx = (inner + 255) / 256;
  if (bx > 1024) bx = 1024;
  return dim3((unsigned)(bx ? bx : 1), (unsigned)(rows < 65535 ? (rows ? rows : 1) : 65535));
}

cudaError_t launch_word_reduce_u64(const uint64_t* w, size_t count, int op, int shift, uint64_t mask, uint32_t p,
                                   int32_t* out, int accumulate, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_word_reduce_u64<<<blocks_for(count), 256, 0, s>>>(w, count, op, shift, mask, p, out, accumulate);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_redq_u64(uint64_t* w, size_t count, int t, int e, uint32_t p, int* overflow, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_redq_u64<<<blocks_for(count), 256, 0, s>>>(w, count, t, e, p, overflow);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_uncompress_u64(const uint64_t* w, size_t srows, size_t scols, size_t lrows, size_t lcols, int t,
                                  int e, int slots, int reversed, int column_axis, uint32_t p, int32_t* out,
                                  int* overflow, cudaStream_t s) {
  const bool covered = column_axis ? (srows >= lrows && scols * (size_t)slots >= lcols)
                                   : (scols >= lcols && srows * (size_t)slots >= lrows);
  if (lrows * lcols && !covered) cudaMemsetAsync(out, 0, lrows * lcols * sizeof(int32_t), s);
  if (srows * scols == 0) return cudaGetLastError();
  k_uncompress_u64<<<grid_rows(scols, srows), 256, 0, s>>>(w, srows, scols, lrows, lcols, t, e, slots, reversed,
                                                            column_axis, p, out, overflow);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_and_compress_u64(const uint64_t* w, size_t rows, size_t cols, size_t ldw, int t, int d, int e,
                                           uint32_t p, uint64_t* out, size_t ldo, cudaStream_t s) {
  const size_t count = rows * ((cols + e - 1) / e);
  if (count == 0) return cudaSuccess;
  k_reduce_and_compress_u64<<<blocks_for(count), 256, 0, s>>>(w, rows, cols, ldw, t, d, e, p, out, ldo);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_uncompress_full_u64(const uint64_t* cc, size_t ldcc, size_t m, size_t n, int t, int qs, int ts,
                                       uint32_t p, int32_t* c, size_t ldc, cudaStream_t s) {
  if (m * n == 0) return cudaSuccess;
  k_uncompress_full_u64<<<grid_rows(n, m), 256, 0, s>>>(cc, ldcc, m, n, t, qs, ts, p, c, ldc);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qgk
