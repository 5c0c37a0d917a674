// qg_pack.cu — HBM-bound kernels: seeded residue generation (K0), the four
// packings (K1-K3 + outer rows), REDQ, digit scatter (uncompress, K6) and the
// common-entry reduction. Each thread produces whole words, so every output
// store is a coalesced 8-byte write; input residues are read once.
#include <type_traits>
#include "qg_kernels.h"
#include "qg_device.cuh"

namespace qgk {

// K0: random_residue_matrix, prng.hpp:31-38 — element (r, c) of the matrix is
// SplitMix64 output number r*cols + c, reduced mod p (prng.hpp:25). The
// 64-bit `%` is emulated in software on the GPU (26 % of HBM speed, r1); it is
// replaced by an exact Barrett reduction: with magic = floor((2^64-1)/p),
// q = mulhi(x, magic) is floor(x/p) or one less (x magic / 2^64 > x/p - 1), so
// x - q p lies in [0, 2p) and one conditional subtraction gives x mod p.
template <typename TOut>
__global__ void k_gen_residues(uint64_t seed, uint32_t p, uint64_t magic, size_t row0, size_t rows, size_t cols,
                               TOut* __restrict__ dst) {
  const size_t total = rows * cols;
  const size_t base = row0 * cols;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < total;
       i += (size_t)gridDim.x * blockDim.x) {
    const uint64_t x = splitmix64_at(seed, base + i);
    uint64_t r = x - __umul64hi(x, magic) * p;
    if (r >= p) r -= p;
    store_residue(dst + i, (uint32_t)r);
  }
}

// Panel geometry of the common dimension: k residues split into panels of
// panel_len (the last may be short), each packed on its own into
// ceil(len/e) words and stored at a stride of panel_words (>= those words;
// the padding words are zero). One panel of length k is the plain layout;
// several reproduce blocked_accumulate's per-panel packing (gemm.hpp:460-478).
struct Panels {
  size_t k, panel_len;
  unsigned panel_words, npanels;
  __device__ __forceinline__ bool locate(unsigned gw_all, int e, size_t* base, int* len) const {
    const unsigned pi = gw_all / panel_words, gw = gw_all - pi * panel_words;
    const size_t pstart = (size_t)pi * panel_len;
    const size_t plen = (k - pstart) < panel_len ? (k - pstart) : panel_len;
    const size_t words = (plen + e - 1) / e;
    if (gw >= words) return false;
    *base = pstart + (size_t)gw * e;
    const size_t rem = pstart + plen - *base;
    *len = (int)(rem < (size_t)e ? rem : (size_t)e);
    return true;
  }
};

// A packed word in the backend's representation: DoubleWord (an exact double)
// or Int64Word (the uint64 itself), word.hpp:10-54.
__device__ __forceinline__ void store_word(double* p, uint64_t r) { *p = __ull2double_rn(r); }
__device__ __forceinline__ void store_word(uint64_t* p, uint64_t r) { *p = r; }

// K1: compress_rows_reversed, gemm.hpp:104-118 + compress_reverse,
// pack.hpp:59-70. Word (i, g) = sum_s a[i][g e + s] Q^(d - s); a short final
// group is shifted up by Q^(e - len).
template <typename TIn, typename TOut>
__global__ void k_pack_rows_reversed(const TIn* __restrict__ a, size_t m, size_t lda, int t, int e,
                                     Panels pn, TOut* __restrict__ ca, size_t ldca) {
  const unsigned W = pn.panel_words * pn.npanels;
  for (size_t i = blockIdx.y; i < m; i += gridDim.y) {
    const TIn* row = a + i * lda;
    for (unsigned g = blockIdx.x * blockDim.x + threadIdx.x; g < W; g += gridDim.x * blockDim.x) {
      size_t base;
      int len;
      uint64_t r = 0;
      if (pn.locate(g, e, &base, &len)) {
        for (int s = 0; s < len; ++s) r = (r << t) | residue_bits(row[base + s]);
        r <<= t * (e - len);
      }
      store_word(ca + i * ldca + g, r);
    }
  }
}

// K2: compress_cols_forward, gemm.hpp:122-140 + compress_forward,
// pack.hpp:47-54. Word (g, j) = sum_s b[g e + s][j] Q^s; lanes run along j so
// every load and store is coalesced.
template <typename TIn, typename TOut>
__global__ void k_pack_cols_forward(const TIn* __restrict__ b, size_t n, size_t ldb, int t, int e,
                                    Panels pn, TOut* __restrict__ cb, size_t ldcb) {
  const unsigned W = pn.panel_words * pn.npanels;
  for (unsigned g = blockIdx.y; g < W; g += gridDim.y) {
    size_t base;
    int len;
    const bool live = pn.locate(g, e, &base, &len);
    for (size_t j = blockIdx.x * (size_t)blockDim.x + threadIdx.x; j < n;
         j += (size_t)gridDim.x * blockDim.x) {
      uint64_t r = 0;
      if (live)
        for (int s = len - 1; s >= 0; --s) r = (r << t) | residue_bits(b[(base + s) * ldb + j]);
      store_word(cb + g * ldcb + j, r);
    }
  }
}

// K3: compress_outer_cols, gemm.hpp:145-158: word (i, h) = sum_s b[i][h e + s] Q^s.
template <typename TIn, typename TOut>
__global__ void k_pack_outer_cols(const TIn* __restrict__ b, size_t rows, size_t cols, size_t ldb,
                                  int t, int e, TOut* __restrict__ cb, size_t ldcb) {
  const size_t H = (cols + e - 1) / e;
  for (size_t i = blockIdx.y; i < rows; i += gridDim.y) {
    const TIn* row = b + i * ldb;
    for (size_t h = blockIdx.x * (size_t)blockDim.x + threadIdx.x; h < H;
         h += (size_t)gridDim.x * blockDim.x) {
      const size_t base = h * e;
      const int len = (int)((cols - base) < (size_t)e ? (cols - base) : (size_t)e);
      uint64_t r = 0;
      for (int s = len - 1; s >= 0; --s) r = (r << t) | residue_bits(row[base + s]);
      store_word(cb + i * ldcb + h, r);
    }
  }
}

// Tiled packings for the v4 contraction (qg_dot.cu, k_gemm_tiled): the same
// words as K1 / K2, stored as dense zero-padded 128 x BK blocks so that one
// pipeline stage of the contraction is one contiguous chunk per operand.
//   CA_t[tm][kt][r][c] = CA[128 tm + r][BK kt + c]   (compress_rows_reversed words)
//   CB_t[tn][kt][r][c] = CB[BK kt + c][128 tn + r]   (compress_cols_forward words, transposed)
// Balanced digits (qg_gpu_plan.balanced): residue v enters as v - p when
// v > p/2, so the words are signed integers (exact in double).
__device__ __forceinline__ long long balanced_digit(uint64_t v, uint32_t p) {
  return v > (p >> 1) ? (long long)v - (long long)p : (long long)v;
}

template <typename TIn, int BK, bool BAL>
__global__ void k_pack_a_tiled(const TIn* __restrict__ a, size_t m, size_t k, size_t lda, int t, int e,
                               unsigned Kt, size_t total, double* __restrict__ ca_t, uint32_t p) {
  const size_t K = (k + e - 1) / e;
  // 32-bit index arithmetic (the host keeps total < 2^32 on this path): a
  // 64-bit division by the runtime Kt per word cost more than the loads
  const unsigned tot = (unsigned)total;
  for (unsigned idx = blockIdx.x * blockDim.x + threadIdx.x; idx < tot; idx += gridDim.x * blockDim.x) {
    const unsigned c = idx % BK;
    const unsigned rest = idx / BK;
    const unsigned r = rest & 127;
    const unsigned rest2 = rest >> 7;
    const unsigned kt = rest2 % Kt, tm = rest2 / Kt;
    const size_t row = (size_t)tm * 128 + r, gw = (size_t)kt * BK + c;
    if (BAL) {
      long long w = 0;
      if (row < m && gw < K) {
        const size_t base = gw * e;
        const int len = (int)((k - base) < (size_t)e ? (k - base) : (size_t)e);
        const TIn* src = a + row * lda + base;
        for (int s = 0; s < len; ++s) w = w * (1ll << t) + balanced_digit(residue_bits(src[s]), p);
        w *= 1ll << (t * (e - len));
      }
      ca_t[idx] = __ll2double_rn(w);
    } else {
      uint64_t w = 0;
      if (row < m && gw < K) {
        const size_t base = gw * e;
        const int len = (int)((k - base) < (size_t)e ? (k - base) : (size_t)e);
        const TIn* src = a + row * lda + base;
        for (int s = 0; s < len; ++s) w = (w << t) | residue_bits(src[s]);
        w <<= t * (e - len);
      }
      ca_t[idx] = __ull2double_rn(w);
    }
  }
}

// compress_cols_forward (gemm.hpp:122-140) words in the tiled transposed
// layout: CB_t[tn][kt][r][c] = word (BK kt + c) of column 128 tn + r. One CTA
// per 32 columns x 16 consecutive words (thousands of CTAs, so no partial last
// wave): lane = column (each residue load is a coalesced 256-byte row
// segment), the 8 warps split the 16 words; the 32 x 16 words then leave
// through shared memory as 128-byte row runs of the output blocks. The grid
// covers the zero padding of the layout too.
template <typename TIn, int BK, bool BAL>
__global__ void __launch_bounds__(256) k_pack_b_tiled(const TIn* __restrict__ b, size_t k, size_t n, size_t ldb,
                                                      int t, int e, unsigned Kt, double* __restrict__ cb_t,
                                                      uint32_t p) {
  __shared__ double tile[32][17];
  const size_t K = (k + e - 1) / e;
  const size_t w0 = (size_t)blockIdx.x * 16, n0 = (size_t)blockIdx.y * 32;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const size_t col = n0 + lane;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int cl = warp + 8 * h;
    const size_t gw = w0 + cl;
    double wd;
    if (BAL) {
      long long w = 0;
      if (col < n && gw < K) {
        const size_t base = gw * e;
        const int len = (int)((k - base) < (size_t)e ? (k - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = w * (1ll << t) + balanced_digit(residue_bits(b[(base + s) * ldb + col]), p);
      }
      wd = __ll2double_rn(w);
    } else {
      uint64_t w = 0;
      if (col < n && gw < K) {
        const size_t base = gw * e;
        const int len = (int)((k - base) < (size_t)e ? (k - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = (w << t) | residue_bits(b[(base + s) * ldb + col]);
      }
      wd = __ull2double_rn(w);
    }
    tile[lane][cl] = wd;
  }
  __syncthreads();
  const size_t Wpad = (size_t)Kt * BK;
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int i = threadIdx.x + 256 * h;
    const int r = i >> 4, cl = i & 15;
    const size_t nn = n0 + r, w = w0 + cl;
    if (w < Wpad) {
      const size_t kt = w / BK, c = w % BK;
      cb_t[(((nn >> 7) * Kt + kt) * 128 + (nn & 127)) * BK + c] = tile[r][cl];
    }
  }
}

// compress_outer_cols (gemm.hpp:145-158) words in the tiled transposed layout
// of the mixed-variant contraction: CBo_t[tn][kt][r][c] = word (row BK kt + c,
// group 128 tn + r) = sum_s B[BK kt + c][(128 tn + r) e + s] Q^s.
template <typename TIn, int BK, bool BAL = false>
__global__ void __launch_bounds__(256) k_pack_outer_tiled(const TIn* __restrict__ b, size_t k, size_t n, size_t ldb,
                                                          int t, int e, unsigned Kt, double* __restrict__ bo_t,
                                                          uint32_t p = 0) {
  __shared__ double tile[64 * (BK + 1)];
  const size_t H = (n + e - 1) / e;
  const size_t blk = blockIdx.x >> 1, half = blockIdx.x & 1;
  const size_t kt = blk % Kt, tn = blk / Kt;
  const int r = threadIdx.x & 63, cg = threadIdx.x >> 6;
  const size_t hcol = tn * 128 + half * 64 + r;
  for (int c = cg; c < BK; c += 4) {
    const size_t l = kt * BK + c;
    double wd;
    if (BAL) {  // balanced digits (v - p for v > p/2): a signed word, exact in double
      long long w = 0;
      if (hcol < H && l < k) {
        const size_t base = hcol * e;
        const int len = (int)((n - base) < (size_t)e ? (n - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = w * (1ll << t) + balanced_digit(residue_bits(b[l * ldb + base + s]), p);
      }
      wd = __ll2double_rn(w);
    } else {
      uint64_t w = 0;
      if (hcol < H && l < k) {
        const size_t base = hcol * e;
        const int len = (int)((n - base) < (size_t)e ? (n - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = (w << t) | residue_bits(b[l * ldb + base + s]);
      }
      wd = __ull2double_rn(w);
    }
    tile[r * (BK + 1) + c] = wd;
  }
  __syncthreads();
  double* out = bo_t + blk * (size_t)(128 * BK) + half * (size_t)(64 * BK);
  for (int i = threadIdx.x; i < 64 * BK; i += 256) out[i] = tile[(i / BK) * (BK + 1) + i % BK];
}

template <typename TIn, int BK, bool BAL = false>
static cudaError_t pack_outer_tiled_t(const TIn* src, size_t k, size_t n, size_t ld, int t, int e, double* dst,
                                      cudaStream_t s, uint32_t p = 0) {
  const size_t H = (n + e - 1) / e;
  const unsigned Kt = (unsigned)((k + BK - 1) / BK);
  const size_t Nt = (H + 127) / 128;
  if (Kt == 0 || Nt == 0) return cudaSuccess;
  k_pack_outer_tiled<TIn, BK, BAL><<<(unsigned)(Nt * Kt * 2), 256, 0, s>>>(src, k, n, ld, t, e, Kt, dst, p);
  count_launch();
  return cudaGetLastError();
}

template <typename TIn, bool BAL = false>
static cudaError_t pack_outer_tiled_dt(const TIn* src, size_t k, size_t n, size_t ld, int t, int e, int bk,
                                       double* dst, cudaStream_t s, uint32_t p = 0) {
  switch (bk) {
    case 36: return pack_outer_tiled_t<TIn, 36, BAL>(src, k, n, ld, t, e, dst, s, p);
    case 28: return pack_outer_tiled_t<TIn, 28, BAL>(src, k, n, ld, t, e, dst, s, p);
    case 20: return pack_outer_tiled_t<TIn, 20, BAL>(src, k, n, ld, t, e, dst, s, p);
    case 12: return pack_outer_tiled_t<TIn, 12, BAL>(src, k, n, ld, t, e, dst, s, p);
    case 4: return pack_outer_tiled_t<TIn, 4, BAL>(src, k, n, ld, t, e, dst, s, p);
  }
  return cudaErrorInvalidValue;
}

// compress_outer_rows into the tiled A layout, gemm.hpp:160-176: word (g, l)
// = sum_s A[g e + s][l] Q^s (forward along m), stored in dense 128 x BK
// blocks [g-tile][k-tile][g][l]. One CTA per block; consecutive threads run
// along l, so each run of BK reads is one contiguous row segment and the
// block is written contiguously.
template <typename TIn, int BK, bool BAL = false>
__global__ void __launch_bounds__(256) k_pack_outer_rows_tiled(const TIn* __restrict__ a, size_t m, size_t k,
                                                               size_t lda, int t, int e, unsigned Kt,
                                                               double* __restrict__ ao_t, uint32_t p = 0) {
  const size_t G = (m + e - 1) / e;
  const unsigned kt = blockIdx.x % Kt, tg = blockIdx.x / Kt;
  double* out = ao_t + (size_t)blockIdx.x * (128 * BK);
  for (unsigned idx = threadIdx.x; idx < 128 * BK; idx += 256) {
    const unsigned r = idx / BK, c = idx % BK;
    const size_t g = (size_t)tg * 128 + r, l = (size_t)kt * BK + c;
    if (BAL) {  // balanced digits: a signed word
      long long w = 0;
      if (g < G && l < k) {
        const size_t base = g * e;
        const int len = (int)((m - base) < (size_t)e ? (m - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = w * (1ll << t) + balanced_digit(residue_bits(a[(base + s) * lda + l]), p);
      }
      out[idx] = __ll2double_rn(w);
    } else {
      uint64_t w = 0;
      if (g < G && l < k) {
        const size_t base = g * e;
        const int len = (int)((m - base) < (size_t)e ? (m - base) : (size_t)e);
        for (int s = len - 1; s >= 0; --s) w = (w << t) | residue_bits(a[(base + s) * lda + l]);
      }
      out[idx] = __ull2double_rn(w);
    }
  }
}

// The unpack of mul_full_compressed, gemm.hpp:427-443: output cell
// (g qs + i, h ts + j) is base-Q digit i + j qs of word (g, h). One thread per
// (output row, word column): it reads the word once and writes its ts
// consecutive cells, so a warp's stores cover one contiguous row segment.
// 32-bit index arithmetic only (rows and words per row < 2^31). Like the
// reference (which masks, gemm.hpp:436-441) there is no range check, so the
// call stays asynchronous.
__global__ void k_uncompress_full(const double* __restrict__ cc, size_t ldcc, unsigned m, unsigned n, int t,
                                  int qs, int ts, uint32_t p, uint32_t magic, int32_t* __restrict__ c, size_t ldc) {
  // one thread per word (g, h): the word is read once and its qs x ts digits
  // go to rows g qs + i, columns h ts + j (digit i + j qs)
  const uint64_t mask = (1ull << t) - 1;
  const unsigned H = (n + ts - 1) / ts, G = (m + qs - 1) / qs;
  const bool pair2 = ts == 2 && t <= 31 && (ldc % 2) == 0 && (reinterpret_cast<uintptr_t>(c) & 7) == 0;
  for (unsigned g = blockIdx.y; g < G; g += gridDim.y) {
    const double* wrow = cc + (size_t)g * ldcc;
    for (unsigned h = blockIdx.x * blockDim.x + threadIdx.x; h < H; h += gridDim.x * blockDim.x) {
      const uint64_t bits = __double2ull_rz(wrow[h]);
      const unsigned col0 = h * ts;
      if (pair2 && col0 + 2 <= n) {  // two columns per word: one 8-byte store per row
        for (int i = 0; i < qs && g * qs + i < m; ++i) {
          const uint32_t x0 = (uint32_t)((bits >> (t * i)) & mask), x1 = (uint32_t)((bits >> (t * (i + qs))) & mask);
          const uint32_t r0 = x0 - __umulhi(x0, magic) * p, r1 = x1 - __umulhi(x1, magic) * p;
          *reinterpret_cast<int2*>(c + (size_t)(g * qs + i) * ldc + col0) =
              make_int2((int)(r0 >= p ? r0 - p : r0), (int)(r1 >= p ? r1 - p : r1));
        }
        continue;
      }
      for (int i = 0; i < qs && g * qs + i < m; ++i) {
        int32_t* crow = c + (size_t)(g * qs + i) * ldc;
        for (int j = 0; j < ts && col0 + j < n; ++j) {
          const uint64_t x64 = (bits >> (t * (i + j * qs))) & mask;
          uint32_t r;
          if (t > 31) {
            r = (uint32_t)(x64 % p);  // one-digit words of a wide radix
          } else {
            const uint32_t x = (uint32_t)x64;
            r = x - __umulhi(x, magic) * p;
            r = r >= p ? r - p : r;
          }
          crow[col0 + j] = (int32_t)r;
        }
      }
    }
  }
}

// extract_coefficient (DoubleWord), pack.hpp:78-100, bit for bit on any word:
// ReciprocalMul truncates w * inv_qd (an exact power-of-two scale) to int64
// with the reference's x86 conversion (out of range or NaN -> INT64_MIN);
// AddHighBits adds Q^(2d+1) (round to nearest) and reads the digit from the
// mantissa at bit 52 - t e (shift count taken mod 64, as x86 does).
__device__ __forceinline__ uint32_t extract_coefficient_dev(double w, int t, int d, int e, double inv_qd, int mode,
                                                            uint64_t qmask, uint32_t p) {
  uint64_t digit;
  if (mode == 1) {
    const double anchor = ldexp(1.0, t * (2 * d + 1));
    const uint64_t mant = (uint64_t)__double_as_longlong(__dadd_rn(w, anchor)) & ((1ull << 52) - 1);
    digit = (mant >> ((52 - t * e) & 63)) & qmask;
  } else {
    const double high = __dmul_rn(w, inv_qd);
    const long long v = (high >= -9223372036854775808.0 && high < 9223372036854775808.0)
                            ? __double2ll_rz(high)
                            : (long long)0x8000000000000000ull;
    digit = (uint64_t)v & qmask;
  }
  return (uint32_t)(digit % p);
}

__global__ void k_extract_coefficients(const double* __restrict__ w, size_t count, int t, int d, int e,
                                       double inv_qd, int mode, uint32_t p, int32_t* __restrict__ out) {
  const uint64_t qmask = t >= 64 ? ~0ull : (1ull << t) - 1;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)extract_coefficient_dev(w[i], t, d, e, inv_qd, mode, qmask, p);
}

// reduce_and_compress, pack.hpp:141-155, on every row of a words matrix: each
// group of e consecutive entries is extracted and packed forward into one word
// (the last group zero-padded). One thread per output word.
__global__ void k_reduce_and_compress(const double* __restrict__ w, size_t rows, size_t cols, size_t ldw, int t,
                                      int d, int e, double inv_qd, int mode, uint32_t p, double* __restrict__ out,
                                      size_t ldo) {
  const uint64_t qmask = t >= 64 ? ~0ull : (1ull << t) - 1;
  const size_t groups = (cols + e - 1) / e, count = rows * groups;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count; i += (size_t)gridDim.x * blockDim.x) {
    const size_t r = i / groups, g = i % groups;
    const size_t c0 = g * e;
    const int len = (int)((cols - c0) < (size_t)e ? (cols - c0) : (size_t)e);
    uint64_t word = 0;
    for (int s = len - 1; s >= 0; --s)
      word = (word << t) | extract_coefficient_dev(w[r * ldw + c0 + s], t, d, e, inv_qd, mode, qmask, p);
    out[r * ldo + g] = __ull2double_rn(word);
  }
}

static unsigned grid1d(size_t work, int threads);

cudaError_t launch_extract_coefficients(const double* w, size_t count, int t, int d, int e, double inv_qd, int mode,
                                        uint32_t p, int32_t* out, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_extract_coefficients<<<grid1d(count, 256), 256, 0, s>>>(w, count, t, d, e, inv_qd, mode, p, out);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_and_compress(const double* w, size_t rows, size_t cols, size_t ldw, int t, int d, int e,
                                       double inv_qd, int mode, uint32_t p, double* out, size_t ldo, cudaStream_t s) {
  const size_t count = rows * ((cols + e - 1) / e);
  if (count == 0) return cudaSuccess;
  k_reduce_and_compress<<<grid1d(count, 256), 256, 0, s>>>(w, rows, cols, ldw, t, d, e, inv_qd, mode, p, out, ldo);
  count_launch();
  return cudaGetLastError();
}

// naive_gemm, gemm.hpp:80-100, on the device: the independent checker behind
// the CLI's verify and --algo naive. 16 x 16 output tiles, 64-bit sums of
// products reduced mod p every `spill` products so they never wrap.
__global__ void __launch_bounds__(256) k_naive_gemm(const uint32_t* __restrict__ a, const uint32_t* __restrict__ b,
                                                    unsigned m, unsigned k, unsigned n, uint32_t p, unsigned spill,
                                                    int32_t* __restrict__ c, size_t ldc) {
  __shared__ uint32_t sa[16][17], sb[16][17];
  const unsigned tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const unsigned row = blockIdx.y * 16 + ty, col = blockIdx.x * 16 + tx;
  uint64_t acc = 0;
  unsigned cnt = 0;
  for (unsigned k0 = 0; k0 < k; k0 += 16) {
    sa[ty][tx] = (row < m && k0 + tx < k) ? a[(size_t)row * k + k0 + tx] : 0u;
    sb[ty][tx] = (k0 + ty < k && col < n) ? b[(size_t)(k0 + ty) * n + col] : 0u;
    __syncthreads();
#pragma unroll
    for (int l = 0; l < 16; ++l) {
      acc += (uint64_t)sa[ty][l] * sb[l][tx];
      if (++cnt == spill) {
        acc %= p;
        cnt = 0;
      }
    }
    __syncthreads();
  }
  if (row < m && col < n) c[(size_t)row * ldc + col] = (int32_t)(acc % p);
}

cudaError_t launch_naive_gemm(const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n, uint32_t p,
                              int32_t* c, size_t ldc, cudaStream_t s) {
  if (m * n == 0) return cudaSuccess;
  if (m > 0xFFFF0ull || n >= (1ull << 31) || k >= (1ull << 32)) return cudaErrorInvalidValue;
  const unsigned __int128 pm = (unsigned __int128)(p - 1) * (p - 1);
  unsigned __int128 room = ((unsigned __int128)1 << 64) - 1 - (p - 1);
  unsigned __int128 sp = pm ? room / pm : ((unsigned __int128)1 << 31);
  const unsigned spill = sp > (1u << 31) ? (1u << 31) : (unsigned)sp;
  const dim3 grid((unsigned)((n + 15) / 16), (unsigned)((m + 15) / 16));
  k_naive_gemm<<<grid, 256, 0, s>>>(a, b, (unsigned)m, (unsigned)k, (unsigned)n, p, spill ? spill : 1, c, ldc);
  count_launch();
  return cudaGetLastError();
}

// redq over a buffer, pack.hpp:124-137: every base-Q digit replaced by itself
// mod p. A word outside [0, 2^(t e)) raises the DigitOverflow flag.
__device__ __forceinline__ uint32_t digit_mod(uint64_t x, int t, uint32_t p, uint32_t magic) {
  if (t > 31) return (uint32_t)(x % p);  // one wide digit (e = 1 plans)
  const uint32_t x32 = (uint32_t)x;
  const uint32_t r = x32 - __umulhi(x32, magic) * p;
  return min(r, r - p);
}

__global__ void k_redq(double* __restrict__ w, size_t count, int t, int e, uint32_t p, uint32_t magic,
                       int* __restrict__ overflow) {
  const int total_bits = t * e;
  const double limit = (double)(1ull << total_bits);
  const uint64_t mask = t >= 64 ? ~0ull : (1ull << t) - 1;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  // four words per thread per round, loads first: four loads in flight
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < count; i0 += 4 * stride) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * stride < count ? w[i0 + u * stride] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= count) break;
      if (!(v[u] >= 0.0) || !(v[u] < limit)) {
        atomicExch(overflow, 1);
        continue;
      }
      const uint64_t bits = __double2ull_rz(v[u]);
      uint64_t r = 0;
      for (int s = 0; s < total_bits; s += t) r |= (uint64_t)digit_mod((bits >> s) & mask, t, p, magic) << s;
      w[i] = __ull2double_rn(r);
    }
  }
}

// uncompress of column-axis words (CC, CB^T-style rows) with e = 4 or 2 slots
// per word and whole words per row: each word's digits leave as one 16- or
// 8-byte vector store (coalesced across the warp), four words per thread
// per round with their loads issued first
template <int SL>
__global__ void k_uncompress_cols_vec(const double* __restrict__ w, size_t srows, size_t scols, int t, int reversed,
                                      uint32_t p, uint32_t magic, int32_t* __restrict__ out,
                                      int* __restrict__ overflow) {
  const double limit = (double)(1ull << (t * SL));
  const uint64_t mask = (1ull << t) - 1;
  const size_t count = srows * scols, stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i0 = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i0 < count; i0 += 4 * stride) {
    double v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) v[u] = i0 + u * stride < count ? w[i0 + u * stride] : 0.0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const size_t i = i0 + u * stride;
      if (i >= count) break;
      if (!(v[u] >= 0.0) || !(v[u] < limit)) {
        atomicExch(overflow, 1);
        continue;
      }
      const uint64_t bits = __double2ull_rz(v[u]);
      int32_t d[SL];
#pragma unroll
      for (int s = 0; s < SL; ++s) {
        const int di = reversed ? SL - 1 - s : s;
        d[s] = (int32_t)digit_mod((bits >> (t * di)) & mask, t, p, magic);
      }
      // word (si, sj) -> out[si][sj * SL .. + SL): the flat word index i times SL
      if (SL == 4)
        reinterpret_cast<int4*>(out)[i] = make_int4(d[0], d[1], d[2], d[SL - 1]);
      else
        reinterpret_cast<int2*>(out)[i] = make_int2(d[0], d[SL - 1]);
    }
  }
}

__global__ void k_uncompress(const double* __restrict__ w, size_t srows, size_t scols,
                             size_t lrows, size_t lcols, int t, int e, int slots, int reversed,
                             int column_axis, uint32_t p, uint32_t magic, int32_t* __restrict__ out,
                             int* __restrict__ overflow) {
  const int total_bits = t * e;
  const double limit = (double)(1ull << total_bits);
  const uint64_t mask = t >= 64 ? ~0ull : (1ull << t) - 1;
  for (size_t si = blockIdx.y; si < srows; si += gridDim.y) {
    for (size_t sj = blockIdx.x * (size_t)blockDim.x + threadIdx.x; sj < scols; sj += (size_t)gridDim.x * blockDim.x) {
      const double v = w[si * scols + sj];
      if (!(v >= 0.0) || !(v < limit)) {
        atomicExch(overflow, 1);
        continue;
      }
      const uint64_t bits = __double2ull_rz(v);
      for (int s = 0; s < slots; ++s) {
        const int di = reversed ? slots - 1 - s : s;
        const uint64_t digit = di < e ? (bits >> (t * di)) & mask : 0;
        size_t i = si, j = sj;
        if (column_axis) j = sj * slots + s;
        else i = si * slots + s;
        if (i < lrows && j < lcols) out[i * lcols + j] = (int32_t)digit_mod(digit, t, p, magic);
      }
    }
  }
}

// reduce_common_entry over a buffer, gemm.hpp:247-250.
__global__ void k_reduce_common(const double* __restrict__ acc, size_t count, uint32_t qmask,
                                uint32_t p, int32_t* __restrict__ c) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < count;
       i += (size_t)gridDim.x * blockDim.x)
    c[i] = (int32_t)(((uint32_t)(__double2ull_rz(acc[i]) & qmask)) % p);
}

// ---------------------------------------------------------------- launchers
static unsigned grid1d(size_t work, int threads) {
  size_t blocks = (work + threads - 1) / threads;
  const size_t cap = 148 * 16;
  if (blocks > cap) blocks = cap;
  return (unsigned)(blocks ? blocks : 1);
}

// panel_len 0 = one panel of the whole dimension; panel_words 0 = unpadded.
static Panels make_panels(size_t k, int e, size_t panel_len, size_t panel_words) {
  Panels pn;
  pn.k = k;
  pn.panel_len = (panel_len == 0 || panel_len > k) ? k : panel_len;
  if (pn.panel_len == 0) pn.panel_len = 1;
  const size_t words = (pn.panel_len + e - 1) / e;
  pn.panel_words = (unsigned)(panel_words ? panel_words : words);
  pn.npanels = (unsigned)((k + pn.panel_len - 1) / pn.panel_len);
  return pn;
}

static dim3 grid2d(size_t inner, size_t outer, int threads) {
  size_t bx = (inner + threads - 1) / threads;
  if (bx < 1) bx = 1;
  if (bx > 65535) bx = 65535;
  size_t by = outer < 65535 ? outer : 65535;
  if (by < 1) by = 1;
  return dim3((unsigned)bx, (unsigned)by);
}

cudaError_t launch_gen_residues(uint64_t seed, uint32_t p, size_t row0, size_t rows, size_t cols,
                                void* dst, int dtype, cudaStream_t s) {
  const size_t total = rows * cols;
  if (total == 0) return cudaSuccess;
  if (p == 0) return cudaErrorInvalidValue;
  const uint64_t magic = ~0ull / p;
  if (dtype == 0)
    k_gen_residues<double><<<grid1d(total, 256), 256, 0, s>>>(seed, p, magic, row0, rows, cols, (double*)dst);
  else
    k_gen_residues<uint32_t><<<grid1d(total, 256), 256, 0, s>>>(seed, p, magic, row0, rows, cols, (uint32_t*)dst);
  count_launch();
  return cudaGetLastError();
}

template <typename TIn, typename TOut>
static cudaError_t pack_dispatch(int kind, const TIn* src, size_t rows, size_t cols, size_t ld,
                                 int t, int e, TOut* dst, size_t ldd, size_t panel_len,
                                 size_t panel_words, cudaStream_t s) {
  if (rows == 0 || cols == 0) return cudaSuccess;
  switch (kind) {
    case PACK_ROWS_REVERSED: {  // common dimension = cols
      const Panels pn = make_panels(cols, e, panel_len, panel_words);
      k_pack_rows_reversed<TIn, TOut><<<grid2d((size_t)pn.panel_words * pn.npanels, rows, 128), 128, 0, s>>>(
          src, rows, ld, t, e, pn, dst, ldd);
      break;
    }
    case PACK_COLS_FORWARD: {  // common dimension = rows
      const Panels pn = make_panels(rows, e, panel_len, panel_words);
      k_pack_cols_forward<TIn, TOut><<<grid2d(cols, (size_t)pn.panel_words * pn.npanels, 128), 128, 0, s>>>(
          src, cols, ld, t, e, pn, dst, ldd);
      break;
    }
    case PACK_OUTER_COLS: {
      const size_t H = (cols + e - 1) / e;
      k_pack_outer_cols<TIn, TOut><<<grid2d(H, rows, 128), 128, 0, s>>>(src, rows, cols, ld, t, e, dst, ldd);
      break;
    }
    case PACK_OUTER_ROWS: {  // compress_outer_rows, gemm.hpp:161-178: forward words down columns
      const Panels pn = make_panels(rows, e, rows, 0);
      k_pack_cols_forward<TIn, TOut><<<grid2d(cols, (size_t)pn.panel_words, 128), 128, 0, s>>>(
          src, cols, ld, t, e, pn, dst, ldd);
      break;
    }
  }
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_pack(int kind, const void* src, int dtype, size_t rows, size_t cols, size_t ld,
                        int t, int e, double* dst, size_t ldd, size_t panel_len,
                        size_t panel_words, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_dispatch<double>(kind, (const double*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
    case 1: return pack_dispatch<uint32_t>(kind, (const uint32_t*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
    default: return pack_dispatch<int32_t>(kind, (const int32_t*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
  }
}

// The same four packings into Int64Word (uint64) words.
cudaError_t launch_pack_u64(int kind, const void* src, int dtype, size_t rows, size_t cols, size_t ld, int t, int e,
                            uint64_t* dst, size_t ldd, size_t panel_len, size_t panel_words, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_dispatch<double>(kind, (const double*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
    case 1: return pack_dispatch<uint32_t>(kind, (const uint32_t*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
    default: return pack_dispatch<int32_t>(kind, (const int32_t*)src, rows, cols, ld, t, e, dst, ldd, panel_len, panel_words, s);
  }
}


template <typename TIn, int BK, bool BAL>
static cudaError_t pack_tiled_t(bool b_operand, const TIn* src, size_t rows, size_t cols, size_t ld, int t,
                                int e, double* dst, cudaStream_t s, uint32_t p) {
  if (b_operand) {  // src is k x n; blocks over (n, k-words)
    const size_t K = (rows + e - 1) / e;
    const unsigned Kt = (unsigned)((K + BK - 1) / BK);
    const size_t Nt = (cols + 127) / 128;
    if (Kt == 0 || Nt == 0) return cudaSuccess;
    const dim3 grid((unsigned)(((size_t)Kt * BK + 15) / 16), (unsigned)(Nt * 4));
    if (grid.y > 65535) return cudaErrorInvalidValue;
    k_pack_b_tiled<TIn, BK, BAL><<<grid, 256, 0, s>>>(src, rows, cols, ld, t, e, Kt, dst, p);
  } else {  // src is m x k
    const size_t K = (cols + e - 1) / e;
    const unsigned Kt = (unsigned)((K + BK - 1) / BK);
    const size_t Mt = (rows + 127) / 128;
    const size_t total = Mt * Kt * 128 * (size_t)BK;
    if (total == 0) return cudaSuccess;
    if (total >= (size_t(1) << 32)) return cudaErrorInvalidValue;  // 32-bit word index (32 GiB of words)
    k_pack_a_tiled<TIn, BK, BAL><<<grid1d(total, 256), 256, 0, s>>>(src, rows, cols, ld, t, e, Kt, total, dst, p);
  }
  count_launch();
  return cudaGetLastError();
}

template <typename TIn, bool BAL>
static cudaError_t pack_tiled_bk(bool b_operand, const TIn* src, size_t rows, size_t cols, size_t ld, int t,
                                 int e, int bk, double* dst, cudaStream_t s, uint32_t p) {
  switch (bk) {
    case 52: return pack_tiled_t<TIn, 52, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 44: return pack_tiled_t<TIn, 44, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 36: return pack_tiled_t<TIn, 36, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 28: return pack_tiled_t<TIn, 28, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 20: return pack_tiled_t<TIn, 20, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 12: return pack_tiled_t<TIn, 12, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
    case 4: return pack_tiled_t<TIn, 4, BAL>(b_operand, src, rows, cols, ld, t, e, dst, s, p);
  }
  return cudaErrorInvalidValue;
}

template <typename TIn>
static cudaError_t pack_tiled_dt(bool b_operand, const TIn* src, size_t rows, size_t cols, size_t ld, int t,
                                 int e, int bk, double* dst, cudaStream_t s, uint32_t p, bool balanced) {
  return balanced ? pack_tiled_bk<TIn, true>(b_operand, src, rows, cols, ld, t, e, bk, dst, s, p)
                  : pack_tiled_bk<TIn, false>(b_operand, src, rows, cols, ld, t, e, bk, dst, s, p);
}

cudaError_t launch_pack_tiled(bool b_operand, const void* src, int dtype, size_t rows, size_t cols,
                              size_t ld, int t, int e, int bk, double* dst, cudaStream_t s, uint32_t p,
                              bool balanced) {
  switch (dtype) {
    case 0: return pack_tiled_dt<double>(b_operand, (const double*)src, rows, cols, ld, t, e, bk, dst, s, p, balanced);
    case 1: return pack_tiled_dt<uint32_t>(b_operand, (const uint32_t*)src, rows, cols, ld, t, e, bk, dst, s, p, balanced);
    default: return pack_tiled_dt<int32_t>(b_operand, (const int32_t*)src, rows, cols, ld, t, e, bk, dst, s, p, balanced);
  }
}

cudaError_t launch_pack_outer_tiled(const void* src, int dtype, size_t k, size_t n, size_t ld, int t, int e,
                                    int bk, double* dst, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_outer_tiled_dt<double>((const double*)src, k, n, ld, t, e, bk, dst, s);
    case 1: return pack_outer_tiled_dt<uint32_t>((const uint32_t*)src, k, n, ld, t, e, bk, dst, s);
    default: return pack_outer_tiled_dt<int32_t>((const int32_t*)src, k, n, ld, t, e, bk, dst, s);
  }
}

template <typename TIn, int BK, bool BAL = false>
static cudaError_t pack_outer_rows_tiled_t(const TIn* src, size_t m, size_t k, size_t ld, int t, int e, double* dst,
                                           cudaStream_t s, uint32_t p = 0) {
  const size_t G = (m + e - 1) / e;
  const unsigned Kt = (unsigned)((k + BK - 1) / BK);
  const size_t blocks = (G + 127) / 128 * Kt;
  if (blocks == 0) return cudaSuccess;
  if (blocks >= (1ull << 31)) return cudaErrorInvalidValue;
  k_pack_outer_rows_tiled<TIn, BK, BAL><<<(unsigned)blocks, 256, 0, s>>>(src, m, k, ld, t, e, Kt, dst, p);
  count_launch();
  return cudaGetLastError();
}

template <typename TIn, bool BAL = false>
static cudaError_t pack_outer_rows_tiled_dt(const TIn* src, size_t m, size_t k, size_t ld, int t, int e, int bk,
                                            double* dst, cudaStream_t s, uint32_t p = 0) {
  switch (bk) {
    case 36: return pack_outer_rows_tiled_t<TIn, 36, BAL>(src, m, k, ld, t, e, dst, s, p);
    case 28: return pack_outer_rows_tiled_t<TIn, 28, BAL>(src, m, k, ld, t, e, dst, s, p);
    case 20: return pack_outer_rows_tiled_t<TIn, 20, BAL>(src, m, k, ld, t, e, dst, s, p);
    case 12: return pack_outer_rows_tiled_t<TIn, 12, BAL>(src, m, k, ld, t, e, dst, s, p);
    case 4: return pack_outer_rows_tiled_t<TIn, 4, BAL>(src, m, k, ld, t, e, dst, s, p);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_pack_outer_rows_tiled(const void* src, int dtype, size_t m, size_t k, size_t ld, int t, int e,
                                         int bk, double* dst, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_outer_rows_tiled_dt<double>((const double*)src, m, k, ld, t, e, bk, dst, s);
    case 1: return pack_outer_rows_tiled_dt<uint32_t>((const uint32_t*)src, m, k, ld, t, e, bk, dst, s);
    default: return pack_outer_rows_tiled_dt<int32_t>((const int32_t*)src, m, k, ld, t, e, bk, dst, s);
  }
}

cudaError_t launch_pack_outer_tiled_bal(const void* src, int dtype, size_t k, size_t n, size_t ld, int t, int e, int bk,
                                        double* dst, uint32_t p, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_outer_tiled_dt<double, true>((const double*)src, k, n, ld, t, e, bk, dst, s, p);
    case 1: return pack_outer_tiled_dt<uint32_t, true>((const uint32_t*)src, k, n, ld, t, e, bk, dst, s, p);
    default: return pack_outer_tiled_dt<int32_t, true>((const int32_t*)src, k, n, ld, t, e, bk, dst, s, p);
  }
}

cudaError_t launch_pack_outer_rows_tiled_bal(const void* src, int dtype, size_t m, size_t k, size_t ld, int t, int e,
                                             int bk, double* dst, uint32_t p, cudaStream_t s) {
  switch (dtype) {
    case 0: return pack_outer_rows_tiled_dt<double, true>((const double*)src, m, k, ld, t, e, bk, dst, s, p);
    case 1: return pack_outer_rows_tiled_dt<uint32_t, true>((const uint32_t*)src, m, k, ld, t, e, bk, dst, s, p);
    default: return pack_outer_rows_tiled_dt<int32_t, true>((const int32_t*)src, m, k, ld, t, e, bk, dst, s, p);
  }
}

cudaError_t launch_uncompress_full(const double* cc, size_t ldcc, size_t m, size_t n, int t, int qs, int ts,
                                   uint32_t p, int32_t* c, size_t ldc, cudaStream_t s) {
  if (m * n == 0) return cudaSuccess;
  if (m >= (1u << 31) || n >= (1u << 31)) return cudaErrorInvalidValue;
  const unsigned H = (unsigned)((n + ts - 1) / ts);
  const size_t G = (m + qs - 1) / qs;
  const dim3 grid((H + 255) / 256, (unsigned)(G < 65535 ? G : 65535));
  k_uncompress_full<<<grid, 256, 0, s>>>(cc, ldcc, (unsigned)m, (unsigned)n, t, qs, ts, p,
                                         (uint32_t)(0x100000000ull / p), c, ldc);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_redq(double* w, size_t count, int t, int e, uint32_t p, int* overflow,
                        cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_redq<<<grid1d(count, 256), 256, 0, s>>>(w, count, t, e, p, (uint32_t)(0x100000000ull / p), overflow);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_uncompress(const double* w, size_t srows, size_t scols, size_t lrows,
                              size_t lcols, int t, int e, int slots, int reversed, int column_axis,
                              uint32_t p, int32_t* out, int* overflow, cudaStream_t s) {
  // zero only what no stored word covers (ResidueMatrix's zero fill)
  const bool covered = column_axis ? (srows >= lrows && scols * (size_t)slots >= lcols)
                                   : (scols >= lcols && srows * (size_t)slots >= lrows);
  if (lrows * lcols && !covered) cudaMemsetAsync(out, 0, lrows * lcols * sizeof(int32_t), s);
  const size_t count = srows * scols;
  if (count == 0) return cudaGetLastError();
  // whole words per row (lcols = scols * slots, lrows = srows), slots = e = 4 or 2,
  // 16 / 8-byte aligned output: vector stores
  if (column_axis && slots == e && (e == 4 || e == 2) && t <= 31 && lrows == srows && lcols == scols * (size_t)e &&
      (reinterpret_cast<uintptr_t>(out) % (4 * e)) == 0) {
    const uint32_t magic = (uint32_t)(0x100000000ull / p);
    if (e == 4)
      k_uncompress_cols_vec<4><<<grid1d(count, 256), 256, 0, s>>>(w, srows, scols, t, reversed, p, magic, out, overflow);
    else
      k_uncompress_cols_vec<2><<<grid1d(count, 256), 256, 0, s>>>(w, srows, scols, t, reversed, p, magic, out, overflow);
    count_launch();
    return cudaGetLastError();
  }
  const size_t gx = (scols + 255) / 256;
  const dim3 grid((unsigned)(gx < 4096 ? gx : 4096), (unsigned)(srows < 65535 ? srows : 65535));
  k_uncompress<<<grid, 256, 0, s>>>(w, srows, scols, lrows, lcols, t, e, slots, reversed, column_axis, p,
                                    (uint32_t)(0x100000000ull / p), out, overflow);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_reduce_common(const double* acc, size_t count, uint32_t qmask, uint32_t p,
                                 int32_t* c, cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  k_reduce_common<<<grid1d(count, 256), 256, 0, s>>>(acc, count, qmask, p, c);
  count_launch();
  return cudaGetLastError();
}

// extract_all, pack.hpp:104-119, over `count` words: the e base-Q digits of
// every word, least significant first, unreduced (each in [0, Q-1]); a word
// that is negative or not below Q^e raises *overflow (DigitOverflow).
// W = double (DoubleWord) or uint64_t (Int64Word).
template <class W>
__global__ void k_extract_digits(const W* __restrict__ w, size_t count, int t, int e, uint64_t* __restrict__ out,
                                 int* overflow) {
  const size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  if (i >= count) return;
  const W v = w[i];
  const int total = t * e;
  bool bad;
  if constexpr (std::is_same<W, double>::value)
    bad = !(v >= 0.0) || !(v < exp2((double)total));  // NaN and negative words included
  else
    bad = total < 64 && (uint64_t)v >= (1ull << total);
  if (bad) {
    atomicExch(overflow, 1);
    return;
  }
  const uint64_t bits = std::is_same<W, double>::value ? __double2ull_rz((double)v) : (uint64_t)v;
  const uint64_t mask = t >= 64 ? ~0ull : ((1ull << t) - 1);
  for (int s = 0; s < e; ++s) {
    const int sh = s * t;
    out[i * e + s] = sh < 64 ? (bits >> sh) & mask : 0ull;
  }
}

cudaError_t launch_extract_digits(const void* w, bool u64, size_t count, int t, int e, uint64_t* out, int* overflow,
                                  cudaStream_t s) {
  if (count == 0) return cudaSuccess;
  if (u64)
    k_extract_digits<uint64_t><<<grid1d(count, 256), 256, 0, s>>>((const uint64_t*)w, count, t, e, out, overflow);
  else
    k_extract_digits<double><<<grid1d(count, 256), 256, 0, s>>>((const double*)w, count, t, e, out, overflow);
  count_launch();
  return cudaGetLastError();
}

}  // namespace qgk
