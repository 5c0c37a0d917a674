// qg_kernels.h — internal launcher declarations (not part of the C ABI).
#pragma once
#include <cstddef>
#include <cstdint>
#include <cuda_runtime.h>

namespace qgk {

enum PackKind { PACK_ROWS_REVERSED = 0, PACK_COLS_FORWARD = 1, PACK_OUTER_COLS = 2, PACK_OUTER_ROWS = 3 };

void count_launch();

cudaError_t launch_gen_residues(uint64_t seed, uint32_t p, size_t row0, size_t rows, size_t cols,
                                void* dst, int dtype, cudaStream_t s);
// panel_len / panel_words: see Panels in qg_pack.cu (0, 0 = plain layout).
cudaError_t launch_pack(int kind, const void* src, int dtype, size_t rows, size_t cols, size_t ld,
                        int t, int e, double* dst, size_t ldd, size_t panel_len,
                        size_t panel_words, cudaStream_t s);
cudaError_t launch_pack_u64(int kind, const void* src, int dtype, size_t rows, size_t cols, size_t ld, int t, int e,
                            uint64_t* dst, size_t ldd, size_t panel_len, size_t panel_words, cudaStream_t s);
// Int64Word backend (qg_word64.cu); a_dtype / b_dtype -1 = uint64 words
cudaError_t launch_gemm_u64(int mode, const void* a, int a_dtype, size_t lda, const void* b, int b_dtype, size_t ldb,
                            size_t M, size_t N, size_t K, int sh, uint64_t mask, uint64_t* d, size_t ldd,
                            cudaStream_t s);
cudaError_t launch_word_reduce_u64(const uint64_t* w, size_t count, int op, int shift, uint64_t mask, uint32_t p,
                                   int32_t* out, int accumulate, cudaStream_t s);
cudaError_t launch_redq_u64(uint64_t* w, size_t count, int t, int e, uint32_t p, int* overflow, cudaStream_t s);
cudaError_t launch_uncompress_u64(const uint64_t* w, size_t srows, size_t scols, size_t lrows, size_t lcols, int t,
                                  int e, int slots, int reversed, int column_axis, uint32_t p, int32_t* out,
                                  int* overflow, cudaStream_t s);
cudaError_t launch_reduce_and_compress_u64(const uint64_t* w, size_t rows, size_t cols, size_t ldw, int t, int d, int e,
                                           uint32_t p, uint64_t* out, size_t ldo, cudaStream_t s);
cudaError_t launch_uncompress_full_u64(const uint64_t* cc, size_t ldcc, size_t m, size_t n, int t, int qs, int ts,
                                       uint32_t p, int32_t* c, size_t ldc, cudaStream_t s);
cudaError_t launch_redq(double* w, size_t count, int t, int e, uint32_t p, int* overflow,
                        cudaStream_t s);
cudaError_t launch_uncompress(const double* w, size_t srows, size_t scols, size_t lrows,
                              size_t lcols, int t, int e, int slots, int reversed, int column_axis,
                              uint32_t p, int32_t* out, int* overflow, cudaStream_t s);
// extract_all (pack.hpp:104-119) of every word: e unreduced digits per word.
cudaError_t launch_extract_digits(const void* w, bool u64, size_t count, int t, int e, uint64_t* out, int* overflow,
                                  cudaStream_t s);
cudaError_t launch_reduce_common(const double* acc, size_t count, uint32_t qmask, uint32_t p,
                                 int32_t* c, cudaStream_t s);

// Tensor-core (DMMA) contraction C = A (M x K words) x B (K x N words).
// Common variant (launch_dot_dmma): k-blocks of kb_stages pipeline stages of
// `bk` words each, per-block digit extraction, mod-p int32 epilogue
// (accumulate: add the existing C first). Mixed variant (launch_right_dmma):
// exact sums, fused REDQ (redq) or raw words.
struct GemmArgs {
  const double* a;
  size_t lda;
  const double* b;
  size_t ldb;
  int M, N, K;
  int kb_stages;        // stages per k-block; 0 = single block
  double anchor;        // 2^(t d + 52)
  uint32_t qmask, p;
  int accumulate;
  int32_t* c;
  size_t ldc;
  int t, e;             // REDQ digit geometry
  double* cc;
  size_t ldcc;
  int debug;            // experiments only (QG_DEBUG_MODE)
  int pack_period;      // packed digit sums: reduce both 16-bit lanes every this many flushes
  unsigned skew_ns;     // start delay of warps 4..7 (desynchronises the flushes of SMSP warp pairs)
  int balanced;         // balanced (signed) digits: round-to-nearest extraction, biased by Q/2
  uint32_t corr;        // balanced: (p - (#extractions * Q/2) mod p) mod p, added in the epilogue
  double redq_off2;     // balanced REDQ: sum_s (Q/2) Q^s + 2^52 (makes every signed digit an unsigned one)
  uint32_t redq_ybias;  // balanced REDQ: p ceil(Q/2 / p) - Q/2, so x + ybias = D (mod p) and >= 0
  int group;            // tile raster: rows per group (0 = 8)
  int* tile_counter;    // tiled kernels: dynamic tile schedule from this zeroed counter (NULL = static)
  int anchored_kb;      // K4A (qg_anchor.cu): k-block words of the anchored contraction, 0 = K4
  int anch_shift;       // K4A: digit d sits at bits [anch_shift, anch_shift + t) of an accumulator's low word
  double anchor1;  // K4A: the odd output columns start from this second anchor = anchor + Q^(d+1) (the
                        // difference is invisible to the digit field): two distinct values keep the C operand
                        // of the restart DMMAs a fixed register quad
};
cudaError_t launch_dot_dmma(const GemmArgs& a, int bk, cudaStream_t s, const char** variant);
cudaError_t launch_right_dmma(const GemmArgs& a, bool redq, cudaStream_t s, const char** variant);
// K4A: anchored accumulators, integer-pipe block flush (balanced plans; a.anchor = A0,
// a.anchor1, a.anch_shift, a.anchored_kb set; the tiled layout's stage depth is kb_words).
// repack: ReduceAndCompress fused into the epilogue (CC words in a.cc / a.ldcc packed under a.t, a.e; p < 256;
// the caller zeroes CC first unless a.e divides 32), else int32 C.
cudaError_t launch_dot_anchor(const GemmArgs& a, int kb_words, int* tile_counter, cudaStream_t s,
                              const char** variant, bool repack = false);
// Same contraction on the tiled layout (a = CA_t, b = CB_t; lda/ldb unused).
cudaError_t launch_dot_tiled(const GemmArgs& a, int bk, cudaStream_t s, const char** variant);
// Tiled kernels: claim tiles dynamically from an atomic counter (on) or
// statically every gridDim.x-th tile (off); QG_DYN overrides.
void set_dynamic_tiles(int enable);
// The same with ReduceAndCompress fused into the epilogue (p < 256): CC words
// (a.cc, a.ldcc) = C's rows packed forward in groups of a.e under Q = 2^a.t.
// Words that straddle 32-column warp segments are accumulated with atomics:
// the caller zeroes CC first unless a.e divides 32.
cudaError_t launch_dot_tiled_repack(const GemmArgs& a, int bk, cudaStream_t s, const char** variant);
// Mixed variant on the tiled layout: a = A_t (residues, e = 1 blocks), b =
// CBo_t (compress_outer_cols words, transposed blocks); REDQ between k-blocks
// (kb_stages) and in the epilogue, CC m x N (N = ceil(n/e)).
cudaError_t launch_right_tiled(const GemmArgs& a, int bk, bool redq, cudaStream_t s, const char** variant);
// balanced operands (a.balanced): signed residues / words in, canonical CC out
cudaError_t launch_pack_outer_tiled_bal(const void* src, int dtype, size_t k, size_t n, size_t ld, int t, int e, int bk,
                                        double* dst, uint32_t p, cudaStream_t s);
cudaError_t launch_pack_outer_rows_tiled_bal(const void* src, int dtype, size_t m, size_t k, size_t ld, int t, int e,
                                             int bk, double* dst, uint32_t p, cudaStream_t s);
// CBo_t[tn][kt][r][c] = compress_outer_cols(B)[BK kt + c][128 tn + r].
cudaError_t launch_pack_outer_rows_tiled(const void* src, int dtype, size_t m, size_t k, size_t ld, int t, int e,
                                         int bk, double* dst, cudaStream_t s);
cudaError_t launch_extract_coefficients(const double* w, size_t count, int t, int d, int e, double inv_qd, int mode,
                                        uint32_t p, int32_t* out, cudaStream_t s);
cudaError_t launch_reduce_and_compress(const double* w, size_t rows, size_t cols, size_t ldw, int t, int d, int e,
                                       double inv_qd, int mode, uint32_t p, double* out, size_t ldo, cudaStream_t s);
cudaError_t launch_naive_gemm(const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n, uint32_t p,
                              int32_t* c, size_t ldc, cudaStream_t s);
cudaError_t launch_uncompress_full(const double* cc, size_t ldcc, size_t m, size_t n, int t, int qs, int ts,
                                   uint32_t p, int32_t* c, size_t ldc, cudaStream_t s);
cudaError_t launch_pack_outer_tiled(const void* src, int dtype, size_t k, size_t n, size_t ld, int t, int e,
                                    int bk, double* dst, cudaStream_t s);
// Tiled packings: A (m x k residues) -> CA_t, B (k x n residues) -> CB_t.
cudaError_t launch_pack_tiled(bool b_operand, const void* src, int dtype, size_t rows, size_t cols,
                              size_t ld, int t, int e, int bk, double* dst, cudaStream_t s,
                              uint32_t p = 0, bool balanced = false);

// Small products (qg_small.cu): the tiled contraction with 64x64 tiles and
// the k stages split over a cluster of `splits` CTAs (grid z), reduced over
// distributed shared memory. a = CA_t, b = CB_t (the tiled layout of stage
// depth bk, Kt stages).
struct SmallArgs {
  const double* a;
  const double* b;
  int M, N, K, Kt;      // rows of A, columns of B, words, stages of the layout
  int balanced;
  int kb_stages;        // stages per k-block inside a split; 0 = the split is one block
  int split_stages;     // stages per split
  double anchor;
  uint32_t qmask, p;
  uint32_t corr;        // balanced: (p - (#extractions * Q/2) mod p) mod p
  int32_t* c;
  size_t ldc;
  int nstages;          // set by the launcher: shared-memory ring depth
};
cudaError_t launch_small_tiled(const SmallArgs& a, int bk, int splits, cudaStream_t s, const char** variant);

// Reference high-part semantics (word.hpp:28-30): acc += trunc(a*b*2^-td).
struct HighArgs {
  const double* ca;
  size_t ldca;
  const double* cb;
  size_t ldcb;
  int M, N, K;
  double inv_qd;
  int kb_words;         // 0 = single block
  uint32_t qmask, p;
  double* acc;          // raw accumulators (qg_packed_common_product) or NULL
  int32_t* c;           // reduced C or NULL
  size_t ldc;
};
cudaError_t launch_dot_highpart(const HighArgs& a, cudaStream_t s, const char** variant);

}  // namespace qgk
