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
cudaError_t launch_redq(double* w, size_t count, int t, int e, uint32_t p, int* overflow,
                        cudaStream_t s);
cudaError_t launch_uncompress(const double* w, size_t srows, size_t scols, size_t lrows,
                              size_t lcols, int t, int e, int slots, int reversed, int column_axis,
                              uint32_t p, int32_t* out, int* overflow, cudaStream_t s);
cudaError_t launch_reduce_common(const double* acc, size_t count, uint32_t qmask, uint32_t p,
                                 int32_t* c, cudaStream_t s);

// Tensor-core (DMMA) contraction of CA (M x K words) by CB (K x N words) with
// per-k-block digit extraction and a mod-p int32 epilogue.
struct DotArgs {
  const double* ca;
  size_t ldca;
  const double* cb;
  size_t ldcb;
  int M, N, K;          // K = packed words
  int kb_steps;         // 4-word k-steps per block; 0 = single block
  int sh_base;          // 1075 + t*d
  uint32_t qmask;       // Q - 1
  uint32_t p;
  int reduce_each;      // reduce digit sums mod p at every flush (huge k)
  int32_t* c;
  size_t ldc;
};
cudaError_t launch_dot_dmma(const DotArgs& a, cudaStream_t s, const char** variant);

// Mixed variant: CC = A (M x K residues as double) x CBo (K x N words); epilogue
// REDQ (redq=1) or raw words (redq=0).
struct RightArgs {
  const double* a;
  size_t lda;
  const double* cb;
  size_t ldcb;
  int M, N, K;
  int t, e;
  uint32_t p;
  int redq;
  double* cc;
  size_t ldcc;
};
cudaError_t launch_right_dmma(const RightArgs& a, cudaStream_t s, const char** variant);

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
