/* qgemm_b200.h — C ABI of the B200-native compressed modular GEMM.
 *
 * Drop-in boundary for the reference's C++ header API (namespace qgemm,
 * /root/reference/proj/include/qgemm/). The reference has no FFI: its
 * boundary is the header-level functions cited beside each entry point
 * below. Here they are plain C: integer status, plain structs, caller-owned
 * buffers, no exceptions, no torch types. Device entry points are
 * stream-ordered (`stream` is a cudaStream_t; NULL = legacy default stream)
 * and take DEVICE pointers; the qg_host_* entry points take HOST buffers and
 * do their own host<->device copies (the reference-facing value-semantics
 * calls). Every device computation runs in hand-written sm_100a kernels;
 * there is no CPU fallback: without a usable CUDA device the calls return
 * QG_CUDA_ERROR.
 *
 * Layouts are exactly CompressedMatrix::data (matrix.hpp:44-63):
 *   CA  (compress_rows_reversed) m x ceil(k/e) row-major words
 *   CB  (compress_cols_forward)  ceil(k/e) x n row-major words
 *   CBo (compress_outer_cols)    k x ceil(n/e) row-major words
 *   CC  (right product / repack) m x ceil(n/e) row-major words
 * Residues on the device are stored as double (exact small integers) or as
 * uint32 (ResidueMatrix, matrix.hpp:14-26); results C are int32 row-major.
 */
#ifndef QGEMM_B200_H
#define QGEMM_B200_H
#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QG_ABI_VERSION 1

/* Status codes: 0 = ok, then the exception classes of errors.hpp:8-34 in
 * declaration order, then std::invalid_argument (plan.hpp:128-129,
 * gemm.hpp:455), then device-side failures. */
typedef enum {
  QG_OK = 0,
  QG_INVALID_MODULUS = 1,      /* errors.hpp:13 */
  QG_NO_COMPRESSION = 2,       /* errors.hpp:16 */
  QG_SLOT_OVERFLOW = 3,        /* errors.hpp:19 */
  QG_DIGIT_OVERFLOW = 4,       /* errors.hpp:22 */
  QG_DIMENSION_MISMATCH = 5,   /* errors.hpp:25 */
  QG_PLAN_MISMATCH = 6,        /* errors.hpp:28 */
  QG_UNSUPPORTED_ALGORITHM = 7,/* errors.hpp:31 */
  QG_PARSE_ERROR = 8,          /* errors.hpp:34 */
  QG_INVALID_ARGUMENT = 9,     /* std::invalid_argument */
  QG_CUDA_ERROR = 10,
  QG_NCCL_ERROR = 11,
  QG_NOT_EXACT = 12            /* a k-block violates the FP64 exactness bound */
} qg_status;

/* ExtractionMode, plan.hpp:14-17 */
enum { QG_EXTRACT_RECIPROCAL_MUL = 0, QG_EXTRACT_ADD_HIGH_BITS = 1 };

/* CompressionPlan, plan.hpp:29-42. Identical field meaning. */
typedef struct {
  uint32_t p;       /* prime modulus */
  int32_t t;        /* Q = 2^t */
  int32_t d;        /* packing degree */
  int32_t e;        /* residues per word, e = d + 1 */
  int32_t beta;     /* exact bits of the word backend (53 for double) */
  uint64_t kmax;    /* largest legal common dimension for this t */
  double inv_qd;    /* 2^(-t d) */
  int32_t extraction;
} qg_plan;

/* A plan plus the k-block size the FP64 tensor-core contraction flushes at
 * (FFLAS-style blocking, gemm.hpp:450-489, done in registers). kblock_words
 * packed words per block; each block is both legal for Eq. 3
 * (kblock_words*e <= kmax) and exact for a DMMA FMA chain (Eq. G). */
typedef struct {
  qg_plan plan;
  uint64_t kblock_words;
  uint64_t max_exact_words; /* Eq. G bound for (p, t, e), informational */
  /* 1: residues enter the packed words in balanced form (v > p/2 -> v - p),
   * so every digit is signed with |digit| <= (p/2)^2 per product; digit d is
   * read by rounding to nearest. Twice the exact block of
   * the unsigned packing at the same (t, e). Tiled path only. */
  int32_t balanced;
  /* 1 (balanced plans, tiled path): anchored accumulation —
   * every k-block starts from the anchor 1.5*2^E inside the DMMA chain, so the
   * block's digit is read from fixed bits of the accumulator on the integer
   * pipe instead of by one FP64 add per accumulator. kblock_words is then
   * bounded by qg_max_exact_block_anchored and is an odd multiple of 4. Any
   * entry without an anchored kernel runs the same blocks with the FP64 flush
   * (an anchored block is always within Eq. G). */
  int32_t anchored;
} qg_gpu_plan;

/* PackOrientation, matrix.hpp:28-39: direction 0 Forward / 1 Reversed;
 * axis 0 Row / 1 Column; slots residues per word along the packed axis. */
typedef struct {
  int32_t direction;
  int32_t axis;
  int32_t slots;
} qg_orientation;
enum { QG_FORWARD = 0, QG_REVERSED = 1 };
enum { QG_ROW = 0, QG_COLUMN = 1 };

/* Element type of residue buffers. */
typedef enum { QG_F64 = 0, QG_U32 = 1, QG_I32 = 2 } qg_dtype;

/* ---------------------------------------------------------------- host */
int qg_abi_version(void);
const char* qg_status_string(int status);

/* plan_compression, plan.hpp:125-159 */
int qg_plan_compression(uint32_t p, uint64_t k, int beta, int mode, qg_plan* out);
/* uncompressed_plan, plan.hpp:164-179 */
int qg_uncompressed_plan(uint32_t p, uint64_t k, int beta, qg_plan* out);
/* plan_packed_axis, plan.hpp:186-203 */
int qg_plan_packed_axis(uint32_t p, uint64_t k, uint64_t axis_len, int beta, qg_plan* out);
/* choose_panel, plan.hpp:209-224 */
int qg_choose_panel(uint32_t p, uint64_t k, int beta, uint64_t* out);
/* largest block (packed words) for which a DMMA contraction of this plan is
 * provably exact (Eq. G with rho = 1, unfused products). */
int qg_max_exact_block(const qg_plan* plan, uint64_t* words);
/* k-block an existing plan for the tensor-core path (reference plan kept). */
int qg_gpu_plan_from(const qg_plan* plan, uint64_t k, qg_gpu_plan* out);
/* choose (t, e, kblock, balanced) for common dimension k on the tensor-core
 * path: minimises predicted contraction time over all exact blocked plans. */
int qg_plan_gpu(uint32_t p, uint64_t k, qg_gpu_plan* out);
/* qg_plan_gpu with flags: QG_PLAN_UNSIGNED_ONLY restricts to unsigned digits
 * (words bit-compatible with the reference packing, for the row layouts). */
enum { QG_PLAN_UNSIGNED_ONLY = 1, QG_PLAN_NO_ANCHOR = 2 };
int qg_plan_gpu_ex(uint32_t p, uint64_t k, int flags, qg_gpu_plan* out);
/* Eq. G bound for balanced digits (qg_gpu_plan.balanced = 1). */
int qg_max_exact_block_balanced(const qg_plan* plan, uint64_t* words);
/* Largest k-block (words) of the anchored accumulation for (p, t, e): every
 * partial sum of a block stays in one binade [2^E, 2^(E+1)) and Eq. G holds
 * with the fixed ulp 2^(E-52). *exponent (may be NULL) gets
 * the E of that block, 0 if no block is exact. */
int qg_max_exact_block_anchored(const qg_plan* plan, uint64_t* words, int* exponent);
/* qg_plan_gpu_ex flag: consider anchored plans too (the default planner does
 * once QG_PLAN_ANCHORED is set; the planner picks by predicted time). */
/* Eq. 3 bound (residues per k-block) that the contraction enforces for a GPU
 * plan, recomputed from (p, t): largest_common_dim (plan.hpp:113-115), capped
 * by a smaller plan.kmax, for unsigned plans; the balanced-digit bound
 * ((2^(t-1) - 1) / floor(p/2)^2) for balanced ones. plan.kmax itself always
 * stays the reference's meaning. */
int qg_gpu_plan_kmax(const qg_gpu_plan* gplan, uint64_t* kmax);

/* -------------------------------------------------- device (stream-ordered) */
/* random_residue_matrix, prng.hpp:31-38 (SplitMix64 stream, counter-based):
 * rows [row0, row0+rows) of the rows_total x cols matrix of seed. */
int qg_gen_residues(uint64_t seed, uint32_t p, size_t row0, size_t rows, size_t cols,
                    void* dst, qg_dtype dtype, void* stream);

/* compress_rows_reversed, gemm.hpp:104-118 (+ compress_reverse, pack.hpp:59-70).
 * A: m x k residues (lda elements), CA: m x ceil(k/e) (ldca words). */
int qg_compress_rows_reversed(const qg_plan* plan, const void* a, qg_dtype dtype, size_t m,
                              size_t k, size_t lda, double* ca, size_t ldca, void* stream);
/* compress_cols_forward, gemm.hpp:122-140 (+ compress_forward, pack.hpp:47-54). */
int qg_compress_cols_forward(const qg_plan* plan, const void* b, qg_dtype dtype, size_t k,
                             size_t n, size_t ldb, double* cb, size_t ldcb, void* stream);
/* compress_outer_cols, gemm.hpp:145-158: k x n residues -> k x ceil(n/e) words. */
int qg_compress_outer_cols(const qg_plan* plan, const void* b, qg_dtype dtype, size_t rows,
                           size_t cols, size_t ldb, double* cb, size_t ldcb, void* stream);
/* compress_outer_rows, gemm.hpp:161-178: m x k residues -> ceil(m/e) x k words. */
int qg_compress_outer_rows(const qg_plan* plan, const void* a, qg_dtype dtype, size_t rows,
                           size_t cols, size_t lda, double* ca, size_t ldca, void* stream);

/* packed_common_product, gemm.hpp:210-244, with the reference's own
 * per-product high-part semantics (word.hpp:28-30): acc = sum_g
 * trunc(CA*CB*2^-td), bit-identical doubles. m x n accumulators. */
int qg_packed_common_product(const qg_plan* plan, const double* ca, const double* cb,
                             size_t m, size_t n, size_t k, double* acc, void* stream);
/* reduce_common_entry over a buffer, gemm.hpp:247-250. */
int qg_reduce_common(const qg_plan* plan, const double* acc, size_t count, int32_t* c,
                     void* stream);

/* mul_common_compressed(ca, cb), gemm.hpp:263-271, + blocked_accumulate's
 * mod-p accumulation between k-blocks (gemm.hpp:450-489), fused: one DMMA
 * contraction kernel, in-register per-block digit extraction, mod-p epilogue.
 * C: m x n int32 (ldc). k = logical common dimension (residues). */
int qg_mul_common(const qg_gpu_plan* gplan, const double* ca, const double* cb, size_t m,
                  size_t n, size_t k, int32_t* c, size_t ldc, void* stream);
/* mul_common_repacked, gemm.hpp:275-280: C rows re-packed forward in groups
 * of e (ReduceAndCompress, pack.hpp:141-155). cc: m x ceil(n/e) words.
 * workspace: m*n int32 (device) or NULL to allocate internally. */
int qg_mul_common_repacked(const qg_gpu_plan* gplan, const double* ca, const double* cb,
                           size_t m, size_t n, size_t k, double* cc, int32_t* workspace,
                           void* stream);

/* mul_common_repacked on the tiled layout: the contraction with
 * ReduceAndCompress (pack.hpp:141-155) fused into its epilogue — C's rows
 * leave as forward words of e residues under gplan->plan (t, e); no int32 C
 * in HBM (p < 256 on the 128x128-tile kernel; otherwise through an int32
 * workspace). cc: m x ceil(n/e) words (ldcc). */
int qg_mul_common_repacked_tiled(const qg_gpu_plan* gplan, const double* ca_t, const double* cb_t, size_t m,
                                 size_t n, size_t k, double* cc, size_t ldcc, void* stream);
/* mul_common_repacked(A, B) on device residues in one call (tiled packs into
 * stream-ordered workspaces + qg_mul_common_repacked_tiled). */
int qg_mul_common_repacked_compressed(const qg_gpu_plan* gplan, const void* a, size_t lda, const void* b, size_t ldb,
                                      qg_dtype dtype, size_t m, size_t k, size_t n, double* cc, size_t ldcc,
                                      void* stream);
/* mul_common_repacked(A, B, plan), gemm.hpp:275-280, on HOST data: cc gets
 * m x ceil(n/e) words, bit-identical to compress_outer_cols(C, plan). */
int qg_host_mul_common_repacked(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                size_t n, double* cc);
int qg_host_mul_common_repacked_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m,
                                    size_t k, size_t n, double* cc);

/* ---- tiled packed layout (the B200 fast path for the dot-product variant).
 * The same words as compress_rows_reversed / compress_cols_forward, stored as
 * dense, zero-padded 128 x BK blocks so that one pipeline stage of the
 * contraction is one contiguous chunk per operand:
 *   CA_t[tm][kt][r][c] = CA[128 tm + r][BK kt + c]
 *   CB_t[tn][kt][r][c] = CB[BK kt + c][128 tn + r]   (B transposed)
 * qg_tiled_stage_words gives the BK a plan runs with; qg_tiled_words the
 * buffer size in doubles for `rows` (m for CA_t, n for CB_t). */
int qg_tiled_stage_words(const qg_gpu_plan* gplan, uint64_t k, uint32_t* bk);
size_t qg_tiled_words(size_t rows, size_t k, int e, uint32_t bk);
int qg_pack_a_tiled(const qg_gpu_plan* gplan, uint32_t bk, const void* a, qg_dtype dtype, size_t m,
                    size_t k, size_t lda, double* ca_t, void* stream);
int qg_pack_b_tiled(const qg_gpu_plan* gplan, uint32_t bk, const void* b, qg_dtype dtype, size_t k,
                    size_t n, size_t ldb, double* cb_t, void* stream);
/* qg_mul_common on tiled operands. Products whose 128 x 128 tiles would fill
 * less than half of the SMs (config 1: 16 tiles), odd n / ldc and C not
 * 8-byte aligned run on 64 x 64 tiles with the k stages split over a
 * thread-block cluster (qg_small.cu); the rest on the persistent 128 x 128
 * kernel (qg_dot.cu). */
int qg_mul_common_tiled(const qg_gpu_plan* gplan, const double* ca_t, const double* cb_t, size_t m,
                        size_t n, size_t k, int32_t* c, size_t ldc, void* stream);

/* mul_common_compressed(A, B, plan), gemm.hpp:254-261 (compress_rows_reversed
 * + compress_cols_forward + packed_common_product + reduce_common_entry, with
 * blocked_accumulate's k-blocks, gemm.hpp:450-489) on device residues in one
 * call: a m x k (lda), b k x n (ldb), both of `dtype`; C m x n int32 (ldc).
 * Tiled packs into stream-ordered workspaces + qg_mul_common_tiled; plans with
 * one-digit words wider than 31 bits run on the reference layout. */
int qg_mul_common_compressed(const qg_gpu_plan* gplan, const void* a, size_t lda, const void* b, size_t ldb,
                             qg_dtype dtype, size_t m, size_t k, size_t n, int32_t* c, size_t ldc, void* stream);

/* ---- mixed variant on the tiled layout (the B200 fast path of
 * mul_right_compressed). A's residues as dense 128 x BK blocks (e = 1), B's
 * compress_outer_cols words transposed into 128 x BK blocks; the contraction
 * REDQs the exact accumulators in place between k-blocks of
 * gplan->kblock_words residues (qg_plan_right_gpu) and in its epilogue.
 * cc: m x ceil(n/e) words, bit-identical to mul_right_compressed's under the
 * same plan. */
int qg_plan_right_gpu(uint32_t p, uint64_t k, uint64_t n, qg_gpu_plan* out);
int qg_right_tiled_stage(const qg_gpu_plan* gplan, uint64_t k, uint32_t* bk);
int qg_pack_residues_tiled(uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda,
                           double* a_t, void* stream);
int qg_pack_outer_cols_tiled(const qg_plan* plan, uint32_t bk, const void* b, qg_dtype dtype, size_t k,
                             size_t n, size_t ldb, double* bo_t, void* stream);
int qg_mul_right_tiled(const qg_gpu_plan* gplan, const double* a_t, const double* bo_t, size_t m, size_t k,
                       size_t n, double* cc, size_t ldcc, void* stream);

/* ---- left and full compression on the tiled layout, gemm.hpp:340-445.
 * Both contract with the REDQ kernel of the mixed variant; only the operand
 * packs differ.
 *
 * Left (mul_left_compressed(compress_outer_rows(A), B), gemm.hpp:340-371):
 * A's compress_outer_rows words (ceil(m/e) x k, pack.hpp / gemm.hpp:160-176)
 * as 128 x BK blocks, B's residues transposed into 128 x BK blocks (e = 1).
 * cc: ceil(m/e) x n post-REDQ words, digit s of cc[g][j] = C[g e + s][j]
 * (qg_uncompress with {Forward, Row, e} unpacks it). gplan: any qg_gpu_plan
 * whose kblock_words bounds the in-place REDQ blocks (qg_plan_right_gpu(p,
 * k, m) picks one; qg_gpu_plan_from-style {plan, kblock = k} keeps the
 * reference's single block). */
int qg_pack_outer_rows_tiled(const qg_plan* plan, uint32_t bk, const void* a, qg_dtype dtype, size_t m,
                             size_t k, size_t lda, double* ao_t, void* stream);
int qg_pack_residues_b_tiled(uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n, size_t ldb,
                             double* b_t, void* stream);
int qg_mul_left_tiled(const qg_gpu_plan* gplan, const double* ao_t, const double* b_t, size_t m, size_t k,
                      size_t n, double* cc, size_t ldcc, void* stream);
/* Balanced-digit operands of the right/left contractions, for plans with
 * gplan->balanced (qg_plan_right_gpu picks them for odd p): residue v enters
 * as v - p when v > p/2, halving every digit's bound, so k-blocks between
 * in-place REDQs are about twice as long. The CC words out are the same
 * canonical (unsigned) words. */
int qg_pack_residues_tiled_bal(uint32_t p, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda,
                               double* a_t, void* stream);
int qg_pack_residues_b_tiled_bal(uint32_t p, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n,
                                 size_t ldb, double* b_t, void* stream);
int qg_pack_outer_cols_tiled_bal(const qg_plan* plan, uint32_t bk, const void* b, qg_dtype dtype, size_t k, size_t n,
                                 size_t ldb, double* bo_t, void* stream);
int qg_pack_outer_rows_tiled_bal(const qg_plan* plan, uint32_t bk, const void* a, qg_dtype dtype, size_t m, size_t k,
                                 size_t lda, double* ao_t, void* stream);

/* Full (mul_full_compressed, gemm.hpp:377-445): rows of A packed in base Q
 * with dq+1 slots (qg_pack_outer_rows_tiled under {t, e = dq+1}), columns of
 * B in base Theta = 2^theta_exponent with dtheta+1 slots
 * (qg_pack_outer_cols_tiled under {t = theta_exponent, e = dtheta+1}). The
 * contraction REDQs all (dq+1)(dtheta+1) base-Q digits in place every
 * kblock_words residues; cc: ceil(m/(dq+1)) x ceil(n/(dtheta+1)) words, and
 * qg_uncompress_full scatters digit i + j (dq+1) of cc[g][h] to
 * C[g (dq+1) + i][h (dtheta+1) + j]. */
typedef struct {
  qg_plan base; /* e = (dq+1)(dtheta+1), d = e-1 */
  int32_t dq, dtheta, theta_exponent;
} qg_full_plan;
/* plan_full, plan.hpp:229-252 */
int qg_plan_full(uint32_t p, uint64_t k, int beta, qg_full_plan* out);
/* B200 planner: same slot split, free radix, k-blocked (kblock_words out). */
int qg_plan_full_gpu(uint32_t p, uint64_t k, qg_full_plan* out, uint64_t* kblock_words);
int qg_full_tiled_stage(const qg_full_plan* fp, uint64_t kblock_words, uint64_t k, uint32_t* bk);
int qg_mul_full_tiled(const qg_full_plan* fp, uint64_t kblock_words, const double* ao_t, const double* bo_t,
                      size_t m, size_t k, size_t n, double* cc, size_t ldcc, void* stream);
int qg_uncompress_full(const qg_full_plan* fp, const double* cc, size_t ldcc, size_t m, size_t n, int32_t* c,
                       size_t ldc, void* stream);

/* packed_right_product + redq_in_place = mul_right_compressed(a, cb),
 * gemm.hpp:285-325: CC = REDQ(A x CBo). A: m x k residues as double (lda),
 * CBo: k x ceil(n/e) words. cc: m x ceil(n/e). */
int qg_mul_right(const qg_plan* plan, const double* a, size_t lda, const double* cbo,
                 size_t m, size_t k, size_t n, double* cc, void* stream);
/* packed_right_product alone (pre-REDQ words), gemm.hpp:285-310. */
int qg_packed_right_product(const qg_plan* plan, const double* a, size_t lda,
                            const double* cbo, size_t m, size_t k, size_t n, double* cc,
                            void* stream);

/* packed_left_product, gemm.hpp:340-364 (DoubleWord, reference layout):
 * CA (compress_outer_rows words, ceil(m/e) x k, ldca) x B (k x n residues of
 * `dtype`, ldb) -> cc (ceil(m/e) x n pre-REDQ words). qg_mul_left adds the
 * REDQ of mul_left_compressed(ca, b), gemm.hpp:366-371. */
int qg_packed_left_product(const qg_plan* plan, const double* ca, size_t ldca, const void* b, qg_dtype dtype,
                           size_t ldb, size_t m, size_t k, size_t n, double* cc, void* stream);
int qg_mul_left(const qg_plan* plan, const double* ca, size_t ldca, const void* b, qg_dtype dtype, size_t ldb,
                size_t m, size_t k, size_t n, double* cc, void* stream);
/* extract_all, pack.hpp:104-119, over `count` words: digits[i*e + s] = digit s
 * of word i (unreduced); QG_DIGIT_OVERFLOW if a word is negative or >= Q^e. */
int qg_extract_digits(const qg_plan* plan, const double* words, size_t count, uint64_t* digits, void* stream);
int qg_extract_digits_u64(const qg_plan* plan, const uint64_t* words, size_t count, uint64_t* digits,
                          void* stream);
/* Device memory for callers without the CUDA headers (include/qgemm_b200.hpp):
 * synchronous copies on the legacy default stream (the stream the entry
 * points use when passed NULL). */
int qg_device_alloc(size_t bytes, void** ptr);
int qg_device_free(void* ptr);
int qg_copy_to_device(void* dst, const void* src, size_t bytes);
int qg_copy_to_host(void* dst, const void* src, size_t bytes);

/* redq_in_place, gemm.hpp:313-316 / redq, pack.hpp:124-137. Words that do
 * not fit e digits make the call return QG_DIGIT_OVERFLOW (checked on the
 * device, reported after a stream sync). */
int qg_redq(const qg_plan* plan, double* words, size_t count, void* stream);
/* uncompress, gemm.hpp:182-204 (+ extract_all, pack.hpp:104-119). */
int qg_uncompress(const qg_plan* plan, qg_orientation o, const double* words,
                  size_t stored_rows, size_t stored_cols, size_t logical_rows,
                  size_t logical_cols, int32_t* out, void* stream);

/* --------------------------------------------- host buffers (value semantics) */
/* mul_common_compressed(A, B, plan), gemm.hpp:254-260, on HOST ResidueMatrix
 * data (uint32 row-major). Uses the tensor-core path with the plan k-blocked
 * for exactness. Copies in, computes on the current device, copies C out. */
int qg_host_mul_common(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                       size_t k, size_t n, uint32_t* c);
/* Same, under an explicit k-blocked GPU plan (qg_plan_gpu): k may exceed
 * plan.kmax; blocks are packed, contracted and accumulated mod p on device. */
int qg_host_mul_common_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b,
                           size_t m, size_t k, size_t n, uint32_t* c);
/* blocked_accumulate(A, B, plan, kpanel), gemm.hpp:450-489 on HOST data:
 * panels of kpanel residues, each packed under `plan`, mod-p accumulation. */
/* mul_common_compressed over `ngpus` devices of this process:
 * rows of A and C sharded over devices[] (128-row multiples), B packed once on
 * devices[0] into the tiled layout and broadcast as packed words by one
 * grouped ncclBroadcast (NVLink / NVSwitch), every device packs and contracts
 * its own rows; host buffers in / out as qg_host_mul_common_gpu. NCCL is
 * dlopen'ed (libnccl.so.2) at the first call; QG_NCCL_ERROR if absent. */
int qg_host_mul_common_multi(const qg_gpu_plan* gplan, const int* devices, int ngpus, const uint32_t* a,
                             const uint32_t* b, size_t m, size_t k, size_t n, uint32_t* c);
/* The multi-process (one rank per GPU) host path in two halves around the
 * caller's all-gather (paper_0803_1975_b200/dist.py):
 * qg_host_pack_b_slot_tiled uploads columns [c0, c0+cols) of the HOST B
 * (k x ldb uint32) and packs them into cb_slot (that slot of the tiled CB_t,
 * stage depth bk) on `stream`; qg_host_mul_common_packed_b streams the HOST
 * row shard A (m x k) up in chunks, packs and contracts it against the
 * DEVICE CB_t (all n columns, gathered) and streams C (m x n) back; its
 * contractions wait on ready_event (a cudaEvent_t recorded after the gather;
 * NULL = none) while A's upload and packing already run. */
int qg_host_pack_b_slot_tiled(const qg_gpu_plan* gplan, uint32_t bk, const uint32_t* b, size_t ldb, size_t k,
                              size_t c0, size_t cols, double* cb_slot, void* stream);
int qg_host_mul_common_packed_b(const qg_gpu_plan* gplan, const uint32_t* a, size_t m, size_t k, const double* cb_t,
                                size_t n, uint32_t* c, void* ready_event);
int qg_host_blocked_accumulate(const qg_plan* plan, const uint32_t* a, const uint32_t* b,
                               size_t m, size_t k, size_t n, size_t kpanel, uint32_t* c);
/* mul_right_compressed(A, compress_outer_cols(B)), gemm.hpp:320-325, on HOST
 * data: cc gets the post-REDQ words (m x ceil(n/e)). */
int qg_host_mul_right(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m,
                      size_t k, size_t n, double* cc);

/* The same under a blocked GPU plan (qg_plan_right_gpu(p, k, n)): in-place
 * REDQ every gplan->kblock_words residues; words equal
 * compress_outer_cols(C) under gplan->plan. */
int qg_host_mul_right_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                          size_t n, double* cc);
/* mul_left_compressed(compress_outer_rows(A, plan), B), gemm.hpp:366-371, on
 * HOST data: cc gets the post-REDQ words (ceil(m/e) x n). */
int qg_host_mul_left(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                     size_t n, double* cc);
/* ... under a blocked GPU plan (qg_plan_right_gpu(p, k, m)). */
int qg_host_mul_left_gpu(const qg_gpu_plan* gplan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                         size_t n, double* cc);
/* mul_full_compressed(A, B, fp), gemm.hpp:377-445, on HOST data: c = A B mod
 * p (m x n uint32). kblock_words = 0 means one block (the reference's
 * k <= kmax condition applies); otherwise qg_plan_full_gpu's blocking. */
int qg_host_mul_full(const qg_full_plan* fp, uint64_t kblock_words, const uint32_t* a, const uint32_t* b,
                     size_t m, size_t k, size_t n, uint32_t* c);

/* extract_coefficient (DoubleWord), pack.hpp:78-100, elementwise over count
 * words, in the plan's extraction mode (ReciprocalMul or AddHighBits), bit
 * for bit the reference's result on any word. out: int32 residues. */
int qg_extract_coefficients(const qg_plan* plan, const double* words, size_t count, int32_t* out, void* stream);
/* reduce_and_compress, pack.hpp:141-155, on each of `rows` rows of `cols`
 * accumulated words (ldw): extract every entry, pack groups of e forward.
 * out: rows x ceil(cols/e) words (ldo). */
int qg_reduce_and_compress(const qg_plan* plan, const double* words, size_t rows, size_t cols, size_t ldw,
                           double* out, size_t ldo, void* stream);

/* naive_gemm, gemm.hpp:80-100: C = A B mod p with 64-bit sums, no packing.
 * The independent device checker of the CLI's verify / --algo naive. */
int qg_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n, int32_t* c,
                  size_t ldc, void* stream);
int qg_host_naive_gemm(uint32_t p, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                       uint32_t* c);
/* uncompress (gemm.hpp:182-204) of HOST words into HOST residues. */
int qg_host_uncompress(const qg_plan* plan, qg_orientation o, const double* words, size_t stored_rows,
                       size_t stored_cols, size_t logical_rows, size_t logical_cols, uint32_t* out);
/* random_residue_matrix(rows, cols, PrimeModulus(p), seed), prng.hpp:31-38,
 * generated on the device and copied to HOST memory. */
int qg_host_random_residue_matrix(size_t rows, size_t cols, uint32_t p, uint64_t seed, uint32_t* out);
/* PhaseSeconds of the last host-data call on this thread (gemm.hpp
 * PhaseSeconds, reported by bench.hpp:67-152): multiply = device time of the
 * contraction kernels, convert = the rest of the call (transfers, packing,
 * extraction). The split is measured only while qg_set_phase_timing(1) is in
 * effect (timing events slow the pipelined host path); otherwise multiply is 0
 * and convert the whole call. */
void qg_set_phase_timing(int enable);
void qg_last_phase_seconds(double* multiply, double* convert);

/* ------------------------------------------------- Int64Word backend
 * word.hpp:36-54: packed words are uint64, word products wrap mod 2^64, plans
 * may use beta up to 63 (t e <= 62). Same entry points as the DoubleWord ones
 * with uint64 word buffers; the common product adds Int64Word::high_part =
 * ((a b) >> t d) & (Q-1) per term. Integer kernels on the CUDA cores (no FP64
 * tensor path for 64-bit words); bit-identical to the reference's Int64Word
 * results. */
int qg_compress_rows_reversed_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t m, size_t k, size_t lda,
                                  uint64_t* ca, size_t ldca, void* stream);
int qg_compress_cols_forward_u64(const qg_plan* plan, const void* b, qg_dtype dtype, size_t k, size_t n, size_t ldb,
                                 uint64_t* cb, size_t ldcb, void* stream);
int qg_compress_outer_cols_u64(const qg_plan* plan, const void* b, qg_dtype dtype, size_t rows, size_t cols,
                               size_t ldb, uint64_t* out, size_t ldo, void* stream);
int qg_compress_outer_rows_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t rows, size_t cols,
                               size_t lda, uint64_t* out, size_t ldo, void* stream);
/* packed_common_product<Int64Word> gemm.hpp:210-244 (groups = packed words per row) */
int qg_packed_common_product_u64(const qg_plan* plan, const uint64_t* ca, const uint64_t* cb, size_t m, size_t n,
                                 size_t groups, uint64_t* acc, void* stream);
int qg_reduce_common_u64(const qg_plan* plan, const uint64_t* acc, size_t count, int32_t* c, void* stream);
int qg_extract_coefficients_u64(const qg_plan* plan, const uint64_t* words, size_t count, int32_t* out, void* stream);
int qg_reduce_and_compress_u64(const qg_plan* plan, const uint64_t* words, size_t rows, size_t cols, size_t ldw,
                               uint64_t* out, size_t ldo, void* stream);
int qg_redq_u64(const qg_plan* plan, uint64_t* words, size_t count, void* stream);
int qg_uncompress_u64(const qg_plan* plan, qg_orientation o, const uint64_t* words, size_t stored_rows,
                      size_t stored_cols, size_t logical_rows, size_t logical_cols, int32_t* out, void* stream);
/* packed_right_product / mul_right_compressed <Int64Word>, gemm.hpp:285-325;
 * a: m x k residues (dtype, lda), cbo: k x ceil(n/e) words, cc: m x ceil(n/e) */
int qg_packed_right_product_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t lda, const uint64_t* cbo,
                                size_t m, size_t k, size_t n, uint64_t* cc, void* stream);
int qg_mul_right_u64(const qg_plan* plan, const void* a, qg_dtype dtype, size_t lda, const uint64_t* cbo, size_t m,
                     size_t k, size_t n, uint64_t* cc, void* stream);
/* packed_left_product / mul_left_compressed <Int64Word>, gemm.hpp:340-371;
 * ca: ceil(m/e) x k words, b: k x n residues (dtype, ldb), cc: ceil(m/e) x n */
int qg_packed_left_product_u64(const qg_plan* plan, const uint64_t* ca, const void* b, qg_dtype dtype, size_t ldb,
                               size_t m, size_t k, size_t n, uint64_t* cc, void* stream);
int qg_mul_left_u64(const qg_plan* plan, const uint64_t* ca, const void* b, qg_dtype dtype, size_t ldb, size_t m,
                    size_t k, size_t n, uint64_t* cc, void* stream);
/* mul_full_compressed<Int64Word>, gemm.hpp:377-445 (device residues in, int32 C) */
int qg_mul_full_u64(const qg_full_plan* fp, const void* a, qg_dtype adt, const void* b, qg_dtype bdt, size_t m,
                    size_t k, size_t n, int32_t* c, size_t ldc, void* stream);
/* host-data entries (value semantics) */
int qg_host_mul_common_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                           uint32_t* c);
int qg_host_blocked_accumulate_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k,
                                   size_t n, size_t kpanel, uint32_t* c);
int qg_host_mul_right_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                          uint64_t* cc);
int qg_host_mul_left_i64(const qg_plan* plan, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                         uint64_t* cc);
int qg_host_mul_full_i64(const qg_full_plan* fp, const uint32_t* a, const uint32_t* b, size_t m, size_t k, size_t n,
                         uint32_t* c);
int qg_host_uncompress_u64(const qg_plan* plan, qg_orientation o, const uint64_t* words, size_t stored_rows,
                           size_t stored_cols, size_t logical_rows, size_t logical_cols, uint32_t* out);

/* ----------------------------------------------- matrix files (matrix_io.hpp)
 * "M <p> <rows> <cols>" then rows*cols whitespace-separated residues in
 * [0, p-1], row-major (matrix_io.hpp:14-22). Readers return QG_PARSE_ERROR
 * with the reference's message (qg_last_error()); *data is malloc'd, release
 * it with qg_free. */
int qg_parse_matrix(const char* text, size_t len, uint32_t* p, size_t* rows, size_t* cols, uint32_t** data);
int qg_read_matrix_file(const char* path, uint32_t* p, size_t* rows, size_t* cols, uint32_t** data);
int qg_write_matrix_file(const char* path, uint32_t p, const uint32_t* data, size_t rows, size_t cols);
void qg_free(void* ptr);

/* Tile schedule of the tiled contraction kernels: 1 = tiles claimed from an
 * atomic counter (a CTA that starts late, its SM held by another kernel such
 * as an NCCL all-gather, takes fewer tiles), 0 = static round robin. Process-wide. */
void qg_set_dynamic_tiles(int enable);

/* ------------------------------------------------------------ diagnostics */
/* qg_last_error(): description of the last failure on this thread (CUDA
 * error string, or the parse error text of a matrix file). */
/* Number of kernels this library launched since load (the bench's
 * gpu_launches evidence). */
uint64_t qg_kernel_launches(void);
/* CUDA error string behind the last QG_CUDA_ERROR of this thread. */
const char* qg_last_error(void);
/* Name of the contraction kernel variant the last qg_mul_common used. */
const char* qg_last_kernel(void);

#ifdef __cplusplus
}
#endif
#endif /* QGEMM_B200_H */
