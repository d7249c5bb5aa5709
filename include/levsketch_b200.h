/*
 * levsketch_b200 — C ABI of the B200 (sm_100a) sketched leverage-score path.
 *
 * The reference (levsketch, arXiv 1812.07903; pure Python/numpy) has no native
 * boundary: its hot path is the Python call chain
 *     leverage_sketched_trunc -> apply_sketch/consume_rows -> thin_svd/truncate
 *     -> _approx_basis -> _block_scores -> scores_to_distribution -> make_plan
 * (reference pkg/src/levsketch/leverage.py:115-132, sketch.py:289-319,
 *  svd.py:30-54, order.py:51-100).  Each entry point below replaces one of the
 * numpy kernels of that chain; the Python package paper_1812_07903_b200 binds
 * them with ctypes and keeps the reference API above them.
 *
 * Conventions
 *  - extern "C", plain pointers and sizes, no torch types.
 *  - All array pointers are DEVICE pointers owned by the caller unless noted
 *    "host".  Matrices are row-major with an explicit leading dimension (in
 *    elements).
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *  - No allocation inside: every entry that needs scratch has a
 *    *_workspace_bytes query; the caller passes `ws`/`ws_bytes`.
 *  - Return value: LVSK_OK or an error code mapping 1:1 onto the reference's
 *    exception classes (errors.py:4-41); lvsk_last_error() returns a
 *    thread-local message.  Device-side data errors (non-finite input) are
 *    reported through a caller-provided device flag, checked by the host
 *    after synchronisation.
 *  - Reentrant; no global mutable state except the thread-local message.
 */
#ifndef LEVSKETCH_B200_H
#define LEVSKETCH_B200_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define LVSK_API __attribute__((visibility("default")))
#else
#define LVSK_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* Status codes ↔ reference errors.py classes. */
enum {
  LVSK_OK = 0,
  LVSK_ERR_CONFIGURATION = 1, /* ConfigurationError      errors.py:38-39 */
  LVSK_ERR_DIMENSION = 2,     /* DimensionMismatchError  errors.py:18-19 */
  LVSK_ERR_FORMAT = 3,        /* FormatError             errors.py:6-7   */
  LVSK_ERR_CAPACITY = 4,      /* CapacityError           errors.py:14-15 */
  LVSK_ERR_UNSUPPORTED = 5,   /* UnsupportedFamilyError  errors.py:34-35 */
  LVSK_ERR_DEGENERATE = 6,    /* DegenerateInputError    errors.py:26-27 */
  LVSK_ERR_INCOMPATIBLE = 7,  /* IncompatibleSketchError errors.py:22-23 */
  LVSK_ERR_CUDA = 8           /* CUDA runtime failure (no reference class) */
};

/* Element type of the input matrix X. */
enum { LVSK_F32 = 0, LVSK_F64 = 1, LVSK_BF16 = 2 };

/* Device-flag bits written by kernels (OR-ed into *flags). */
enum { LVSK_FLAG_NONFINITE = 1, LVSK_FLAG_NEGATIVE = 2, LVSK_FLAG_BADINDEX = 4 };

/* One OSNAP block (CountSketch: s = 1 block covering all k rows).
 * Mirrors SketchState.__init__ (reference sketch.py:232-239). */
typedef struct {
  uint64_t a;        /* multiply-shift multiplier (odd) */
  uint64_t b;        /* multiply-shift offset */
  uint64_t sign_key; /* splitmix sign key */
  int64_t offset;    /* first sketch row of the block */
  int64_t size;      /* rows in the block */
} lvsk_hash_block;

LVSK_API const char* lvsk_last_error(void);
LVSK_API int32_t lvsk_abi_version(void);

/* Scheduling hint (no reference counterpart: the reference runs one pass at a
 * time on the CPU).  passes = how many independent pipeline passes the caller
 * keeps in flight on separate streams (paper_1812_07903_b200.BatchRunner).  At
 * >= 2 the latency-bound cooperative kernels leave SMs to the other stream's
 * HBM-bound passes: KF (lvsk_chol_fold, d <= 1024) runs at most 24 CTAs and K7
 * (lvsk_argsort_f64) gives each CTA at least 8192 keys.  Results are
 * unchanged (both kernels are deterministic for any CTA count).  Process-wide;
 * takes effect at the next launch (a captured CUDA graph keeps the value it
 * was captured with).  Default 1. */
LVSK_API int32_t lvsk_set_inflight(int32_t passes);
LVSK_API int32_t lvsk_get_inflight(void);

/* ---- K1: CountSketch / OSNAP on dense rows ------------------------------
 * Replaces SketchState._update_hashed + _scatter_add + _two_sum
 * (reference sketch.py:260-266, 173-191, 166-170) as driven by consume_rows
 * (sketch.py:289-312).  Rows X[0..n) carry GLOBAL indices row0..row0+n-1.
 * The compensated state (hi, lo), k x d float64 row-major, is read from
 * (hi_in, lo_in) and written to (hi_out, lo_out) (may alias; hi_in = lo_in = NULL
 * starts from the zero state without reading it; lo_out = NULL writes the
 * folded sketch hi + lo — the value lvsk_fold_compensated returns — to
 * hi_out instead of the pair).  Contributions to
 * one bucket are applied in ascending row index, each as a TwoSum, which is
 * the reference's exact operation sequence: the result is bit-identical.
 * blocks: HOST array of s blocks.  scale = 1/sqrt(s) (float64). */
LVSK_API size_t lvsk_hashed_workspace_bytes(int64_t n, int32_t s, int64_t k);
LVSK_API int32_t lvsk_hashed_sketch(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx,
                           uint64_t row0, const lvsk_hash_block* blocks, int32_t s, double scale,
                           const double* hi_in, const double* lo_in, double* hi_out, double* lo_out,
                           int64_t k, void* ws, size_t ws_bytes, int32_t* flags, void* stream);

/* Bucket / sign of arbitrary global indices (KAT parity of the hash family;
 * reference sketch.py:151-159).  buckets_out, signs_out: s x n. */
LVSK_API int32_t lvsk_hash_rows(const uint64_t* idx, int64_t n, const lvsk_hash_block* blocks, int32_t s,
                       int64_t* buckets_out, double* signs_out, void* stream);

/* merge(): hi_out, lo_out = TwoSum(hi1, hi2), lo1 + lo2 + err
 * (reference sketch.py:352-355); count elements; may alias the inputs. */
LVSK_API int32_t lvsk_merge_compensated(const double* hi1, const double* lo1, const double* hi2,
                               const double* lo2, double* hi_out, double* lo_out, int64_t count,
                               void* stream);

/* SketchState.data for the hashed families: out = hi + lo
 * (reference sketch.py:258); may alias. */
LVSK_API int32_t lvsk_fold_compensated(const double* hi, const double* lo, double* out, int64_t count,
                                       void* stream);

/* ---- K3: SRHT ------------------------------------------------------------
 * Replaces SketchState.data's SRHT branch + fwht (reference sketch.py:248-257,
 * 364-385): SX[t,:] = (H_m D X)[sample[t], :] / divisor, H_m unnormalised
 * Walsh-Hadamard of order m = 2^L >= n (rows >= n are the zero padding).
 * signs: m int8 (+1/-1) or NULL for all +1; sample: k int64, each in [0, m).
 * SX: k x d float64 (overwritten).  divisor = sqrt(k) for SRHT, 1 for fwht(). */
LVSK_API size_t lvsk_srht_workspace_bytes(int64_t m, int64_t d, int32_t dtype, int64_t k);
LVSK_API int32_t lvsk_srht(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx, int64_t m,
                  const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX,
                  void* ws, size_t ws_bytes, int32_t* flags, void* stream);
/* Row-block SRHT (extension: the sketch is linear in the rows, so
 * ranks holding row blocks sum their partials — the reference's
 * run_distributed rejects SRHT, dist.py:95-98, and still does here): X holds
 * the GLOBAL rows row0 .. row0+n-1 of the m-row matrix, signs the global m
 * signs; SX receives this block's contribution (/ divisor) and the sum over
 * blocks is lvsk_srht of the whole matrix.  One-pass kernel conditions: fp32
 * X, 16-byte aligned rows, d % 4 == 0, d <= 4096, k <= 4096, row0 % 2048 == 0
 * (else LVSK_ERR_UNSUPPORTED).  Workspace: lvsk_srht_workspace_bytes. */
LVSK_API int32_t lvsk_srht_rows(const float* X, int64_t n, int64_t d, int64_t ldx, int64_t row0, int64_t m,
                                const int8_t* signs, const int64_t* sample, int64_t k, double divisor, double* SX,
                                void* ws, size_t ws_bytes, int32_t* flags, void* stream);

/* ---- K4: Gaussian sketch (extension: the reference rejects "gaussian",
 * sketch.py:74-75) ----------------------------------------------------------
 * SX (+)= Z X / sqrt(k), Z[j,i] = the bf16 value with bits
 * MAG[w & 0x7FFF] | (w & 0x8000), w = 16-bit field (j & 3) of
 * mix64(key + phi ((i << 24) | (j >> 2))) — splitmix64 as a counter-based
 * stream, key = (seed_hi ^ 0x47415553) << 32 | seed_lo — and
 * MAG[L] = bf16(Phi^-1(1/2 + (L + 1/2) / 65536)): the inverse normal CDF of a
 * 16-bit uniform, the same N(0,1) (up to 16-bit quantisation and bf16
 * rounding) for every entry (csrc/gauss_gen.cuh; oracle/levsketch_oracle.py
 * gaussian_z, bit-exact).  k <= 2^26, row0 + n <= 2^40.  Rows carry global
 * indices row0..  SX: k x d float64; accumulate != 0 adds to SX instead of
 * overwriting. */
LVSK_API size_t lvsk_gaussian_workspace_bytes(int64_t n, int64_t d, int64_t k, int32_t dtype);
LVSK_API int32_t lvsk_gaussian_sketch(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx,
                             uint64_t row0, uint64_t seed, int64_t k, double* SX, int32_t accumulate,
                             void* ws, size_t ws_bytes, int32_t* flags, void* stream);
/* Materialise Z (k x n float32, row-major) for KAT parity. */
LVSK_API int32_t lvsk_gaussian_entries(uint64_t seed, int64_t k, uint64_t row0, int64_t n, float* Z,
                              void* stream);
/* The generator's magnitude table MAG (32768 bf16 bit patterns, see
 * csrc/gauss_gen.cuh), built host-side; count >= 32768. */
LVSK_API int32_t lvsk_gaussian_tables(uint16_t* out, int64_t count);

/* ---- K5: leverage pass --------------------------------------------------
 * Replaces _block_scores (reference leverage.py:88-95):
 *     scores[i] = sum_c (X[i,:] . M[:,c])^2,  i < n.
 * M is d x r row-major, float32 for F32/BF16 inputs (M_lo optional: the
 * low-order part of a float64 M split hi+lo, may be NULL) and float64 for F64
 * inputs.  scores: n float64.  Non-finite X sets LVSK_FLAG_NONFINITE. */
LVSK_API int32_t lvsk_rowsumsq_gemm(const void* X, int32_t dtype, int64_t n, int64_t d, int64_t ldx,
                           const void* M, const void* M_lo, int64_t r, double* scores,
                           int32_t* flags, void* stream);

/* K5 on tcgen05 tensor cores (fp32 X, 3xTF32 split, TMEM accumulators):
 * same result as lvsk_rowsumsq_gemm for F32 inputs, with M supplied
 * TRANSPOSED (r x d row-major) as an exact-TF32 high part Mt_hi and the
 * float32 remainder Mt_lo = M^T - Mt_hi.  Mt_hi_bf16 (optional, r x d
 * bfloat16 = bf16(Mt_hi)) selects the r <= 64 kernel that runs the x_lo
 * correction as a BF16 MMA.  Returns LVSK_ERR_UNSUPPORTED when the shape is
 * not covered (r > 128, rows not 16-byte aligned); callers then use
 * lvsk_rowsumsq_gemm. */
LVSK_API int32_t lvsk_leverage_tf32x3(const float* X, int64_t n, int64_t d, int64_t ldx, const float* Mt_hi,
                                      const float* Mt_lo, const void* Mt_hi_bf16, int64_t r, double* scores,
                                      int32_t* flags, void* stream);

/* K5 on tcgen05 for bf16 X (BASELINE config 5): Mt is (2*r_pad) x d bf16 with
 * rows [0, r) = bf16(M^T), rows [r_pad, r_pad + r) = bf16(M^T - hi), zeros
 * elsewhere; r_pad in {32, 64, 128}. */
LVSK_API int32_t lvsk_leverage_bf16(const void* X, int64_t n, int64_t d, int64_t ldx, const void* Mt, int64_t r,
                                    int64_t r_pad, double* scores, int32_t* flags, void* stream);

/* K5 operand split of a float64 fold M (d x r, row-major), one launch.
 * bf16_mode = 0: Mt_hi / Mt_lo (r x d float32) as lvsk_leverage_tf32x3 takes
 * them, and Mt_bf16 (r x d bfloat16, optional) = bf16(Mt_hi).
 * bf16_mode = 1: Mt_bf16 is the (2*r_pad) x d operand of lvsk_leverage_bf16;
 * rows [r, r_pad) and [r_pad + r, 2*r_pad) are left untouched (zero them once). */
LVSK_API int32_t lvsk_split_fold(const double* M, int64_t d, int64_t r, int32_t bf16_mode, int64_t r_pad,
                                 float* Mt_hi, float* Mt_lo, void* Mt_bf16, void* stream);

/* ---- K2 / K6: CSR rows (extension G2; BASELINE config 4) -----------------
 * Same semantics as lvsk_hashed_sketch / lvsk_rowsumsq_gemm on the densified
 * rows (bit-exact for K2: zero entries leave the TwoSum state unchanged).
 * row_ptr: n+1 int64 (row_ptr[0] may be nonzero: col/val point at element
 * row_ptr[0]); col: int32, strictly increasing per row, in [0, d);
 * val: F32 or F64.  Bad indices set LVSK_FLAG_BADINDEX, non-finite values
 * LVSK_FLAG_NONFINITE.  hi_in = lo_in = NULL means a zero input state (not
 * read); lo_out = NULL writes the folded sketch hi + lo to hi_out instead of
 * the pair (as lvsk_hashed_sketch).  K6 takes M as float32 d x r (r <= 256). */
LVSK_API size_t lvsk_hashed_csr_workspace_bytes(int64_t n, int32_t s, int64_t k);
LVSK_API int32_t lvsk_hashed_sketch_csr(const int64_t* row_ptr, const int32_t* col, const void* val,
                                        int32_t val_dtype, int64_t n, int64_t d, uint64_t row0,
                                        const lvsk_hash_block* blocks, int32_t s, double scale,
                                        const double* hi_in, const double* lo_in, double* hi_out,
                                        double* lo_out, int64_t k, void* ws, size_t ws_bytes, int32_t* flags,
                                        void* stream);
LVSK_API int32_t lvsk_rowsumsq_csr(const int64_t* row_ptr, const int32_t* col, const void* val,
                                   int32_t val_dtype, int64_t n, int64_t d, const float* M, int64_t r,
                                   double* scores, int32_t* flags, void* stream);
/* K6 with a prepared operand (r = 128; reference: the same _block_scores,
 * leverage.py:88-95).  lvsk_rowsumsq_csr_prepare turns the fold's M (float32
 * d x 128) once into bf16 [M_hi | M_lo] operand images of the hot column
 * window (the first 64 * LVSK_K6_HOTBLOCKS column ids, default 640) in `prep`
 * (lvsk_rowsumsq_csr_prep_bytes(d, r) bytes, 16-byte aligned; 0 = not
 * available for this r, use lvsk_rowsumsq_csr); lvsk_rowsumsq_csr_prepared
 * then scores CSR row blocks with the hot window on tcgen05 and only the
 * columns beyond it gathered from M.  Rows must be strictly increasing
 * (violations set LVSK_FLAG_BADINDEX). */
LVSK_API size_t lvsk_rowsumsq_csr_prep_bytes(int64_t d, int64_t r);
LVSK_API int32_t lvsk_rowsumsq_csr_prepare(const float* M, int64_t d, int64_t r, void* prep, size_t prep_bytes,
                                           void* stream);
LVSK_API int32_t lvsk_rowsumsq_csr_prepared(const int64_t* row_ptr, const int32_t* col, const void* val,
                                            int32_t val_dtype, int64_t n, int64_t d, const float* M, int64_t r,
                                            const void* prep, size_t prep_bytes, double* scores, int32_t* flags,
                                            void* stream);

/* ---- fold ------------------------------------------------------------------
 * KF: the certified Cholesky JL fold (replaces the reference's
 * svd + truncate + V'/sigma' basis, leverage.py:75-85 / svd.py:41-74, for the
 * JL variant).  G: d x d float64 symmetric (upper
 * triangle read, leading dimension ldg), Pi: d x r float64 row-major.
 * Writes M = R^-1 Pi (d x r, R^T R = G, R upper with positive diagonal) and
 * diag[3] = {info (0 = positive definite), trace(G), trace(G^-1)}; the caller
 * certifies trace(G) * trace(G^-1) < 1/sv_tol^2 before using M.  The kernel
 * also evaluates that certificate on the device: when info != 0, a trace is
 * not finite and positive, or trace(G) * trace(G^-1) >= cert_limit, it adds 1
 * to *cert_fail (if non-NULL) — so a stream of unsynchronised folds keeps a
 * count of uncertified results.  One cooperative launch; stream-capturable. */
LVSK_API size_t lvsk_chol_fold_workspace_bytes(int64_t d, int64_t r);
LVSK_API int32_t lvsk_chol_fold(const double* G, int64_t d, int64_t ldg, const double* Pi, int64_t r, double* M,
                                double* diag, double cert_limit, int32_t* cert_fail, void* ws, size_t ws_bytes,
                                void* stream);

/* KG: G = SX^T SX (k x d float64 SX, row-major, leading dimension ldsx) on
 * the int8 tensor cores (Ozaki scheme: per-column power-of-two scaling,
 * seven exact 7-bit slices, exact int32 slice products, float64 recombination;
 * error class of a float64 GEMM).  Writes the 256 x 256 block upper triangle
 * of G (ldg >= d; the entries below the diagonal blocks are untouched);
 * k <= 18000; a non-finite SX raises LVSK_FLAG_NONFINITE in *flags.
 * Replaces the Gram DGEMM of the fold (svd.py:30-37 / leverage.py:75-85
 * through factor.cu).  Stream-capturable. */
LVSK_API size_t lvsk_gram_workspace_bytes(int64_t k, int64_t d);
/* KD: the same block upper triangle (64 x 64 tiles, bi <= bj) of
 * G = SX^T SX on the float64 tensor cores (DMMA), k split into row slices
 * summed in a fixed order (deterministic); the fold's Gram for d < 2048.
 * ws: lvsk_syrk_workspace_bytes (0 bytes when one slice suffices).
 * Stream-capturable. */
LVSK_API size_t lvsk_syrk_workspace_bytes(int64_t k, int64_t d);
LVSK_API int32_t lvsk_syrk_f64(const double* SX, int64_t k, int64_t d, int64_t ldsx, double* G, int64_t ldg,
                               void* ws, size_t ws_bytes, void* stream);
LVSK_API int32_t lvsk_gram_f64(const double* SX, int64_t k, int64_t d, int64_t ldsx, double* G, int64_t ldg,
                               void* ws, size_t ws_bytes, int32_t* flags, void* stream);

/* ---- ordering -------------------------------------------------------------
 * scores_to_distribution (order.py:51-63): p = scores / sum(scores), with
 * the sum a deterministic two-level float64 reduction.  Sets
 * LVSK_FLAG_NONFINITE / LVSK_FLAG_NEGATIVE in *flags; *total receives the sum. */
LVSK_API size_t lvsk_normalize_workspace_bytes(int64_t n);
LVSK_API int32_t lvsk_normalize_scores(const double* scores, int64_t n, double* p_out, double* total,
                              void* ws, size_t ws_bytes, int32_t* flags, void* stream);
/* Deterministic float64 sum of x[0..n) into *out (device). */
LVSK_API int32_t lvsk_sum_f64(const double* x, int64_t n, double* out, void* ws, size_t ws_bytes, void* stream);

/* K7: stable argsort of float64 keys.  descending != 0 reproduces
 * np.argsort(-p, kind="stable") (make_plan "dec", order.py:89-90); descending
 * == 0 reproduces np.argsort(keys, kind="stable") ("dec_swor", order.py:95-99).
 * NaNs sort last; -0.0 == +0.0.  idx_out: n int64. */
LVSK_API size_t lvsk_argsort_workspace_bytes(int64_t n);
LVSK_API int32_t lvsk_argsort_f64(const double* keys, int64_t n, int32_t descending, int64_t* idx_out,
                         void* ws, size_t ws_bytes, void* stream);

/* KM: the multi-rank global order.  R runs in global (rank) order, run q of
 * length run_off[q+1] - run_off[q] (run_off: HOST array of R + 1 offsets,
 * run_off[0] = 0); each rank sorted its run with lvsk_argsort_f64: run_idx
 * holds that local stable order (int32, local to the run) and sorted_keys the
 * run's keys in that order (keys_q[run_idx_q[i]]), both concatenated run
 * after run.  idx_out (n int64) receives the stable argsort of the
 * concatenated keys — identical to lvsk_argsort_f64 on them (make_plan "dec"
 * over all ranks, order.py:89-90; run_distributed concatenates the
 * per-worker scores in worker order, dist.py:126-129).  A local index outside
 * its run sets LVSK_FLAG_BADINDEX. */
LVSK_API size_t lvsk_merge_runs_workspace_bytes(int64_t n, int32_t runs);
LVSK_API int32_t lvsk_merge_argsort_runs(const double* sorted_keys, const int32_t* run_idx, const int64_t* run_off,
                                int32_t runs, int32_t descending, int64_t* idx_out, void* ws, size_t ws_bytes,
                                int32_t* flags, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* LEVSKETCH_B200_H */
