/*
 * krr_b200.h — C-ABI of the B200-native sketch-preconditioned KRR hot path.
 *
 * This is the drop-in boundary for the reference's C++ operator / preconditioner /
 * solver interfaces (reference = /root/reference/proj, a CPU-only Eigen library).
 * Every entry point below names the reference interface it replaces (file:line).
 * Plain pointers and sizes only; no torch, no Eigen, no C++ types.
 *
 * Conventions (mirroring the reference):
 *   - All matrices are ROW-MAJOR fp64 (reference types.hpp:11-13: Matrix is
 *     Eigen::RowMajor).  Multi-column vectors (n x t) are row-major too.
 *   - Host pointers in, host pointers out, unless the function name ends in
 *     `_device` (then all array pointers are device pointers on the context's GPU).
 *   - Every function returns a krr_status.  On failure, krr_last_error() returns a
 *     thread-local message.  Status codes map 1:1 onto the reference's exception
 *     types (types.hpp:18-64); the Python / C++ mirrors rethrow the matching type.
 *   - Calls are synchronous at return (the reference's pure-function semantics).
 *     A context is used by one host thread at a time.
 *   - There is no CPU fallback: every compute entry point runs CUDA kernels on the
 *     context's device and fails with KRR_ERR_CUDA if the device is unusable.
 */
#ifndef KRR_B200_H
#define KRR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRR_B200_ABI_VERSION 1

typedef enum krr_status {
    KRR_OK = 0,
    KRR_ERR_DIMENSION_MISMATCH = 1,    /* types.hpp:18  DimensionMismatch   (std::invalid_argument) */
    KRR_ERR_NOT_POSITIVE_DEFINITE = 2, /* types.hpp:22  NotPositiveDefinite (std::runtime_error)   */
    KRR_ERR_SINGULAR_TRIANGULAR = 3,   /* types.hpp:26  SingularTriangular  (std::runtime_error)   */
    KRR_ERR_BREAKDOWN = 4,             /* types.hpp:48  BreakdownDetected   (std::runtime_error)   */
    KRR_ERR_NON_POSITIVE_LAMBDA = 5,   /* types.hpp:38  NonPositiveLambda   (std::invalid_argument) */
    KRR_ERR_INVALID_ARGUMENT = 6,      /* std::invalid_argument thrown by validate()/pcg_solve      */
    KRR_ERR_CUDA = 7,                  /* device error (no reference equivalent)                   */
    KRR_ERR_NCCL = 8,                  /* collective error (no reference equivalent)               */
    KRR_ERR_STATE = 9,                 /* call out of order (e.g. matvec before krr_set_data)      */
    KRR_ERR_CALLBACK = 10,             /* a user operator callback reported failure                */
    KRR_ERR_IO = 11,                   /* model file I/O or format error (std::runtime_error, io.cpp) */
    KRR_ERR_NO_CONVERGENCE = 12        /* types.hpp:34  NoConvergence       (std::runtime_error)   */
} krr_status;

typedef struct krr_ctx krr_ctx;

/* Per-right-hand-side PCG statistics: reference solver.hpp:29-34 (RhsStats).
 * residual_history is returned through a separate caller buffer. */
typedef struct krr_rhs_stats {
    int32_t iterations;
    int32_t converged;
    double final_residual;
} krr_rhs_stats;

/* ---------------------------------------------------------------- misc */
const char* krr_last_error(void);
int krr_abi_version(void);
/* Number of CUDA devices visible (0 on a CPU-only host; never an error). */
int krr_device_count(void);

/* ---------------------------------------------------------------- context */
/* Single-GPU context on `device`. */
int krr_ctx_create(int device, krr_ctx** out);
/* Rank `rank` of `world` (one process per GPU).  `nccl_id` is the 128-byte
 * ncclUniqueId produced by krr_nccl_unique_id on rank 0 and broadcast by the
 * caller (bench.py uses torch.distributed for that broadcast only).  world = 1 gives a
 * one-rank communicator (the data path then needs no collective). */
int krr_nccl_unique_id(void* out_128_bytes);
int krr_ctx_create_dist(int device, int rank, int world, const void* nccl_id, krr_ctx** out);
int krr_ctx_destroy(krr_ctx* ctx);
/* Number of kernels this context launched so far (bench.py's gpu_launches claim). */
int krr_ctx_launch_count(krr_ctx* ctx, int64_t* out);

/* Tuning / diagnostic knobs (no reference equivalent):
 *   "k1_path"     -1|0|1|3  fused mat-vec kernel: auto (default: INT8-slice tensor-core kernel
 *                         where faster: 27 <= d <= 96, when the data's exponent range allows, else FP64 DMMA) |
 *                         FP64 DMMA | tcgen05 INT8 slices | K1-I8X (INT8 slices, exact integer exp argument;
 *                         Gaussian, d <= 96, |x| sqrt(2 scale) < 256; otherwise the request runs the auto choice)
 *   "k1t_path"    -1|0|1  16-column batches of multi-RHS mat-mats / batched PCG: auto (default:
 *                         K1T-I8 — INT8-slice dot products on K-streamed operands + DMMA E.V —
 *                         for the Gaussian kernel with 20 <= d <= 448, else the DMMA K1T) |
 *                         DMMA K1T | K1T-I8 where supported
 *   "k1_resident" 1|0  keep the column tile of the DMMA mat-vec in shared memory (default 1)
 *   "k1_warps" 8|16, "k1_grouped" 1|0  DMMA mat-vec shape (defaults 8, 1)
 *   "batched_rhs" 1|0  multi-RHS solves / mat-mats through the batched kernel (default 1)
 *   "exp_mode"    1|0  table exp (default) | libdevice exp in the Gaussian epilogue
 *   "i8_debug"    bits  profiling only (K1-I8: 1 skip MMAs, 2 skip exp, 4 clock trace;
 *                         K1T-I8: 4 clock trace)
 *   "pcg_graph"   1|0  single-RHS device PCG as one CUDA graph (conditional WHILE node, device-side
 *                         stop / breakdown decision; default 1) | host-driven loop; same iterates
 *   "emulate_world" W, "emulate_rank" r   test only, single-rank contexts: the next
 *                         krr_set_data builds rank r of W's K1 schedule (tiles, owned slots,
 *                         diagonal on rank 0) with no collective, so K v returns that rank's
 *                         partial — the multi-rank K1 checked on one GPU (sum over r = K v)
 *   "poison_batched" 1|0  test only: fill the batched (t > 1) PCG vectors with NaN bytes whenever
 *                         they are (re)used, standing in for stale contents of an earlier call
 *   "nccl_always" 1|0  test only, contexts with a communicator: run the collectives even with
 *                         world = 1 (identity all-reduces), so one GPU exercises the multi-rank
 *                         data path, NCCL inside the graph-resident PCG loop included */
int krr_set_option(krr_ctx* ctx, const char* key, double value);
/* Arithmetic of the fused mat-vec (SURVEY §8b krr_set_precision; north-star "optional fp32
 * mode, reported separately"): 64 = fp64, oracle-matching (default); 32 = fp32-accuracy K1
 * (three bf16 parts per value on tcgen05 kind::f16, fp32 epilogue, d <= 128; relative error
 * of K v ~1e-6).  PCG vectors, dots and the preconditioner stay fp64 in both modes;
 * multi-RHS solves run column by column in fp32 mode. */
int krr_set_precision(krr_ctx* ctx, int bits);
/* the sketch-and-solve random-features baseline of `krr bench`.
 * train_random_features_baseline (solver.cpp:175-193): w (s x t, row-major) =
 * (Z^T Z + lambda I)^{-1} Z^T Y with Z = RFF(X of krr_set_data; W s x d, b s from
 * krr_rff_realize), no jitter (NotPositiveDefinite on failure).  Single-rank. */
int krr_rf_baseline_train(krr_ctx* ctx, const double* W, const double* b, int64_t s, const double* Y, int64_t t,
                          double lambda, double* w_out);
/* baseline_predict_scores (solver.cpp:195-197): out (m x t) = RFF(Xq) w. */
int krr_rf_baseline_predict(krr_ctx* ctx, const double* Xq, int64_t m, const double* W, const double* b, int64_t s,
                            const double* w, int64_t t, double* out);
/* the reference's KRRM model file (io.cpp:192-261), byte-identical layout
 * ("KRRM", version 1, metadata JSON as nlohmann dumps it, X n x d, C n x t fp64), so models
 * trained here feed the reference's `krr predict` / `krr eval`.  Gaussian models only.
 * Errors (bad magic, unsupported version, truncation, trailing bytes, non-finite entries,
 * invalid dimensions) -> KRR_ERR_IO with the reference's messages. */
int krr_model_save(const char* path, double sigma, double lambda, uint64_t seed, const double* label_map,
                   int64_t nlabels, const double* X, int64_t n, int64_t d, const double* C, int64_t t);
int krr_model_info(const char* path, int64_t* n, int64_t* d, int64_t* t, int64_t* nlabels, double* sigma,
                   double* lambda, uint64_t* seed);
int krr_model_load(const char* path, double* label_map, double* X, double* C);
/* QualityReport (precond.hpp:35-47). */
typedef struct krr_quality_report {
    int32_t passed;
    int32_t pad_;
    double cond1_value;          /* |(I-P) K (I-P)| by power iteration */
    double cond2_ratio_low;      /* eigenvalue range of Sigma^-1 (B'KB) Sigma^-1 on range(P) */
    double cond2_ratio_high;
    int64_t rank_of_p;
    int64_t sketch_size;
    double lambda;
    double cond1_threshold;      /* 0.1 lambda */
    double spectrum_cut;         /* 0.05 lambda */
    double ratio_low_threshold;  /* 0.9 */
    double ratio_high_threshold; /* 1.1 */
} krr_quality_report;
/* quality_test (precond.cpp:60-100) of the context's raw sketch (after krr_rff_build /
 * krr_sketch_upload, before krr_precond_build) against the Gaussian K of krr_set_data:
 * eig(Z'Z) by cuSOLVER syevd, the retained basis by GEMM, condition 1 by power iteration
 * through the fused K1 (start vector from mt19937_64(7), tol 1e-4, 500 iterations),
 * condition 2 through the multi-RHS K1T.  Single-rank. */
int krr_quality_test(krr_ctx* ctx, double lambda, krr_quality_report* out);
/* adaptive_build (precond.cpp:107-138) for the Gaussian / RFF chain: s = s0, doubling
 * until quality_test passes or s reaches s_max; attempt a draws its RFF map with master
 * seed master_seed + a * 0xD1B54A32D192ED03 (sketches.hpp:16); then builds the Woodbury
 * preconditioner (lambda_p, jitter retry) from the final sketch on the context.
 * history (nullable) receives up to max_history reports. */
int krr_adaptive_build(krr_ctx* ctx, double lambda, double lambda_p, int64_t s0, int64_t s_max,
                       uint64_t master_seed, krr_quality_report* history, int max_history, int* n_history,
                       int64_t* final_size, int* passed, int* jitter_used);
/* Read a knob back: "k1_path", "k1t_path", "exp_mode", "batched_rhs", and (after krr_set_data)
 * "k1_path_effective" (0 DMMA / 1 I8 / 2 column 0 of a 16-column K1T-I8 pass, d >= 160 / 3 K1-I8X:
 * the kernel a mat-vec runs now), "i8x_exponent" (K1-I8X's global exponent E, 0 when not prepared
 * or out of range), "k1t_path_effective"
 * (the kernel a 16-column batch runs now; may prepare the K1T-I8 operands), "i8_supported",
 * "precision" (64 | 32), "build_gram_ms" / "build_cholesky_ms" / "build_trsm_ms" (CUDA-event
 * split of the last krr_precond_build: Z^T Z + lambda_p I, Cholesky with its retry, U = L^-1 Z^T)
 * and "nccl_nranks" (ncclCommCount of the context's communicator; 1 without one). */
int krr_get_option(krr_ctx* ctx, const char* key, double* value);

/* ---------------------------------------------------------------- data + kernel operator */
/* Uploads X (n x d, row-major) to the device (replicated on every rank) and
 * precomputes the row norms.  Replaces the data half of gram_matrix
 * (kernels.cpp:72-77).  sigma > 0 (KernelSpec::validate, kernels.cpp:37-38). */
int krr_set_data(krr_ctx* ctx, const double* X, int64_t n, int64_t d, double sigma);

/* out = (K + lambda I) V for the Gaussian kernel, K never stored.  V and out are
 * n x t row-major host buffers.  Replaces the dense `apply_a` lambda of
 * solve_regularized (solver.cpp:75-77) applied to gram_matrix (kernels.cpp:72-88):
 * K_ij = exp(-max(0, |x_i|^2 + |x_j|^2 - 2 x_i.x_j) / (2 sigma^2)), K_ii = 1,
 * exact symmetry.  This is the LinearOperator adapter (solver.hpp:15). */
int krr_kernel_matvec(krr_ctx* ctx, double lambda, const double* V, int64_t t, double* out);
/* Same with device-resident V/out (n x t, row-major, on the context's device). */
int krr_kernel_matvec_device(krr_ctx* ctx, double lambda, const double* dV, int64_t t,
                             double* dOut);

/* Rectangular K(A, X)·C with A = Xq (m x d host), the support set being the data
 * already set on the context: cross_gram(Xq, X)·C (kernels.cpp:103-121,
 * solver.cpp:135-139, predict_scores).  No diagonal forcing.  C is n x t. */
int krr_predict_scores(krr_ctx* ctx, const double* Xq, int64_t m, const double* C, int64_t t,
                       double* out);

/* ---------------------------------------------------------------- random Fourier features */
/* Host-side, reference-identical draw of the RFF tables: RffMap ctor
 * (sketches.cpp:24-35) seeded with stage_seed(master, 0) (sketches.cpp:18-20):
 * mt19937_64(master + 0x9E3779B97F4A7C15); W (s x d) row by row from
 * normal_distribution(0, 1/sigma), then b (s) from uniform_real_distribution(0, 2pi).
 * Pure host RNG (libstdc++), no device needed. */
int krr_rff_realize(uint64_t master_seed, int64_t d, int64_t s, double sigma, double* W,
                    double* b);
/* Z = sqrt(2/s) cos(X W^T + b) on the device for the context's data
 * (RffMap::apply + SketchChain::apply_rows, sketches.cpp:37-41,207-211).
 * Z stays on the device (row-sharded across ranks). */
int krr_rff_build(krr_ctx* ctx, const double* W, const double* b, int64_t s);
/* Download the device Z (n x s row-major) — test/inspection helper. */
int krr_rff_download(krr_ctx* ctx, double* Z);
/* Upload an explicit Z (n x s) instead of building it from W, b — lets
 * build_preconditioner(z, lambda_p) (precond.hpp:28) take any sketch. */
int krr_sketch_upload(krr_ctx* ctx, const double* Z, int64_t n, int64_t s);

/* solve_regularized (solver.hpp:82-84, solver.cpp:69-94) with the reference's own signature: a
 * caller-supplied dense K (n x n row-major, symmetric), Y n x t; A v = K v + lambda v on the
 * device (cuBLAS DGEMV), M = the context's Woodbury preconditioner when use_precond (built for
 * n rows).  Per-column PCG as the reference's sequential loop.  Single rank.  The on-the-fly
 * path (krr_set_data + krr_pcg_solve) is the one that scales: K is n^2 doubles here. */
int krr_solve_regularized_dense(krr_ctx* ctx, const double* K, int64_t n, const double* Y, int64_t t, double lambda,
                                int use_precond, double tau, int max_iter, double* C, krr_rhs_stats* stats,
                                double* residual_history, int64_t* total_matvecs);

/* ---------------------------------------------------------------- kernel families + sketch chains */
/* KernelSpec (kernels.hpp:15-27).  family 0 = Gaussian (sigma > 0), 1 = polynomial
 * k(x, z) = (gamma x.z + offset)^degree (gamma > 0, offset >= 0, degree >= 1);
 * KernelSpec::validate's rules and messages (kernels.cpp:36-44) -> KRR_ERR_INVALID_ARGUMENT. */
typedef struct krr_kernel_spec {
    int32_t family;
    int32_t degree;
    double sigma;
    double gamma;
    double offset;
} krr_kernel_spec;
/* krr_set_data for either family.  For the polynomial kernel the fused K1 / K1T kernels
 * contract the augmented inputs [sqrt(gamma) x, sqrt(offset)] (kernels.cpp:56-62) on the
 * FP64 tensor path and raise p_ij to the degree in the epilogue (ipow, kernels.cpp:10-14);
 * K_ii = ipow(|xa_i|^2) is applied by the finish kernel (kernels.cpp:89-99 keeps the
 * diagonal, unlike the Gaussian K_ii = 1).  The polynomial kernel runs on the DMMA K1 or on
 * K1-I8 (INT8 slices, p = gamma x.z + c formed in the epilogue; auto for d >= 55); the fp32
 * mode is Gaussian-only (precision 32 is rejected). */
int krr_set_data_kernel(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const krr_kernel_spec* kernel);

/* ChainSpec (sketches.hpp:96-107): first 0 = RandomFourier (Gaussian kernel), 1 =
 * TensorSketch (polynomial kernel); optional SRHT stage s2 and Gaussian stage s3 (0 = absent),
 * non-increasing sizes (ChainSpec::validate, sketches.cpp:155-165). */
typedef struct krr_chain_spec {
    int32_t first;
    int32_t pad_;
    int64_t s1, s2, s3;
} krr_chain_spec;
/* A realized SketchChain's tables (sketches.hpp:109-127), caller-owned host arrays.  Unused
 * stages' pointers may be NULL.  in_dim = d (RFF) or d + 1 (TensorSketch on augmented inputs).
 *   rff_w s1 x d, rff_b s1                      (RffMap)
 *   ts_hash degree x in_dim, ts_sign same       (TensorSketchMap)
 *   srht_sign next_pow2(s1), srht_rows s2       (SrhtMap)
 *   gauss_proj s3 x (s2 ? s2 : s1)              (GaussianMap) */
typedef struct krr_chain_tables {
    int32_t first;
    int32_t degree;
    int64_t in_dim, s1, s2, s3;
    const double* rff_w;
    const double* rff_b;
    const uint32_t* ts_hash;
    const double* ts_sign;
    const double* srht_sign;
    const int64_t* srht_rows;
    const double* gauss_proj;
} krr_chain_tables;
/* Host-side, reference-identical stage draws with the map's OWN seed (realize_chain applies
 * stage_seed(master, k) = master + (k+1) 0x9E3779B97F4A7C15 for stage k = 0, 1, 2):
 * TensorSketchMap ctor (sketches.cpp:51-69), SrhtMap ctor (:95-109), GaussianMap ctor (:128-135). */
int krr_tensorsketch_realize(uint64_t seed, int64_t in_dim, int64_t s, int degree, uint32_t* hash, double* sign);
int krr_srht_realize(uint64_t seed, int64_t in_dim, int64_t s, double* sign, int64_t* rows);
int krr_gaussmap_realize(uint64_t seed, int64_t in_dim, int64_t s, double* proj);
/* SketchChain::apply_rows (sketches.cpp:194-211) on the device for m query rows Xq (m x d,
 * the context's d and kernel): Z (m x out_dim, host).  RFF stage = K2; TensorSketch = count
 * sketches + radix-2 transforms in shared memory (bitwise the reference algorithm's
 * operations); SRHT = pad / sign / Walsh-Hadamard / sample (bitwise); Gaussian stage = DGEMM. */
int krr_chain_apply(krr_ctx* ctx, const krr_chain_tables* tables, const double* Xq, int64_t m, double* Z);
/* The same for the context's own data, kept on the device as the sketch Z (row-sharded),
 * ready for krr_precond_build / krr_quality_test (generalises krr_rff_build). */
int krr_chain_build(krr_ctx* ctx, const krr_chain_tables* tables);
/* realize_chain (sketches.cpp:213-242) + krr_chain_build: draws every stage on the host from
 * master_seed and builds Z on the device. */
int krr_chain_build_seeded(krr_ctx* ctx, const krr_chain_spec* spec, uint64_t master_seed);
/* ChainSpec::scaled_to (sketches.cpp:173-192). */
int krr_chain_scaled_to(const krr_chain_spec* spec, int64_t target, krr_chain_spec* out);
/* train (solver.cpp:96-133) for any kernel family and chain: set data, realize + build the
 * chain, Woodbury build (lambda_p <= 0 -> lambda), device PCG; arguments otherwise as krr_train. */
int krr_train_ex(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const double* Y, int64_t t,
                 const krr_kernel_spec* kernel, const krr_chain_spec* chain, double lambda, double lambda_p,
                 uint64_t master_seed, double tau, int max_iter, double* C, krr_rhs_stats* stats,
                 double* residual_history, int64_t* total_matvecs, double* phase_ms);
/* adaptive_build (precond.cpp:107-138) for any chain template (scaled_to(s) per attempt). */
int krr_adaptive_build_ex(krr_ctx* ctx, const krr_chain_spec* chain_template, double lambda, double lambda_p,
                          int64_t s0, int64_t s_max, uint64_t master_seed, krr_quality_report* history,
                          int max_history, int* n_history, int64_t* final_size, int* passed, int* jitter_used);
/* train_random_features_baseline (solver.cpp:175-193) / baseline_predict_scores (:195-197)
 * for any realized chain. */
int krr_rf_baseline_train_ex(krr_ctx* ctx, const krr_chain_tables* tables, const double* Y, int64_t t,
                             double lambda, double* w_out);
int krr_rf_baseline_predict_ex(krr_ctx* ctx, const krr_chain_tables* tables, const double* Xq, int64_t m,
                               const double* w, int64_t t, double* out);
/* KRRM model file with the kernel spec (io.cpp:73-89 kernel_to_json / kernel_from_json). */
int krr_model_save_ex(const char* path, const krr_kernel_spec* kernel, double lambda, uint64_t seed,
                      const double* label_map, int64_t nlabels, const double* X, int64_t n, int64_t d,
                      const double* C, int64_t t);
int krr_model_kernel(const char* path, krr_kernel_spec* kernel);

/* ---------------------------------------------------------------- preconditioner */
/* build_preconditioner (precond.cpp:20-40): G = Z^T Z + lambda_p I; Cholesky;
 * on failure retry ONCE with 1e-12 trace(G)/s added to the diagonal, then
 * KRR_ERR_NOT_POSITIVE_DEFINITE; U = L^-1 Z^T (stored in place of Z).
 * lambda_p <= 0 -> KRR_ERR_NON_POSITIVE_LAMBDA.  *jitter_used (nullable)
 * reports whether the retry fired. */
int krr_precond_build(krr_ctx* ctx, double lambda_p, int* jitter_used);
/* Preconditioner::apply / apply_columns (precond.cpp:10-18):
 * out = (R - U^T (U R)) / lambda_p, R and out n x t row-major host buffers. */
int krr_precond_apply(krr_ctx* ctx, const double* R, int64_t t, double* out);
/* Download U (s x n row-major, the reference's Preconditioner::u) — test helper. */
int krr_precond_download_u(krr_ctx* ctx, double* U);
/* Read a block of Preconditioner::u (precond.hpp:16, a public member): out (nrows x ncols,
 * row-major) = U[row0 : row0 + nrows, cols[0..ncols)] — the rows are sketch features, the
 * columns data points (zero for columns in another rank's shard).  Lets a caller inspect U
 * at sizes where downloading all s x n of it is impractical (64 GiB at BASELINE config 4). */
int krr_precond_read_u(krr_ctx* ctx, int64_t row0, int64_t nrows, const int64_t* cols, int64_t ncols,
                       double* out);
int krr_precond_drop(krr_ctx* ctx);

/* ---------------------------------------------------------------- PCG */
/* Device-resident PCG on (K + lambda I) C = Y for the context's data
 * (solve_regularized, solver.cpp:69-94, per-column semantics of pcg_solve,
 * solver.cpp:22-67: x0 = 0, recursive residual, stop when |r|/|y| <= tau,
 * BreakdownDetected if p'Ap <= 0).  use_precond != 0 uses the built
 * preconditioner, else plain CG (null M, solver.cpp:37,60).
 * Y, C: n x t row-major host buffers.  stats: t entries.  residual_history
 * (nullable): t x max_iter row-major, entries past stats[j].iterations untouched.
 * total_matvecs (nullable) = sum of iterations (solver.cpp:88). */
int krr_pcg_solve(krr_ctx* ctx, double lambda, const double* Y, int64_t t, double tau,
                  int max_iter, int use_precond, double* C, krr_rhs_stats* stats,
                  double* residual_history, int64_t* total_matvecs);

/* Generic pcg_solve (solver.hpp:55-57) over caller operators: the PCG vector
 * algebra runs on the device; apply_a / apply_m are host callbacks
 * (in, out are host arrays of length n; return 0 on success).  apply_m may be
 * NULL (plain CG).  observer (nullable) sees (it, x) after each update
 * (solver.cpp:54).  Used by the drop-in LinearOperator form of the API. */
typedef int (*krr_operator_cb)(void* user, const double* in, double* out, int64_t n);
typedef void (*krr_observer_cb)(void* user, int it, const double* x, int64_t n);
int krr_pcg_solve_operator(krr_ctx* ctx, int64_t n, krr_operator_cb apply_a, void* user_a,
                           krr_operator_cb apply_m, void* user_m, const double* y, double tau,
                           int max_iter, krr_observer_cb observer, void* user_obs, double* x,
                           krr_rhs_stats* stats, double* residual_history);

/* ---------------------------------------------------------------- end-to-end train */
/* train (solver.cpp:96-133) for the Gaussian kernel with a single RFF stage
 * (ChainSpec{RandomFourier, s1 = s}): set data, realize the chain with
 * master_seed, build Z on the device, build the preconditioner (lambda_p <= 0
 * means "defaults to lambda", solver.cpp:102), solve every column.
 * X n x d, Y n x t, C out n x t (host).  phase_ms (nullable, 4 doubles):
 * rff build, precond build, solve, total — CUDA-event timed. */
int krr_train(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const double* Y, int64_t t,
              double sigma, double lambda, double lambda_p, int64_t s, uint64_t master_seed,
              double tau, int max_iter, double* C, krr_rhs_stats* stats,
              double* residual_history, int64_t* total_matvecs, double* phase_ms);

/* ---------------------------------------------------------------- schedule (host only) */
/* The symmetric super-tile schedule of the fused kernel mat-vec, exported so the
 * multi-rank partition can be checked on a CPU-only host.  For n points and
 * `world` ranks: *super_rows receives the super-tile edge (rows), *num_super the
 * number of super-rows NS, and (if tiles != NULL, capacity max_tiles) the
 * (a, b) pairs (a <= b) owned by `rank`, flattened.  *num_tiles = count. */
int krr_schedule(int64_t n, int world, int rank, int64_t* super_rows, int64_t* num_super,
                 int32_t* tiles, int64_t max_tiles, int64_t* num_tiles);

/* Row shard [*row_begin, *row_end) of the n sketch rows (Z / U) owned by `rank`:
 * contiguous equal blocks of ceil(n / world) rows. */
int krr_shard_rows(int64_t n, int world, int rank, int64_t* row_begin, int64_t* row_end);

/* ---------------------------------------------------------------- synthetic configs */
/* Deterministic generators for BASELINE.json configs 1-5.
 * cfg in 1..5; X n x d, Y n x t (host).  Pure host code (libstdc++ RNG). */
int krr_generate_config(int cfg, int64_t n, int64_t d, int64_t t, uint64_t seed, double* X,
                        double* Y);
/* rlsc_encode (solver.cpp:152-161): +1 for the true class, -1 otherwise. */
int krr_rlsc_encode(const int32_t* classes, int64_t n, int32_t num_classes, double* Y);

/* ---------------------------------------------------------------- measurement */
/* Runs `steps` device-resident (K + lambda I) v mat-vecs (K1 + finish + the
 * all-reduce when world > 1) back to back on the context's stream over a
 * seeded N(0,1) vector and CUDA-event-times them: *total_ms = whole span,
 * *k1_ms = mean duration of the fused K1 kernel launch alone (per step). */
int krr_bench_matvec(krr_ctx* ctx, double lambda, int steps, double* total_ms, double* k1_ms);

/* Diagnostics (micro-benchmarks, tcgen05 probes, kernel clock traces) live in a separate
 * library, libkrr_diag.so (include/krr_diag.h); this header is the drop-in interface only. */

#ifdef __cplusplus
}
#endif

#endif /* KRR_B200_H */
