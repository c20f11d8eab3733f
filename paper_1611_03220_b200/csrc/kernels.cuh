// Host-side launch interface of every CUDA kernel in the library.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "gauss_exp.cuh"

namespace krr {

// ---------------------------------------------------------------- K1 Gaussian mat-vec
struct GaussMatvecPlan {
    const double* L = nullptr;     // n_pad x dp, [x, |x|^2, 1, 0...]
    const double* R = nullptr;     // n_pad x dp, [-2x, 1, |x|^2, 0...]
    const int2* tiles = nullptr;   // owned super-tiles (a <= b)
    int64_t num_tiles = 0;
    const uint8_t* owned = nullptr;  // NS x NS ownership (nullptr: all owned)
    const double* exp_tab = nullptr; // 64 doubles
    int64_t n = 0, n_pad = 0;
    int dp = 0, st = 0, ns = 0;
    bool resident = true;            // keep R_J in shared memory when it fits
    bool warps16 = false;            // 16 warps x (32 x 32) instead of 8 warps x (64 x 32)
    bool grouped = true;             // two phase-offset warp groups (resident shape only)
    ExpConsts ec{};
    const double* kdiag = nullptr;   // polynomial kernel: K_ii per row (nullptr: K_ii = 1)
};
size_t gauss_matvec_smem_bytes(int st);
bool gauss_matvec_resident_ok(int st, int dp);
void gauss_matvec_launch(const GaussMatvecPlan& p, const double* v, double* part, int exp_mode,
                         cudaStream_t stream);
void matvec_finish_launch(const GaussMatvecPlan& p, const double* part, const double* v,
                          double lambda, int add_diag, double* out, cudaStream_t stream);

// K1T: OUT = (K + lambda I) V for T in {8, 16} interleaved right-hand sides (n_pad x T),
// part is NS x n_pad x T.
void gauss_matmat_launch(const GaussMatvecPlan& p, const double* v, int T, double* part, int mode,
                         cudaStream_t stream);
void matmat_finish_launch(const GaussMatvecPlan& p, const double* part, const double* v, int T,
                          double lambda, int add_diag, double* out, cudaStream_t stream);

// K1T-I8: T = 16 right-hand sides, tcgen05 kind::i8 dot products with K-streamed slices and
// DMMA E.V contractions (gauss_matmat_i8.cu).  Gaussian kernel, d <= 448.
int i8s_kp(int64_t d);
size_t i8s_slice_bytes(int64_t n_pad, int64_t d);  // bytes of the K-chunk-major slice buffer
bool i8s_supported(int64_t d, int st);
bool i8s_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp, double kscale,
                        uint8_t* S, int* ex, int* ejs, double* sqs, cudaStream_t stream);
void gauss_matmat_i8_launch(const GaussMatvecPlan& p, const uint8_t* S, const int* ex, const int* ejs,
                            const double* sqs, const double* v, double* part, int kp, cudaStream_t stream,
                            int debug = 0);
void i8s_read_trace(long long* out, int count);
constexpr int64_t kI8T1MinD = 160;  // single-RHS K v through K1T-I8 from d = 160 (when K1-I8 does not apply)
constexpr int64_t kI8TMinD = 20;  // auto path: K1T-I8 from d = 20 (measured crossover, profiles/r2_k1t_i8_crossover.log)

// K1-I8X: K1-I8's tensor-core dot products with an integer exp epilogue that overlaps the MMAs
// (gauss_matvec_i8x.cu).  Gaussian kernel, d <= 96.  prepare returns the global exponent E of
// z = sqrt(2 scale) x (1..8), or 0 when the data is out of its fixed-point range.
bool i8x_supported(int64_t d, int st);
void i8x_read_trace(long long* out, int count);
int i8x_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, double scale, uint8_t* S, long long* sq,
                       cudaStream_t stream);
void gauss_matvec_i8x_launch(const GaussMatvecPlan& p, const uint8_t* S, const long long* sq, int E, const double* v,
                             double* part, int kp, cudaStream_t stream, int debug = 0);

// K1-I8: tcgen05 kind::i8 slice path (gauss_matvec_i8.cu).  Supported for d <= 96.
bool i8_supported(int64_t d, int st);
// K1-F32 (optional fp32-accuracy mode, gauss_matvec_f32.cu): three bf16 parts per value on
// tcgen05 kind::f16, fp32 epilogue.  d <= 128.
bool f32_supported(int64_t d, int st);
int f32_kb(int64_t d);
void f32_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp, double scale,
                        uint8_t* S, float* s, cudaStream_t stream);
void gauss_matvec_f32_launch(const GaussMatvecPlan& p, const uint8_t* S, const float* s, const double* v,
                             float* v32, double* part, int kb, double scale, cudaStream_t stream);
void i8_read_trace(long long* out, int count);
int i8_kp(int64_t d);
// Builds the slices S, row exponents ex (and ex << 20), sq' = kscale' |x|^2 (kscale' of the
// 1/256-octave exp); returns false when the data's exponent range would leave the range
// the fused epilogue handles.
// poly_gamma > 0: prepare for the polynomial kernel (the sq' terms are unused).
bool i8_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp,
                       double kscale, uint8_t* S, int* ex, int* ejs, double* sqs, cudaStream_t stream,
                       double poly_gamma = 0.0);
// poly_degree > 0: the polynomial kernel's epilogue (p = gamma x.z + offset, ipow) instead of exp.
void gauss_matvec_i8_launch(const GaussMatvecPlan& p, const uint8_t* S, const int* ex, const int* ejs,
                            const double* sqs, const double* v, double* part, int kp, cudaStream_t stream,
                            int debug = 0, int poly_degree = 0, double poly_gamma = 0.0, double poly_offset = 0.0);

// Build L / R operands from X (n x d) on the device; rows >= n and cols >= d+2 zeroed.
void build_operands_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, int dp,
                           double* L, double* R, cudaStream_t stream);

// Rectangular cross kernel: out[m] = sum_j exp(-max(0,|a|^2+|x_j|^2-2 a.x_j) scale) c_j
// (predict_scores, solver.cpp:135-139; no diagonal forcing).  Simple DMMA-free
// reference-speed kernel (not on the PCG hot path).
void cross_matvec_launch(const double* Xq, int64_t m, const double* X, int64_t n, int64_t d,
                         const double* c, int64_t t, double scale, double* out,
                         cudaStream_t stream);

// ---------------------------------------------------------------- SURVEY 8f4 (sketch.cu)
// Polynomial-kernel operands L = R = [sqrt(gamma) x, sqrt(c), 0...] (rows >= n zero) and
// kdiag_i = ipow(|xa_i|^2, degree) (nullable; R nullable).
void poly_operands_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, int dp, double sg, double so,
                          int degree, double* L, double* R, double* kdiag, cudaStream_t stream);
// predict_scores for the polynomial kernel: out (m x t) = K(Xq, X) C.
void cross_poly_launch(const double* Xq, int64_t m, const double* X, int64_t n, int64_t d, const double* c,
                       int64_t t, double sg, double so, int degree, double* out, cudaStream_t stream);
// TensorSketch rows: A (m rows, stride lda, in_dim entries) -> Z (m x s).  P = s when s is a
// power of two, else next_pow2(degree (s-1) + 1); tw_* from fft_twiddles(P).  scratch:
// tensorsketch_scratch(P, m) double2 elements (0 -> nullptr allowed).
size_t tensorsketch_scratch(int64_t P, int64_t m);
void tensorsketch_launch(const uint32_t* hash, const double* sign, const double2* tw_fwd, const double2* tw_inv,
                         int64_t in_dim, int64_t s, int64_t P, int degree, const double* A, int64_t lda, int64_t m,
                         double* Z, double2* scratch, cudaStream_t stream);
// SRHT rows: A (m x in_dim) -> Z (m x s); P = next_pow2(in_dim); scratch: srht_scratch(P, m) doubles.
size_t srht_scratch(int64_t P, int64_t m);
void srht_launch(const double* sign, const int64_t* rows, int64_t in_dim, int64_t P, int64_t s, double scale,
                 const double* A, int64_t m, double* Z, double* scratch, cudaStream_t stream);
void div_launch(double* z, int64_t count, double denom, cudaStream_t stream);

// ---------------------------------------------------------------- vector algebra (K7)
// All reductions are deterministic: `nb` fixed block partials then a fixed-order sum.
int vec_blocks(int64_t n);
void dot_partial_launch(const double* a, const double* b, int64_t n, double* partial, int nb,
                        cudaStream_t stream);
void sum_partials_launch(const double* partial, int nb, double* out, cudaStream_t stream);
// alpha = rz / pap (pap summed from pap_part), x += alpha p, r -= alpha ap, rr partials.
// scal[0] <- pap, scal[1] <- alpha (written by block 0).
void pcg_update_xr_launch(const double* pap_part, int nb, const double* rz, double* x, double* r,
                          const double* p, const double* ap, int64_t n, double* rr_part,
                          double* scal, cudaStream_t stream);
// rz_new = sum(rz_part); beta = rz_new / rz_old; p = z + beta p; *rz_out = rz_new.
void pcg_update_p_launch(const double* rz_part, int nb, const double* rz_old, double* rz_out,
                         double* p, const double* z, int64_t n, cudaStream_t stream);
void copy_launch(double* dst, const double* src, int64_t n, cudaStream_t stream);
// Graph-resident PCG loop (krr_capi.cu pcg_graph): the device-side stop decision and the
// rz double-buffer copy.
void pcg_control_launch(const double* scal, int* ctl, double* hist, double* final_rel, double norm_y, double tau,
                        int max_iter, cudaGraphConditionalHandle cond, cudaStream_t stream);
void scalar_copy_launch(double* dst, const double* src, cudaStream_t stream);
void add_scaled_launch(double* out, const double* v, double lambda, int64_t n, cudaStream_t stream);
// Gather column c of an n x t row-major matrix into a contiguous vector (and back).
void gather_col_launch(const double* M, int64_t n, int64_t t, int64_t c, double* out,
                       cudaStream_t stream);
void scatter_col_launch(const double* v, int64_t n, int64_t t, int64_t c, double* M,
                        cudaStream_t stream);

// Batched variants for T independent right-hand sides, vectors n x T row-major,
// partials nb x T, T in {2, 4, 8, 16}; `active` (device, T ints) masks converged columns.
int vecT_blocks(int64_t n, int T);
void dotT_partial_launch(const double* a, const double* b, int64_t n, int T, double* partial, int nb,
                         cudaStream_t stream);
void sumT_partials_launch(const double* partial, int nb, int T, double* out, cudaStream_t stream);
void pcgT_update_xr_launch(const double* pap_part, int nb, int T, const double* rz, const int* active,
                           double* x, double* r, const double* p, const double* ap, int64_t n,
                           double* rr_part, double* pap_out, cudaStream_t stream);
void pcgT_update_p_launch(const double* rz_part, int nb, int T, const double* rz_old, double* rz_out,
                          const int* active, double* p, const double* z, int64_t n, cudaStream_t stream);
// columns [c0, c0 + T) of an n x t row-major block <-> n_pad x T interleaved (zero padded)
void pad_cols_launch(const double* in, int64_t n, int64_t t, int64_t c0, int64_t n_pad, int T, double* out,
                     cudaStream_t stream);
void unpad_cols_launch(const double* in, int64_t n, int64_t t, int64_t c0, int T, double* out,
                       cudaStream_t stream);

// ---------------------------------------------------------------- RFF (K2)
// Wp (s_pad x dp) = W (s x d) zero-padded.
void rff_pad_w_launch(const double* W, int64_t s, int64_t d, int64_t s_pad, int dp, double* Wp,
                      cudaStream_t stream);
// Z (rows x s, row-major) = sqrt(2/s) cos(L[rows] Wp^T + b), L the K1 operand (dp columns).
void rff_features_launch(const double* L, const double* Wp, const double* b, double* Z, int64_t rows,
                         int64_t s, int dp, cudaStream_t stream);
// Z[i][k] = sqrt(2/s) * cos(Z[i][k] + b[k]), in place, Z n x s row-major.

// ---------------------------------------------------------------- preconditioner (K3-K6)
// G (s x s, col-major) diag += add; trace -> *trace (nullable)
void diag_add_launch(double* G, int64_t s, double add, cudaStream_t stream);
void trace_launch(const double* G, int64_t s, double* out, cudaStream_t stream);
// min |L_kk| and a finiteness flag: out[0] = min |diag|, out[1] = 1 if any non-finite entry on diag
void diag_check_launch(const double* G, int64_t s, double* out, cudaStream_t stream);
// B = U^T stored n x s row-major.  Wpart[chunk][k] = sum_{i in chunk} B[i][k] r_i.
int gemvT_chunks(int64_t n, int64_t s);
void gemvT_partial_launch(const double* B, int64_t n, int64_t s, const double* r, double* Wpart,
                          int nchunks, cudaStream_t stream);
void reduce_rows_launch(const double* Wpart, int nchunks, int64_t s, double* W,
                        cudaStream_t stream);
// z_i = (r_i - B[i] . W) / lambda_p, rz partials (nb blocks).
int zrow_blocks(int64_t n);
// K6T (precond_multi.cu): Woodbury apply for T = 8 / 16 interleaved columns on the DMMA path.
// which: 1 = pass 1 (W = B^T R, reduced), 2 = pass 2 (Z = (R - B W) / lambda_p), 3 = both.
// K3-I8 (gram_i8.cu): G = Z^T Z (column-major lower triangle) on tcgen05 INT8 Ozaki slices.
int64_t gram_i8_spad(int64_t s);
size_t gram_i8_scratch_bytes(int64_t rows, int64_t s);
void gram_i8_launch(const double* Z, int64_t rows, int64_t s, double* G, uint8_t* scratch, int* ex,
                    unsigned long long* maxbits, int* bad, int2* tiles, cudaStream_t stream);
// K4 (cholesky.cu): in-place Cholesky of the column-major lower triangle; *info = 1 + first bad pivot.
void cholesky_launch(double* G, int64_t s, int* info, cudaStream_t stream);
// K5 (trsm.cu): U^T = Z L^-T in place (U = L^-1 Z^T), L column-major lower, on DMMA.
void trsm_lower_launch(double* Z, int64_t n, int64_t s, const double* L, cudaStream_t stream);
int k6t_splits(int64_t n, int64_t s);
bool k6t_supported(int64_t s, const void* B);  // even s (16-byte aligned rows of B)
void precond_multi_launch(const double* B, int64_t n, int64_t s, const double* R, double lambda_p, double* Z,
                          double* Wpart, int nsplit, double* W, int T, int which, cudaStream_t stream);
void precond_z_launch(const double* B, int64_t n, int64_t s, const double* W, const double* r,
                      double lambda_p, double* z, double* rz_part, int nb, cudaStream_t stream);

}  // namespace krr
