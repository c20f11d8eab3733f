// K7 — PCG vector algebra (HBM-bound, deterministic reductions) and operand prep.
//
// Reference: pcg_solve (solver.cpp:41-63).  Per iteration:
//   pap = p.ap ; alpha = rz/pap ; x += alpha p ; r -= alpha ap ; |r|^2
//   rz' = r.z  ; p = z + (rz'/rz) p
// Scalars stay on the device (alpha/beta are recomputed inside the kernels from the
// fixed-order block partials), so the host only reads pap and |r|^2 once per
// iteration for the stopping / breakdown decision.
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

__global__ void build_operands_kernel(const double* __restrict__ X, int64_t n, int64_t d,
                                      int64_t n_pad, int dp, double* __restrict__ L,
                                      double* __restrict__ R) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_pad;
         i += warps) {
        double* li = L + i * dp;
        double* ri = R + i * dp;
        if (i >= n) {
            for (int k = lane; k < dp; k += 32) li[k] = ri[k] = 0.0;
            continue;
        }
        const double* xi = X + i * d;
        double sq = 0.0;
        for (int64_t k = lane; k < d; k += 32) {
            const double x = xi[k];
            sq = fma(x, x, sq);
            li[k] = x;
            ri[k] = -2.0 * x;
        }
        sq = warp_sum(sq);
        for (int k = int(d) + lane; k < dp; k += 32) {
            double lv = 0.0, rv = 0.0;
            if (k == d) {
                lv = sq;
                rv = 1.0;
            } else if (k == d + 1) {
                lv = 1.0;
                rv = sq;
            }
            li[k] = lv;
            ri[k] = rv;
        }
    }
}

__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                   int64_t n, double* __restrict__ partial) {
    __shared__ double scr[32];
    double s = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        s = fma(a[i], b[i], s);
    s = block_sum(s, scr);
    if (threadIdx.x == 0) partial[blockIdx.x] = s;
}

// Fixed-order sum of nb partials, executed identically by every calling block.
__device__ __forceinline__ double sum_fixed(const double* __restrict__ part, int nb, double* scr) {
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += part[i];
    s = block_sum(s, scr);
    __shared__ double bcast;
    if (threadIdx.x == 0) bcast = s;
    __syncthreads();
    return bcast;
}

__global__ void sum_partials_kernel(const double* __restrict__ partial, int nb,
                                    double* __restrict__ out) {
    __shared__ double scr[32];
    const double s = sum_fixed(partial, nb, scr);
    if (threadIdx.x == 0) *out = s;
}

__global__ void pcg_update_xr_kernel(const double* __restrict__ pap_part, int nb,
                                     const double* __restrict__ rz, double* __restrict__ x,
                                     double* __restrict__ r, const double* __restrict__ p,
                                     const double* __restrict__ ap, int64_t n,
                                     double* __restrict__ rr_part, double* __restrict__ scal) {
    __shared__ double scr[32];
    const double pap = sum_fixed(pap_part, nb, scr);
    const double alpha = *rz / pap;
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        scal[0] = pap;
        scal[1] = alpha;
    }
    double s = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x) {
        x[i] += alpha * p[i];
        const double ri = r[i] - alpha * ap[i];
        r[i] = ri;
        s = fma(ri, ri, s);
    }
    s = block_sum(s, scr);
    if (threadIdx.x == 0) rr_part[blockIdx.x] = s;
}

__global__ void pcg_update_p_kernel(const double* __restrict__ rz_part, int nb,
                                    const double* __restrict__ rz_old, double* __restrict__ rz_out,
                                    double* __restrict__ p, const double* __restrict__ z,
                                    int64_t n) {
    __shared__ double scr[32];
    const double rz_new = sum_fixed(rz_part, nb, scr);
    const double beta = rz_new / *rz_old;
    if (blockIdx.x == 0 && threadIdx.x == 0) *rz_out = rz_new;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        p[i] = z[i] + beta * p[i];
}

// Device-side PCG control for the graph-resident loop (one thread): the stop/breakdown
// decisions solver.cpp:37-52 makes on the host, from the scalars the iteration left in scal.
// ctl: [0] iterations so far, [1] status (0 running, 1 converged, 2 max_iter, 3 breakdown).
__global__ void pcg_control_kernel(const double* __restrict__ scal, int* __restrict__ ctl,
                                   double* __restrict__ hist, double* __restrict__ final_rel, double norm_y,
                                   double tau, int max_iter, cudaGraphConditionalHandle cond) {
    const int it = ctl[0] + 1;
    ctl[0] = it;
    const double pap = scal[0];
    if (!(pap > 0.0)) {
        ctl[1] = 3;
        cudaGraphSetConditional(cond, 0);
        return;
    }
    const double rel = sqrt(scal[4]) / norm_y;
    hist[it - 1] = rel;
    *final_rel = rel;
    if (rel <= tau) {
        ctl[1] = 1;
        cudaGraphSetConditional(cond, 0);
    } else if (it >= max_iter) {
        ctl[1] = 2;
        cudaGraphSetConditional(cond, 0);
    } else {
        cudaGraphSetConditional(cond, 1);
    }
}

__global__ void scalar_copy_kernel(double* __restrict__ dst, const double* __restrict__ src) { *dst = *src; }

// out_i = out_i + lambda v_i, rounded as the reference's `k * v + lambda * v` (no contraction)
__global__ void add_scaled_kernel(double* __restrict__ out, const double* __restrict__ v, double lambda, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = __dadd_rn(out[i], __dmul_rn(lambda, v[i]));
}

__global__ void copy_kernel(double* __restrict__ dst, const double* __restrict__ src, int64_t n) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        dst[i] = src[i];
}

__global__ void gather_col_kernel(const double* __restrict__ M, int64_t n, int64_t t, int64_t c,
                                  double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = M[i * t + c];
}

__global__ void scatter_col_kernel(const double* __restrict__ v, int64_t n, int64_t t, int64_t c,
                                   double* __restrict__ M) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        M[i * t + c] = v[i];
}

// ---- batched (n x T, row-major) variants for T independent right-hand sides.
// Thread layout: column c = threadIdx.x % T, row slot = threadIdx.x / T, so every
// thread owns one column's running sum; per-column block reduction through smem in
// a fixed order.  T divides blockDim (T in {2, 4, 8, 16}).
__device__ __forceinline__ void block_sum_cols(double v, int T, double* scr, double* out_row) {
    scr[threadIdx.x] = v;
    __syncthreads();
    for (int stride = blockDim.x / 2; stride >= T; stride >>= 1) {
        if (threadIdx.x < stride) scr[threadIdx.x] += scr[threadIdx.x + stride];
        __syncthreads();
    }
    if (threadIdx.x < T) out_row[threadIdx.x] = scr[threadIdx.x];
}

__global__ void dotT_partial_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                    int64_t n, int T, double* __restrict__ partial) {
    __shared__ double scr[256];
    const int c = threadIdx.x % T;
    const int rs = threadIdx.x / T, rper = blockDim.x / T;
    double s = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * rper + rs; i < n; i += int64_t(gridDim.x) * rper)
        s = fma(a[i * T + c], b[i * T + c], s);
    block_sum_cols(s, T, scr, partial + int64_t(blockIdx.x) * T);
}

__global__ void sumT_partials_kernel(const double* __restrict__ partial, int nb, int T,
                                     double* __restrict__ out) {
    const int c = threadIdx.x;
    if (c >= T) return;
    double s = 0.0;
    for (int b = 0; b < nb; ++b) s += partial[int64_t(b) * T + c];
    out[c] = s;
}

// alpha_c = active_c ? rz_c / pap_c : 0 (pap_c summed from the partials);
// x += alpha p, r -= alpha ap, |r|^2 partials.  scal_out[c] <- pap_c (block 0).
__global__ void pcgT_update_xr_kernel(const double* __restrict__ pap_part, int nb, int T,
                                      const double* __restrict__ rz, const int* __restrict__ active,
                                      double* __restrict__ x, double* __restrict__ r,
                                      const double* __restrict__ p, const double* __restrict__ ap,
                                      int64_t n, double* __restrict__ rr_part,
                                      double* __restrict__ pap_out) {
    __shared__ double scr[256];
    __shared__ double alpha[16];
    if (threadIdx.x < T) {
        double pap = 0.0;
        for (int b = 0; b < nb; ++b) pap += pap_part[int64_t(b) * T + threadIdx.x];
        alpha[threadIdx.x] = active[threadIdx.x] ? rz[threadIdx.x] / pap : 0.0;
        if (blockIdx.x == 0) pap_out[threadIdx.x] = pap;
    }
    __syncthreads();
    const int c = threadIdx.x % T;
    const int rs = threadIdx.x / T, rper = blockDim.x / T;
    const double al = alpha[c];
    double s = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * rper + rs; i < n; i += int64_t(gridDim.x) * rper) {
        const int64_t k = i * T + c;
        x[k] += al * p[k];
        const double ri = r[k] - al * ap[k];
        r[k] = ri;
        s = fma(ri, ri, s);
    }
    block_sum_cols(s, T, scr, rr_part + int64_t(blockIdx.x) * T);
}

// beta_c = rz_new_c / rz_old_c; p = z + beta p (active columns); rz_out <- rz_new.
__global__ void pcgT_update_p_kernel(const double* __restrict__ rz_part, int nb, int T,
                                     const double* __restrict__ rz_old, double* __restrict__ rz_out,
                                     const int* __restrict__ active, double* __restrict__ p,
                                     const double* __restrict__ z, int64_t n) {
    __shared__ double beta[16];
    if (threadIdx.x < T) {
        double rzn = 0.0;
        for (int b = 0; b < nb; ++b) rzn += rz_part[int64_t(b) * T + threadIdx.x];
        beta[threadIdx.x] = rzn / rz_old[threadIdx.x];
        if (blockIdx.x == 0) rz_out[threadIdx.x] = active[threadIdx.x] ? rzn : rz_old[threadIdx.x];
    }
    __syncthreads();
    const int c = threadIdx.x % T;
    const int rs = threadIdx.x / T, rper = blockDim.x / T;
    if (!active[c]) return;
    const double be = beta[c];
    for (int64_t i = int64_t(blockIdx.x) * rper + rs; i < n; i += int64_t(gridDim.x) * rper) {
        const int64_t k = i * T + c;
        p[k] = z[k] + be * p[k];
    }
}

// Interleave an n x t row-major block into n_pad x T (zero padded) and back.
__global__ void pad_cols_kernel(const double* __restrict__ in, int64_t n, int64_t t, int64_t c0,
                                int64_t n_pad, int T, double* __restrict__ out) {
    const int64_t total = n_pad * T;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k / T, c = k % T;
        out[k] = (i < n && c0 + c < t) ? in[i * t + c0 + c] : 0.0;
    }
}

__global__ void unpad_cols_kernel(const double* __restrict__ in, int64_t n, int64_t t, int64_t c0, int T,
                                  double* __restrict__ out) {
    const int64_t tc = min(int64_t(T), t - c0);
    const int64_t total = n * tc;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k / tc, c = k % tc;
        out[i * t + c0 + c] = in[i * T + c];
    }
}

// z = (r - y) / lambda_p elementwise (batched Woodbury epilogue after the cuBLAS GEMMs)

unsigned grid_for(int64_t n) {
    return unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 8)));
}

}  // namespace

int vecT_blocks(int64_t n, int T) {
    const int64_t rows_per_block = 256 / T;
    return int(std::max<int64_t>(1, std::min<int64_t>((n + rows_per_block - 1) / rows_per_block, 148 * 4)));
}

void dotT_partial_launch(const double* a, const double* b, int64_t n, int T, double* partial, int nb,
                         cudaStream_t stream) {
    dotT_partial_kernel<<<nb, 256, 0, stream>>>(a, b, n, T, partial);
    KRR_LAUNCH_CHECK();
}

void sumT_partials_launch(const double* partial, int nb, int T, double* out, cudaStream_t stream) {
    sumT_partials_kernel<<<1, 32, 0, stream>>>(partial, nb, T, out);
    KRR_LAUNCH_CHECK();
}

void pcgT_update_xr_launch(const double* pap_part, int nb, int T, const double* rz, const int* active,
                           double* x, double* r, const double* p, const double* ap, int64_t n,
                           double* rr_part, double* pap_out, cudaStream_t stream) {
    pcgT_update_xr_kernel<<<nb, 256, 0, stream>>>(pap_part, nb, T, rz, active, x, r, p, ap, n, rr_part,
                                                  pap_out);
    KRR_LAUNCH_CHECK();
}

void pcgT_update_p_launch(const double* rz_part, int nb, int T, const double* rz_old, double* rz_out,
                          const int* active, double* p, const double* z, int64_t n, cudaStream_t stream) {
    pcgT_update_p_kernel<<<nb, 256, 0, stream>>>(rz_part, nb, T, rz_old, rz_out, active, p, z, n);
    KRR_LAUNCH_CHECK();
}

void pad_cols_launch(const double* in, int64_t n, int64_t t, int64_t c0, int64_t n_pad, int T, double* out,
                     cudaStream_t stream) {
    pad_cols_kernel<<<grid_for(n_pad * T), 256, 0, stream>>>(in, n, t, c0, n_pad, T, out);
    KRR_LAUNCH_CHECK();
}

void unpad_cols_launch(const double* in, int64_t n, int64_t t, int64_t c0, int T, double* out,
                       cudaStream_t stream) {
    unpad_cols_kernel<<<grid_for(n * T), 256, 0, stream>>>(in, n, t, c0, T, out);
    KRR_LAUNCH_CHECK();
}


void build_operands_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, int dp,
                           double* L, double* R, cudaStream_t stream) {
    const unsigned blocks = unsigned(std::min<int64_t>((n_pad + 7) / 8, 148 * 16));
    build_operands_kernel<<<blocks, 256, 0, stream>>>(X, n, d, n_pad, dp, L, R);
    KRR_LAUNCH_CHECK();
}

int vec_blocks(int64_t n) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 4)));
}

void dot_partial_launch(const double* a, const double* b, int64_t n, double* partial, int nb,
                        cudaStream_t stream) {
    dot_partial_kernel<<<nb, kVecThreads, 0, stream>>>(a, b, n, partial);
    KRR_LAUNCH_CHECK();
}

void sum_partials_launch(const double* partial, int nb, double* out, cudaStream_t stream) {
    sum_partials_kernel<<<1, kVecThreads, 0, stream>>>(partial, nb, out);
    KRR_LAUNCH_CHECK();
}

void pcg_update_xr_launch(const double* pap_part, int nb, const double* rz, double* x, double* r,
                          const double* p, const double* ap, int64_t n, double* rr_part,
                          double* scal, cudaStream_t stream) {
    pcg_update_xr_kernel<<<nb, kVecThreads, 0, stream>>>(pap_part, nb, rz, x, r, p, ap, n, rr_part,
                                                         scal);
    KRR_LAUNCH_CHECK();
}

void pcg_update_p_launch(const double* rz_part, int nb, const double* rz_old, double* rz_out,
                         double* p, const double* z, int64_t n, cudaStream_t stream) {
    pcg_update_p_kernel<<<nb, kVecThreads, 0, stream>>>(rz_part, nb, rz_old, rz_out, p, z, n);
    KRR_LAUNCH_CHECK();
}

void pcg_control_launch(const double* scal, int* ctl, double* hist, double* final_rel, double norm_y, double tau,
                        int max_iter, cudaGraphConditionalHandle cond, cudaStream_t stream) {
    pcg_control_kernel<<<1, 1, 0, stream>>>(scal, ctl, hist, final_rel, norm_y, tau, max_iter, cond);
    KRR_LAUNCH_CHECK();
}

void add_scaled_launch(double* out, const double* v, double lambda, int64_t n, cudaStream_t stream) {
    add_scaled_kernel<<<grid_for(n), 256, 0, stream>>>(out, v, lambda, n);
    KRR_LAUNCH_CHECK();
}

void scalar_copy_launch(double* dst, const double* src, cudaStream_t stream) {
    scalar_copy_kernel<<<1, 1, 0, stream>>>(dst, src);
    KRR_LAUNCH_CHECK();
}

void copy_launch(double* dst, const double* src, int64_t n, cudaStream_t stream) {
    copy_kernel<<<grid_for(n), 256, 0, stream>>>(dst, src, n);
    KRR_LAUNCH_CHECK();
}

void gather_col_launch(const double* M, int64_t n, int64_t t, int64_t c, double* out,
                       cudaStream_t stream) {
    gather_col_kernel<<<grid_for(n), 256, 0, stream>>>(M, n, t, c, out);
    KRR_LAUNCH_CHECK();
}

void scatter_col_launch(const double* v, int64_t n, int64_t t, int64_t c, double* M,
                        cudaStream_t stream) {
    scatter_col_kernel<<<grid_for(n), 256, 0, stream>>>(v, n, t, c, M);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
