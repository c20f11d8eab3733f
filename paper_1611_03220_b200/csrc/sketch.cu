// the polynomial kernel's operands and the TensorSketch / SRHT / Gaussian
// sketch stages on the device.
//
//  * poly_operands: the augmented inputs [sqrt(gamma) x, sqrt(c)] (kernels.cpp:56-62) as
//    both K1 operands, so the fused K1 kernels' tensor-core contraction yields
//    p_ij = gamma x_i.x_j + c and the epilogue (gauss_exp.cuh mode 2) raises it to the
//    degree; the diagonal K_ii = ipow(|xa_i|^2, q) is kept per row for the finish kernel
//    (the Gaussian kernel's K_ii = 1 needs no table).
//  * tensorsketch: TensorSketchMap::apply (sketches.cpp:71-93) per row — count sketches
//    (sketches.cpp:43-49), forward radix-2 transforms, product of spectra, inverse, wrap
//    mod s.  One CTA per row (persistent grid); the length-P working vectors live in
//    shared memory when they fit, else in a per-CTA global scratch.  Every floating-point
//    operation is the reference algorithm's own, in its order, with explicit
//    round-to-nearest intrinsics (no FMA contraction), and the twiddles are the host's
//    libstdc++ recurrence w *= w_len (numerics.cpp:28-40), so the features are bitwise
//    those of the CPU restatement.
//  * srht: SrhtMap::apply (sketches.cpp:111-121): pad, sign flip, Walsh-Hadamard
//    butterflies (numerics.cpp:81-95), sample, scale — also bitwise.
//  * The Gaussian stage (sketches.cpp:137-140) is a cuBLAS DGEMM plus the division here.
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

__global__ void poly_operands_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, int dp,
                                     double sg, double so, int degree, double* __restrict__ L,
                                     double* __restrict__ R, double* __restrict__ kdiag) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad;
         i += int64_t(gridDim.x) * blockDim.x) {
        double* li = L + i * dp;
        double* ri = R ? R + i * dp : nullptr;
        double sq = 0.0;
        for (int k = 0; k < dp; ++k) {
            double v = 0.0;
            if (i < n) {
                if (k < d)
                    v = __dmul_rn(sg, X[i * d + k]);
                else if (k == d)
                    v = so;
            }
            li[k] = v;
            if (ri) ri[k] = v;
            sq = __fma_rn(v, v, sq);
        }
        if (kdiag) {
            double r = sq;
            for (int q = 1; q < degree; ++q) r = __dmul_rn(r, sq);
            kdiag[i] = i < n ? r : 0.0;
        }
    }
}

__global__ void cross_poly_kernel(const double* __restrict__ Xq, int64_t m, const double* __restrict__ X, int64_t n,
                                  int64_t d, const double* __restrict__ c, int64_t t, double sg, double so,
                                  int degree, double* __restrict__ out) {
    __shared__ double scr[32];
    const int64_t q = blockIdx.x;
    if (q >= m) return;
    const double* a = Xq + q * d;
    for (int64_t col = 0; col < t; ++col) {
        double acc = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            const double* xj = X + j * d;
            double p = 0.0;
            for (int64_t k = 0; k < d; ++k) p = __fma_rn(__dmul_rn(sg, a[k]), __dmul_rn(sg, xj[k]), p);
            p = __fma_rn(so, so, p);
            double r = p;
            for (int e = 1; e < degree; ++e) r = __dmul_rn(r, p);
            acc = __fma_rn(r, c[j * t + col], acc);
        }
        acc = block_sum(acc, scr);
        if (threadIdx.x == 0) out[q * t + col] = acc;
    }
}

// complex a * b as GCC / Eigen form it: (a.re b.re - a.im b.im, a.re b.im + a.im b.re), no FMA.
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(__dsub_rn(__dmul_rn(a.x, b.x), __dmul_rn(a.y, b.y)),
                        __dadd_rn(__dmul_rn(a.x, b.y), __dmul_rn(a.y, b.x)));
}

// In-place radix-2 transform of buf[0, P) by the CTA: bit-reversal permutation, then
// log2 P butterfly stages; tw holds each stage's twiddles (stage of length `len` at
// offset len/2 - 1).  Ends with a barrier.
__device__ void fft_cta(double2* buf, int64_t P, int logP, const double2* __restrict__ tw, bool inverse) {
    for (int64_t i = threadIdx.x; i < P; i += blockDim.x) {
        const int64_t r = logP ? int64_t(__brevll(uint64_t(i)) >> (64 - logP)) : i;
        if (i < r) {
            const double2 t = buf[i];
            buf[i] = buf[r];
            buf[r] = t;
        }
    }
    __syncthreads();
    for (int64_t half = 1; half < P; half <<= 1) {
        const double2* w = tw + (half - 1);
        for (int64_t k = threadIdx.x; k < P / 2; k += blockDim.x) {
            const int64_t j = k & (half - 1);
            const int64_t i0 = (k - j) * 2 + j;
            const double2 u = buf[i0];
            const double2 v = cmul(buf[i0 + half], w[j]);
            buf[i0] = make_double2(__dadd_rn(u.x, v.x), __dadd_rn(u.y, v.y));
            buf[i0 + half] = make_double2(__dsub_rn(u.x, v.x), __dsub_rn(u.y, v.y));
        }
        __syncthreads();
    }
    if (inverse) {
        const double pd = double(P);
        for (int64_t i = threadIdx.x; i < P; i += blockDim.x)
            buf[i] = make_double2(__ddiv_rn(buf[i].x, pd), __ddiv_rn(buf[i].y, pd));
        __syncthreads();
    }
}

struct TsArgs {
    const uint32_t* __restrict__ hash;  // degree x in_dim
    const double* __restrict__ sign;    // degree x in_dim
    const double2* __restrict__ tw_fwd; // P - 1
    const double2* __restrict__ tw_inv; // P - 1
    const double* __restrict__ A;       // m rows, stride lda, in_dim used
    double* __restrict__ Z;             // m x s
    double2* __restrict__ scratch;      // gridDim.x x 2P (when not in shared memory)
    int64_t in_dim, lda, m, s, P;
    int degree, logP;
    int buf_smem, acc_smem;
};

__global__ void __launch_bounds__(256) tensorsketch_kernel(const TsArgs a) {
    extern __shared__ __align__(16) double2 tsm[];
    double2* gs = a.scratch + int64_t(blockIdx.x) * 2 * a.P;
    double2* buf = a.buf_smem ? tsm : gs;
    double2* acc = a.acc_smem ? tsm + a.P : gs + a.P;
    for (int64_t row = blockIdx.x; row < a.m; row += gridDim.x) {
        const double* x = a.A + row * a.lda;
        double* z = a.Z + row * a.s;
        for (int q = 0; q < a.degree; ++q) {
            for (int64_t i = threadIdx.x; i < a.P; i += blockDim.x) buf[i] = make_double2(0.0, 0.0);
            __syncthreads();
            if (threadIdx.x == 0) {  // countsketch_apply: z[h_j] += g_j x_j, j ascending
                const uint32_t* h = a.hash + int64_t(q) * a.in_dim;
                const double* g = a.sign + int64_t(q) * a.in_dim;
                for (int64_t j = 0; j < a.in_dim; ++j) buf[h[j]].x = __dadd_rn(buf[h[j]].x, __dmul_rn(g[j], x[j]));
            }
            __syncthreads();
            if (a.degree == 1) break;
            fft_cta(buf, a.P, a.logP, a.tw_fwd, false);
            for (int64_t i = threadIdx.x; i < a.P; i += blockDim.x) acc[i] = q == 0 ? buf[i] : cmul(acc[i], buf[i]);
            __syncthreads();
        }
        if (a.degree == 1) {
            for (int64_t b = threadIdx.x; b < a.s; b += blockDim.x) z[b] = buf[b].x;
        } else {
            fft_cta(acc, a.P, a.logP, a.tw_inv, true);
            for (int64_t b = threadIdx.x; b < a.s; b += blockDim.x) {  // out[t mod s] += conv[t], t ascending
                double v = 0.0;
                for (int64_t t = b; t < a.P; t += a.s) v = __dadd_rn(v, acc[t].x);
                z[b] = v;
            }
        }
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) srht_kernel(const double* __restrict__ sign, const int64_t* __restrict__ rows,
                                                   int64_t in_dim, int64_t P, int64_t s, double scale,
                                                   const double* __restrict__ A, int64_t m, double* __restrict__ Z,
                                                   double* __restrict__ scratch, int use_smem) {
    extern __shared__ __align__(16) double hsm[];
    double* h = use_smem ? hsm : scratch + int64_t(blockIdx.x) * P;
    for (int64_t row = blockIdx.x; row < m; row += gridDim.x) {
        const double* x = A + row * in_dim;
        for (int64_t j = threadIdx.x; j < P; j += blockDim.x) h[j] = __dmul_rn(j < in_dim ? x[j] : 0.0, sign[j]);
        __syncthreads();
        for (int64_t half = 1; half < P; half <<= 1) {
            for (int64_t k = threadIdx.x; k < P / 2; k += blockDim.x) {
                const int64_t j = k & (half - 1);
                const int64_t i0 = (k - j) * 2 + j;
                const double u = h[i0], v = h[i0 + half];
                h[i0] = __dadd_rn(u, v);
                h[i0 + half] = __dsub_rn(u, v);
            }
            __syncthreads();
        }
        for (int64_t k = threadIdx.x; k < s; k += blockDim.x) Z[row * s + k] = __dmul_rn(scale, h[rows[k]]);
        __syncthreads();
    }
}

__global__ void div_kernel(double* __restrict__ z, int64_t count, double denom) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < count; i += int64_t(gridDim.x) * blockDim.x)
        z[i] = __ddiv_rn(z[i], denom);
}

int ilog2(int64_t p) {
    int l = 0;
    while ((int64_t(1) << l) < p) ++l;
    return l;
}

constexpr size_t kSmemCap = 220 * 1024;

}  // namespace

void poly_operands_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, int dp, double sg, double so,
                          int degree, double* L, double* R, double* kdiag, cudaStream_t stream) {
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((n_pad + 255) / 256, 148 * 8)));
    poly_operands_kernel<<<blocks, 256, 0, stream>>>(X, n, d, n_pad, dp, sg, so, degree, L, R, kdiag);
    KRR_LAUNCH_CHECK();
}

void cross_poly_launch(const double* Xq, int64_t m, const double* X, int64_t n, int64_t d, const double* c,
                       int64_t t, double sg, double so, int degree, double* out, cudaStream_t stream) {
    if (m == 0) return;
    cross_poly_kernel<<<unsigned(m), 256, 0, stream>>>(Xq, m, X, n, d, c, t, sg, so, degree, out);
    KRR_LAUNCH_CHECK();
}

int tensorsketch_grid(int64_t m) { return int(std::max<int64_t>(1, std::min<int64_t>(m, 148 * 2))); }

size_t tensorsketch_scratch(int64_t P, int64_t m) {
    const bool buf_smem = size_t(P) * 16 <= kSmemCap;
    const bool acc_smem = size_t(P) * 32 <= kSmemCap;
    if (buf_smem && acc_smem) return 0;
    return size_t(tensorsketch_grid(m)) * 2 * size_t(P);  // double2 elements
}

void tensorsketch_launch(const uint32_t* hash, const double* sign, const double2* tw_fwd, const double2* tw_inv,
                         int64_t in_dim, int64_t s, int64_t P, int degree, const double* A, int64_t lda, int64_t m,
                         double* Z, double2* scratch, cudaStream_t stream) {
    if (m == 0) return;
    TsArgs a;
    a.hash = hash;
    a.sign = sign;
    a.tw_fwd = tw_fwd;
    a.tw_inv = tw_inv;
    a.A = A;
    a.Z = Z;
    a.scratch = scratch;
    a.in_dim = in_dim;
    a.lda = lda;
    a.m = m;
    a.s = s;
    a.P = P;
    a.degree = degree;
    a.logP = ilog2(P);
    a.buf_smem = size_t(P) * 16 <= kSmemCap;
    a.acc_smem = size_t(P) * 32 <= kSmemCap;
    if ((!a.buf_smem || !a.acc_smem) && !scratch) fail(KRR_ERR_INVALID_ARGUMENT, "tensorsketch: scratch missing");
    const size_t smem = size_t(P) * 16 * (a.acc_smem ? 2 : (a.buf_smem ? 1 : 0));
    KRR_CUDA(cudaFuncSetAttribute(tensorsketch_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    tensorsketch_kernel<<<unsigned(tensorsketch_grid(m)), 256, smem, stream>>>(a);
    KRR_LAUNCH_CHECK();
}

int srht_grid(int64_t m) { return int(std::max<int64_t>(1, std::min<int64_t>(m, 148 * 4))); }

size_t srht_scratch(int64_t P, int64_t m) {
    return size_t(P) * 8 <= kSmemCap ? 0 : size_t(srht_grid(m)) * size_t(P);
}

void srht_launch(const double* sign, const int64_t* rows, int64_t in_dim, int64_t P, int64_t s, double scale,
                 const double* A, int64_t m, double* Z, double* scratch, cudaStream_t stream) {
    if (m == 0) return;
    const int use_smem = size_t(P) * 8 <= kSmemCap ? 1 : 0;
    if (!use_smem && !scratch) fail(KRR_ERR_INVALID_ARGUMENT, "srht: scratch missing");
    const size_t smem = use_smem ? size_t(P) * 8 : 0;
    KRR_CUDA(cudaFuncSetAttribute(srht_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    srht_kernel<<<unsigned(srht_grid(m)), 256, smem, stream>>>(sign, rows, in_dim, P, s, scale, A, m, Z, scratch,
                                                                use_smem);
    KRR_LAUNCH_CHECK();
}

void div_launch(double* z, int64_t count, double denom, cudaStream_t stream) {
    if (count == 0) return;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((count + 255) / 256, 148 * 8)));
    div_kernel<<<blocks, 256, 0, stream>>>(z, count, denom);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
