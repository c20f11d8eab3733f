// Auxiliary kernels: epilogue constants and the rectangular predict kernel (cross-Gram).
#include <cmath>
#include <cstring>

#include "common.cuh"
#include "kernels.cuh"

namespace krr {

ExpConsts make_exp_consts(double scale) {
    ExpConsts c{};
    const long double ln2 = 0.693147180559945309417232121458176568L;
    const long double l = ln2 / 64.0L;
    c.kscale = double(-(long double)scale * 64.0L / ln2);
    c.neg_scale = -scale;
    long double term = 1.0L;
    double a[6];
    for (int m = 1; m <= 5; ++m) {
        term = term * l / (long double)m;
        a[m] = double(term);
    }
    c.a1 = a[1];
    c.a2 = a[2];
    c.a3 = a[3];
    c.a4 = a[4];
    c.a5 = a[5];
    // exp(-d2 scale) >= 2^-1020 <=> d2 <= 1020 ln2 / scale
    const double d2max = double(1020.0L * ln2 / (long double)scale);
    int64_t bits;
    std::memcpy(&bits, &d2max, sizeof(bits));
    c.hi_under = int(bits >> 32);
    c.degree = 0;
    return c;
}

ExpConsts make_poly_consts(int degree) {
    ExpConsts c{};
    c.degree = degree;
    return c;
}

void make_exp_table(double* tab64) {
    for (int j = 0; j < 64; ++j) tab64[j] = double(exp2l((long double)j / 64.0L));
}

namespace {

__global__ void cross_matvec_kernel(const double* __restrict__ Xq, int64_t m,
                                    const double* __restrict__ X, int64_t n, int64_t d,
                                    const double* __restrict__ c, int64_t t, double scale,
                                    double* __restrict__ out) {
    __shared__ double scr[32];
    const int64_t q = blockIdx.x;
    if (q >= m) return;
    const double* a = Xq + q * d;
    double sqa = 0.0;
    for (int64_t k = 0; k < d; ++k) sqa = fma(a[k], a[k], sqa);
    for (int64_t col = 0; col < t; ++col) {
        double acc = 0.0;
        for (int64_t j = threadIdx.x; j < n; j += blockDim.x) {
            const double* xj = X + j * d;
            double dot = 0.0, sqj = 0.0;
            for (int64_t k = 0; k < d; ++k) {
                dot = fma(a[k], xj[k], dot);
                sqj = fma(xj[k], xj[k], sqj);
            }
            const double e = exp(-fmax(0.0, sqa + sqj - 2.0 * dot) * scale);
            acc = fma(e, c[j * t + col], acc);
        }
        acc = block_sum(acc, scr);
        if (threadIdx.x == 0) out[q * t + col] = acc;
    }
}

}  // namespace

void cross_matvec_launch(const double* Xq, int64_t m, const double* X, int64_t n, int64_t d,
                         const double* c, int64_t t, double scale, double* out,
                         cudaStream_t stream) {
    if (m == 0) return;
    cross_matvec_kernel<<<unsigned(m), 256, 0, stream>>>(Xq, m, X, n, d, c, t, scale, out);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
