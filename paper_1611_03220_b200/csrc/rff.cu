// K2 — fused random-Fourier-feature map  Z = sqrt(2/s) cos(X W^T + b)
// (reference RffMap::apply, sketches.cpp:37-41, stacked by apply_rows :207-211).
//
// One DMMA.8x8x4 contraction per 128 x 128 tile of Z (rows x features) with the
// cos epilogue in registers; Z is written once, row-major, straight from the
// accumulators.  The A operand is the K1 operand L = [x, |x|^2, 1, 0..] (n_pad x dp)
// and W is zero-padded to dp columns, so the two augmented columns contribute exact
// zeros.  Every Z entry is summed in the same k order whatever n is, so
// apply(x_i) == apply_rows(X)[i] bitwise, as the reference test
// test_sketches.cpp:195-207 requires.
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int BM = 128;
constexpr int KC = 16;
constexpr int KS = 20;
constexpr int NTHREADS = 256;
constexpr int STAGE = 2 * BM * KS;

__global__ void __launch_bounds__(NTHREADS) rff_features_kernel(
    const double* __restrict__ L, const double* __restrict__ Wp, const double* __restrict__ b,
    double* __restrict__ Z, int64_t rows, int64_t s, int dp, double scale) {
    extern __shared__ __align__(16) double smem[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1, g = lane >> 2, t4 = lane & 3;
    const int64_t row0 = int64_t(blockIdx.x) * BM;
    const int64_t col0 = int64_t(blockIdx.y) * BM;
    const int nk = (dp + KC - 1) / KC;

    auto issue = [&](int kc, int slot) {
        double* sA = smem + slot * STAGE;
        double* sB = sA + BM * KS;
        const int k0 = kc * KC;
        const int pieces = min(KC, dp - k0) >> 1;
#pragma unroll
        for (int q = 0; q < (2 * BM * (KC / 2)) / NTHREADS; ++q) {
            const int idx = tid + q * NTHREADS;
            const int op = idx / (BM * (KC / 2));
            const int rem = idx % (BM * (KC / 2));
            const int r = rem / (KC / 2), pc = rem % (KC / 2);
            if (pc < pieces) {
                // Rows past the shard are clamped (their results are never stored);
                // Wp is zero-padded to a multiple of 128 feature rows.
                const int64_t ra = min(row0 + r, rows - 1);
                const double* gp = (op ? Wp + (col0 + r) * dp : L + ra * dp) + k0 + pc * 2;
                cp_async16((op ? sB : sA) + r * KS + pc * 2, gp);
            }
        }
    };

    double acc[8][4][2];
#pragma unroll
    for (int ms = 0; ms < 8; ++ms)
#pragma unroll
        for (int ns = 0; ns < 4; ++ns) acc[ms][ns][0] = acc[ms][ns][1] = 0.0;

    issue(0, 0);
    cp_async_commit();
    for (int kc = 0; kc < nk; ++kc) {
        if (kc + 1 < nk) issue(kc + 1, (kc + 1) & 1);
        cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        const double* sA = smem + (kc & 1) * STAGE;
        const double* sB = sA + BM * KS;
        const int nks = min(KC, dp - kc * KC) >> 2;
        const double* aBase = sA + (wm * 64 + g) * KS + t4;
        const double* bBase = sB + (wn * 32 + g) * KS + t4;
#pragma unroll
        for (int ks = 0; ks < KC / 4; ++ks) {
            if (ks < nks) {
                double af[8], bf[4];
#pragma unroll
                for (int ms = 0; ms < 8; ++ms) af[ms] = aBase[ms * 8 * KS + ks * 4];
#pragma unroll
                for (int ns = 0; ns < 4; ++ns) bf[ns] = bBase[ns * 8 * KS + ks * 4];
#pragma unroll
                for (int ms = 0; ms < 8; ++ms)
#pragma unroll
                    for (int ns = 0; ns < 4; ++ns) dmma884(acc[ms][ns][0], acc[ms][ns][1], af[ms], bf[ns]);
            }
        }
        __syncthreads();
    }

#pragma unroll
    for (int ns = 0; ns < 4; ++ns) {
        const int64_t k = col0 + wn * 32 + ns * 8 + 2 * t4;
        const double b0 = k < s ? b[k] : 0.0;
        const double b1 = k + 1 < s ? b[k + 1] : 0.0;
#pragma unroll
        for (int ms = 0; ms < 8; ++ms) {
            const int64_t i = row0 + wm * 64 + ms * 8 + g;
            if (i >= rows) continue;
            double* zr = Z + i * s;
            if (k < s) zr[k] = scale * cos(acc[ms][ns][0] + b0);
            if (k + 1 < s) zr[k + 1] = scale * cos(acc[ms][ns][1] + b1);
        }
    }
}

__global__ void pad_w_kernel(const double* __restrict__ W, int64_t s, int64_t d, int64_t s_pad, int dp,
                             double* __restrict__ Wp) {
    const int64_t total = s_pad * dp;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t r = idx / dp, c = idx % dp;
        Wp[idx] = (r < s && c < d) ? W[r * d + c] : 0.0;
    }
}

}  // namespace

void rff_pad_w_launch(const double* W, int64_t s, int64_t d, int64_t s_pad, int dp, double* Wp,
                      cudaStream_t stream) {
    const int64_t total = s_pad * dp;
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((total + 255) / 256, 148 * 16)));
    pad_w_kernel<<<blocks, 256, 0, stream>>>(W, s, d, s_pad, dp, Wp);
    KRR_LAUNCH_CHECK();
}

void rff_features_launch(const double* L, const double* Wp, const double* b, double* Z, int64_t rows,
                         int64_t s, int dp, cudaStream_t stream) {
    if (rows <= 0) return;
    const double scale = sqrt(2.0 / double(s));
    const size_t smem = sizeof(double) * 2 * STAGE;
    KRR_CUDA(cudaFuncSetAttribute(rff_features_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    dim3 grid(unsigned((rows + BM - 1) / BM), unsigned((s + BM - 1) / BM));
    rff_features_kernel<<<grid, NTHREADS, smem, stream>>>(L, Wp, b, Z, rows, s, dp, scale);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
