// Diagnostics only (libkrr_diag.so, include/krr_diag.h): FP64 / IMMA / exp micro-benchmarks and
// the table-exp probe.  Not part of the drop-in library.
#include <algorithm>

#include "common.cuh"
#include "diag.cuh"

namespace krr {
namespace {
__global__ void debug_exp_kernel(const double* __restrict__ d2, int64_t n, ExpConsts ec,
                                 const double* __restrict__ tab_g, int mode,
                                 double* __restrict__ out) {
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = tab_g[threadIdx.x];
    __syncthreads();
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
         i += int64_t(gridDim.x) * blockDim.x)
        out[i] = mode == 0 ? gauss_exp<0>(d2[i], ec, tab) : gauss_exp<1>(d2[i], ec, tab);
}

// ---- micro-benchmarks
constexpr int MB_ITERS = 4096;

__global__ void mb_dmma_kernel(double* sink, double a, double b) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
    for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) dmma884(acc[i][0], acc[i][1], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    if (s == 12345.678) sink[0] = s;
}

__global__ void mb_dfma_kernel(double* sink, double a, double b) {
    double acc[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i] = double(i) * 1e-3;
    for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fma(acc[i], a, b);
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i];
    if (s == 12345.678) sink[0] = s;
}

// Interleaved: per iteration 8 DMMA (8 x 256 MAC per warp) and 8 x 8 DFMA per thread.
__global__ void mb_mixed_kernel(double* sink, double a, double b) {
    double acc[8][2], f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
        acc[i][0] = acc[i][1] = 0.0;
        f[i] = double(i) * 1e-3;
    }
    for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            dmma884(acc[i][0], acc[i][1], a, b);
#pragma unroll
            for (int j = 0; j < 8; ++j) f[j] = fma(f[j], a, b);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + f[i];
    if (s == 12345.678) sink[0] = s;
}

// Half the warps run the DMMA loop, the other half the DFMA loop: if the two pipes
// are independent the combined rate approaches the sum.
__global__ void mb_split_kernel(double* sink, double a, double b) {
    const int warp = threadIdx.x >> 5;
    double s = 0.0;
    if (warp & 1) {
        double acc[8][2];
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
        for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) dmma884(acc[i][0], acc[i][1], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
    } else {
        double f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = double(i) * 1e-3;
        for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) f[i] = fma(f[i], a, b);
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) s += f[i];
    }
    if (s == 12345.678) sink[0] = s;
}

// Legacy warp-level integer MMA (IMMA m16n8k32 s8 x s8 -> s32): 8 independent accumulators.
__global__ void mb_imma_kernel(int* sink, int a, int b) {
    int acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0;
    for (int it = 0; it < MB_ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
                "{%0,%1,%2,%3};\n"
                : "+r"(acc[i][0]), "+r"(acc[i][1]), "+r"(acc[i][2]), "+r"(acc[i][3])
                : "r"(a), "r"(a), "r"(a), "r"(a), "r"(b), "r"(b));
    }
    int s = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1] + acc[i][2] + acc[i][3];
    if (s == 12345) sink[0] = s;
}

template <int MODE>
__global__ void mb_exp_kernel(double* sink, ExpConsts ec, const double* __restrict__ tab_g) {
    __shared__ double tab[64];
    if (threadIdx.x < 64) tab[threadIdx.x] = tab_g[threadIdx.x];
    __syncthreads();
    double x[8], acc = 0.0;
#pragma unroll
    for (int i = 0; i < 8; ++i) x[i] = 1.0 + 0.37 * i + 1e-3 * threadIdx.x;
    for (int it = 0; it < MB_ITERS / 8; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const double e = gauss_exp<MODE>(x[i], ec, tab);
            acc = fma(e, 0.5, acc);
            x[i] += 1e-7;
        }
    }
    if (acc == 12345.678) sink[0] = acc;
}

}  // namespace
void debug_exp_launch(const double* d2, int64_t n, const ExpConsts& ec, const double* tab,
                      int mode, double* out, cudaStream_t stream) {
    const unsigned blocks = unsigned(std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 1184)));
    debug_exp_kernel<<<blocks, 256, 0, stream>>>(d2, n, ec, tab, mode, out);
    KRR_LAUNCH_CHECK();
}

void microbench_run(const ExpConsts& ec, const double* tab, double* results, cudaStream_t stream) {
    int dev = 0, sms = 0, clk_khz = 0;
    KRR_CUDA(cudaGetDevice(&dev));
    KRR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    KRR_CUDA(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev));
    double* sink = nullptr;
    KRR_CUDA(cudaMalloc(&sink, 64));
    cudaEvent_t e0, e1;
    KRR_CUDA(cudaEventCreate(&e0));
    KRR_CUDA(cudaEventCreate(&e1));
    const unsigned blocks = unsigned(sms * 4);
    const unsigned threads = 256;
    const double warps = double(blocks) * threads / 32.0;
    auto time_it = [&](auto&& launch) {
        launch();  // warm-up
        KRR_CUDA(cudaEventRecord(e0, stream));
        for (int r = 0; r < 5; ++r) launch();
        KRR_CUDA(cudaEventRecord(e1, stream));
        KRR_CUDA(cudaEventSynchronize(e1));
        float ms = 0.f;
        KRR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
        return double(ms) / 5.0 * 1e-3;
    };
    const double t_dmma = time_it([&] { mb_dmma_kernel<<<blocks, threads, 0, stream>>>(sink, 1.0, 1e-9); });
    const double t_dfma = time_it([&] { mb_dfma_kernel<<<blocks, threads, 0, stream>>>(sink, 0.999, 1e-9); });
    const double t_mixed = time_it([&] { mb_mixed_kernel<<<blocks, threads, 0, stream>>>(sink, 0.999, 1e-9); });
    const double t_split = time_it([&] { mb_split_kernel<<<blocks, threads, 0, stream>>>(sink, 0.999, 1e-9); });
    const double t_imma = time_it([&] { mb_imma_kernel<<<blocks, threads, 0, stream>>>(reinterpret_cast<int*>(sink), 0x01010101, 0x01010101); });
    const double t_exp0 = time_it([&] { mb_exp_kernel<0><<<blocks, threads, 0, stream>>>(sink, ec, tab); });
    const double t_exp1 = time_it([&] { mb_exp_kernel<1><<<blocks, threads, 0, stream>>>(sink, ec, tab); });
    KRR_LAUNCH_CHECK();
    const double dmma_flop = warps * MB_ITERS * 8 * 512.0;
    const double dfma_flop = double(blocks) * threads * MB_ITERS * 8 * 2.0;
    const double mixed_flop = dmma_flop + dfma_flop * 8.0;
    const double evals = double(blocks) * threads * (MB_ITERS / 8) * 8;
    results[0] = dmma_flop / t_dmma * 1e-12;
    results[1] = dfma_flop / t_dfma * 1e-12;
    results[2] = mixed_flop / t_mixed * 1e-12;
    results[3] = evals / t_exp0 * 1e-9;
    results[4] = evals / t_exp1 * 1e-9;
    results[5] = sms;
    results[6] = clk_khz / 1000.0;
    // split: half the warps DMMA (dmma_flop / 2), half DFMA (dfma_flop / 2)
    results[7] = (dmma_flop / 2 + dfma_flop / 2) / t_split * 1e-12;
    // legacy IMMA: 16 x 8 x 32 MACs per instruction per warp, 2 ops per MAC
    results[8] = warps * MB_ITERS * 8 * (16.0 * 8 * 32 * 2) / t_imma * 1e-12;
    KRR_CUDA(cudaEventDestroy(e0));
    KRR_CUDA(cudaEventDestroy(e1));
    KRR_CUDA(cudaFree(sink));
}

}  // namespace krr
