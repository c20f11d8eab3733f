// Diagnostic: one-CTA tcgen05 kind::i8 GEMM  C (128 x N, s32) = A (128 x K) . B (N x K)^T
// through the helpers in tc_i8.cuh — validates the descriptor / TMEM mechanics the
// INT8-slice mat-vec relies on (tests/test_gpu_tc.py).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {
namespace {

template <int N>
__global__ void __launch_bounds__(128) i8_probe_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                       int32_t* __restrict__ C, int K) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + 128 * K;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int idx = tid; idx < 128 * K; idx += 128) sA[tc::kmajor_offset(idx / K, idx % K, 128)] = uint8_t(A[idx]);
    for (int idx = tid; idx < N * K; idx += 128) sB[tc::kmajor_offset(idx / K, idx % K, N)] = uint8_t(B[idx]);
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_i8(128, N);
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint64_t da = tc::smem_desc(tc::smem_u32(sA) + ks * 2 * (128 * 16), 128 * 16, 128);
            const uint64_t db = tc::smem_desc(tc::smem_u32(sB) + ks * 2 * (N * 16), N * 16, 128);
            tc::mma_i8(tmem, da, db, idesc, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) C[(warp * 32 + lane) * N + c0 + j] = int32_t(r[j]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, N < 32 ? 32 : N);
}

// MMA throughput: one CTA per SM issues `reps` back-to-back tcgen05.mma (M = 128, N, K = 32)
// on zero operands (no swizzle, K-major) into TMEM; cycles per MMA -> out[blockIdx.x].
template <int N>
__global__ void __launch_bounds__(128) i8_mma_rate_kernel(int reps, int kbytes, long long* out, int naccum) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + N) * kbytes; i += 128) sm[i] = 0;
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_i8(128, N);
        const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 128 * kbytes);
        const long long t0 = clock64();
        if (naccum == -2) {
            // SS mode, descriptors hoisted, 8 MMAs per iteration (pure issue rate)
            const uint64_t da = tc::smem_desc(a, 128, uint32_t(kbytes) * 8);
            const uint64_t db = tc::smem_desc(b, 128, uint32_t(kbytes) * 8);
            tc::mma_i8(tmem, da, db, idesc, 0u);
            for (int r = 0; r < reps / 8; ++r) {
#pragma unroll
                for (int u = 0; u < 8; ++u) tc::mma_i8(tmem, da, db, idesc, 1u);
            }
        } else if (naccum < 0) {
            // TS mode: A (128 x 32 int8 = 8 TMEM columns) at TMEM column 256, D at column 0
            for (int r = 0; r < reps; ++r) {
                const int ks = r % (kbytes / 32);
                const uint64_t db = tc::smem_desc(b + ks * 256, 128, uint32_t(kbytes) * 8);
                tc::mma_i8_ts(tmem, tmem + 256u + uint32_t((r & 7) * 8), db, idesc, r > 0 ? 1u : 0u);
            }
        } else {
            for (int r = 0; r < reps; ++r) {
                const int ks = r % (kbytes / 32);
                const uint64_t da = tc::smem_desc(a + ks * 256, 128, uint32_t(kbytes) * 8);
                const uint64_t db = tc::smem_desc(b + ks * 256, 128, uint32_t(kbytes) * 8);
                const int slot = r % naccum;
                tc::mma_i8(tmem + uint32_t(slot * N), da, db, idesc, r >= naccum ? 1u : 0u);
            }
        }
        tc::mma_commit(&mbar);
        tc::mbar_wait(&mbar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

}  // namespace

double i8_mma_rate(int N, int reps, int kbytes, cudaStream_t stream) {
    int naccum = kbytes >= 1024 ? std::max(1, 512 / N) : 1;  // kbytes >= 1024: rotate accumulators
    if (kbytes >= 1024) kbytes /= 32;
    if (reps < 0) {  // TS mode (A in TMEM)
        reps = -reps;
        naccum = -1;
        if (reps >= 1000000) {  // hoisted-descriptor SS variant
            reps -= 1000000;
            naccum = -2;
        }
    }
    long long* d = nullptr;
    KRR_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
    const size_t smem = size_t(128 + N) * kbytes;
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<148, 128, smem, stream>>>(reps, kbytes, d, naccum);
    };
    if (N == 16) run(i8_mma_rate_kernel<16>);
    else if (N == 32) run(i8_mma_rate_kernel<32>);
    else if (N == 64) run(i8_mma_rate_kernel<64>);
    else if (N == 128) run(i8_mma_rate_kernel<128>);
    else run(i8_mma_rate_kernel<256>);
    KRR_LAUNCH_CHECK();
    long long h[148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    double mx = 0;
    for (long long v : h) mx = std::max(mx, double(v));
    return mx / reps;
}

void i8_probe_launch(const int8_t* A, const int8_t* B, int32_t* C, int K, int N, cudaStream_t stream) {
    const size_t smem = size_t(128 + N) * K;
    if (N == 32) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<32><<<1, 128, smem, stream>>>(A, B, C, K);
    } else if (N == 64) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<64><<<1, 128, smem, stream>>>(A, B, C, K);
    } else {
        fail(KRR_ERR_INVALID_ARGUMENT, "i8 probe: N must be 32 or 64");
    }
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
