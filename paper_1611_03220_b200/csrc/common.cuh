// Shared device/host helpers for the B200 KRR hot path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>

#include "../../include/krr_b200.h"
#include "error.hpp"

namespace krr {


inline void cuda_check(cudaError_t e, const char* what, const char* file, int line) {
    if (e != cudaSuccess)
        fail(KRR_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e) + " (" + file + ":" +
                               std::to_string(line) + ")");
}
// Process-wide count of kernels this library launched (bench.py's gpu_launches).
inline std::atomic<int64_t> g_launches{0};

#define KRR_CUDA(call) ::krr::cuda_check((call), #call, __FILE__, __LINE__)
#define KRR_LAUNCH_CHECK()                                                              \
    do {                                                                                \
        ::krr::g_launches.fetch_add(1, std::memory_order_relaxed);                      \
        ::krr::cuda_check(cudaGetLastError(), "kernel launch", __FILE__, __LINE__);     \
    } while (0)

constexpr int kVecThreads = 256;

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Deterministic block reduction (fixed tree): every thread passes its value,
// thread 0 receives the block sum.  `scratch` holds >= 32 doubles.
__device__ __forceinline__ double block_sum(double v, double* scratch) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();  // protect scratch reuse across consecutive calls
    if (lane == 0) scratch[wid] = v;
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    double s = 0.0;
    if (wid == 0) {
        s = lane < nw ? scratch[lane] : 0.0;
        s = warp_sum(s);
    }
    return s;
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// FP64 tensor-core MMA (DMMA.8x8x4 on sm_100a): D(8x8) += A(8x4, row) * B(4x8, col).
// Thread (g = lane/4, t = lane%4) holds A[g][t], B[t][g], D[g][2t], D[g][2t+1].
__device__ __forceinline__ void dmma884(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}

}  // namespace krr
