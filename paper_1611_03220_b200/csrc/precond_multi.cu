// K6T — the Woodbury apply for T interleaved right-hand sides (T = 8 or 16), the per-iteration
// preconditioner of the batched PCG (BASELINE config 5: t = 16, s = 16384).
//
// Reference: Preconditioner::apply_columns (precond.cpp:15-18): Z = (R - U^T (U R)) / lambda_p.
// On the device U is stored as B = U^T (n x s row-major, precond.cu), R and Z are n x T
// row-major (interleaved columns), so both passes stream B once:
//   pass 1 (K6T-a):  W (s x T) = B^T R    — feature blocks x row splits, deterministic partials
//   pass 2 (K6T-b):  Z = (R - B W) / lambda_p
// At T = 16 each 8-byte element of B feeds 16 FMAs: at the HBM rate (22 B/clk/SM) that is ~70 %
// of the FP64 pipe, so both passes run the contraction on the FP64 tensor path (DMMA
// m8n8k4, one instruction per 256 FMAs) with B tiles staged through a 3-stage cp.async ring;
// the bound is HBM: 2 x 8 n s bytes per apply (config 5: 2 x 68.7 GB).
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int K6T_STAGES = 3;
constexpr int K6T_THREADS = 256;  // 8 warps

__device__ __forceinline__ void cp_async8_zfill(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    const int bytes = valid ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(bytes));
}

// ---- pass 1: Wpart[split][f][T] = sum_{k in split} B[k][f] R[k][.] for a 64-feature block.
// Warp w owns features f0 + 8w .. + 8 (DMMA M), all T columns (T / 8 N tiles); K = rows, 32 per stage.
constexpr int A_FB = 64;          // features per CTA
constexpr int A_KR = 32;          // rows per stage
constexpr int A_LDB = A_FB + 8;   // smem row stride (doubles): the A-fragment reads hit distinct banks
template <int T>
struct PassA {
    static constexpr int LDR = T;
    static constexpr int STAGE = A_KR * A_LDB + A_KR * LDR;  // doubles
    static constexpr size_t SMEM = size_t(K6T_STAGES) * STAGE * sizeof(double);
};

template <int T>
__global__ void __launch_bounds__(K6T_THREADS) k6t_pass_a_kernel(const double* __restrict__ B, int64_t n,
                                                                  int64_t s, const double* __restrict__ R,
                                                                  double* __restrict__ Wpart, int64_t rows_per) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t f0 = int64_t(blockIdx.x) * A_FB;
    const int64_t k0 = int64_t(blockIdx.y) * rows_per;
    const int64_t k1 = min(n, k0 + rows_per);
    const int64_t nchunk = k1 > k0 ? (k1 - k0 + A_KR - 1) / A_KR : 0;
    constexpr int NT = T / 8;
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;

    auto load = [&](int64_t c, int st) {
        double* sb = sm + st * PassA<T>::STAGE;
        double* sr = sb + A_KR * A_LDB;
        const int64_t kb = k0 + c * A_KR;
        for (int e = tid; e < A_KR * A_FB; e += K6T_THREADS) {
            const int r = e / A_FB, f = e % A_FB;
            const bool ok = kb + r < k1 && f0 + f < s;
            cp_async8_zfill(sb + r * A_LDB + f, ok ? B + (kb + r) * s + f0 + f : B, ok);
        }
        for (int e = tid; e < A_KR * T; e += K6T_THREADS) {
            const int r = e / T, cc = e % T;
            const bool ok = kb + r < k1;
            cp_async8_zfill(sr + r * PassA<T>::LDR + cc, ok ? R + (kb + r) * T + cc : R, ok);
        }
    };
#pragma unroll
    for (int st = 0; st < K6T_STAGES - 1; ++st) {
        if (st < nchunk) load(st, st);
        cp_async_commit();
    }
    for (int64_t c = 0; c < nchunk; ++c) {
        if (c + K6T_STAGES - 1 < nchunk) load(c + K6T_STAGES - 1, int((c + K6T_STAGES - 1) % K6T_STAGES));
        cp_async_commit();
        cp_async_wait<K6T_STAGES - 1>();
        __syncthreads();
        const double* sb = sm + int(c % K6T_STAGES) * PassA<T>::STAGE;
        const double* sr = sb + A_KR * A_LDB;
#pragma unroll
        for (int kk = 0; kk < A_KR; kk += 4) {
            const double a = sb[(kk + t4) * A_LDB + warp * 8 + g];  // A[g][t4] = B[k][f]
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[j][0], acc[j][1], a, sr[(kk + t4) * PassA<T>::LDR + j * 8 + g]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    const int64_t f = f0 + warp * 8 + g;
    if (f < s) {
        double* w = Wpart + (int64_t(blockIdx.y) * s + f) * T;
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            w[j * 8 + 2 * t4] = acc[j][0];
            w[j * 8 + 2 * t4 + 1] = acc[j][1];
        }
    }
}

// ---- pass 2: Z[k][.] = (R[k][.] - B[k][:] W) / lambda_p for a 64-row block.
// Warp w owns rows r0 + 8w .. + 8 (DMMA M), all T columns; K = features, 32 per stage.
constexpr int B_RB = 64;          // rows per CTA
constexpr int B_KF = 32;          // features per stage
constexpr int B_LDB = B_KF + 4;   // smem row stride (doubles): A-fragment reads conflict-free
template <int T>
struct PassB {
    static constexpr int STAGE = B_RB * B_LDB + B_KF * T;
    static constexpr size_t SMEM = size_t(K6T_STAGES) * STAGE * sizeof(double);
};

template <int T>
__global__ void __launch_bounds__(K6T_THREADS) k6t_pass_b_kernel(const double* __restrict__ B, int64_t n,
                                                                  int64_t s, const double* __restrict__ W,
                                                                  const double* __restrict__ R, double lambda_p,
                                                                  double* __restrict__ Z) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t r0 = int64_t(blockIdx.x) * B_RB;
    const int64_t nchunk = (s + B_KF - 1) / B_KF;
    constexpr int NT = T / 8;
    double acc[NT][2];
#pragma unroll
    for (int j = 0; j < NT; ++j) acc[j][0] = acc[j][1] = 0.0;

    auto load = [&](int64_t c, int st) {
        double* sb = sm + st * PassB<T>::STAGE;
        double* sw = sb + B_RB * B_LDB;
        const int64_t fb = c * B_KF;
        for (int e = tid; e < B_RB * B_KF; e += K6T_THREADS) {
            const int r = e / B_KF, f = e % B_KF;
            const bool ok = r0 + r < n && fb + f < s;
            cp_async8_zfill(sb + r * B_LDB + f, ok ? B + (r0 + r) * s + fb + f : B, ok);
        }
        for (int e = tid; e < B_KF * T; e += K6T_THREADS) {
            const int f = e / T;
            const bool ok = fb + f < s;
            cp_async8_zfill(sw + e, ok ? W + fb * T + e : W, ok);
        }
    };
#pragma unroll
    for (int st = 0; st < K6T_STAGES - 1; ++st) {
        if (st < nchunk) load(st, st);
        cp_async_commit();
    }
    for (int64_t c = 0; c < nchunk; ++c) {
        if (c + K6T_STAGES - 1 < nchunk) load(c + K6T_STAGES - 1, int((c + K6T_STAGES - 1) % K6T_STAGES));
        cp_async_commit();
        cp_async_wait<K6T_STAGES - 1>();
        __syncthreads();
        const double* sb = sm + int(c % K6T_STAGES) * PassB<T>::STAGE;
        const double* sw = sb + B_RB * B_LDB;
#pragma unroll
        for (int kk = 0; kk < B_KF; kk += 4) {
            const double a = sb[(warp * 8 + g) * B_LDB + kk + t4];  // A[g][t4] = B[row][f]
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(acc[j][0], acc[j][1], a, sw[(kk + t4) * T + j * 8 + g]);
        }
        __syncthreads();
    }
    cp_async_wait<0>();
    const int64_t row = r0 + warp * 8 + g;
    if (row < n) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {  // precond.cpp:12 divides by lambda_p
            const int64_t o = row * T + j * 8 + 2 * t4;
            Z[o] = (R[o] - acc[j][0]) / lambda_p;
            Z[o + 1] = (R[o + 1] - acc[j][1]) / lambda_p;
        }
    }
}

}  // namespace

int k6t_splits(int64_t n, int64_t s) {
    const int64_t fblocks = (s + A_FB - 1) / A_FB;
    int64_t splits = std::max<int64_t>(1, (148 * 4 + fblocks - 1) / fblocks);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, (n + 255) / 256));
    return int(splits);
}

// pass 1 writes Wpart (nsplit x s x T), reduced in fixed order into W (s x T); pass 2 writes Z
// rows [0, n) (the caller's row shard).  The allreduce of W (multi-rank) is the caller's: it
// runs between the passes, so this entry takes a flag for "pass 1 only" / "pass 2 only".
void precond_multi_launch(const double* B, int64_t n, int64_t s, const double* R, double lambda_p, double* Z,
                          double* Wpart, int nsplit, double* W, int T, int which, cudaStream_t stream) {
    if (T != 8 && T != 16) fail(KRR_ERR_INVALID_ARGUMENT, "K6T: T must be 8 or 16");
    if (which & 1) {
        if (n > 0) {
            const int64_t rows_per = (n + nsplit - 1) / nsplit;
            dim3 ga(unsigned((s + A_FB - 1) / A_FB), unsigned(nsplit));
            if (T == 16) {
                KRR_CUDA(cudaFuncSetAttribute(k6t_pass_a_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              int(PassA<16>::SMEM)));
                k6t_pass_a_kernel<16><<<ga, K6T_THREADS, PassA<16>::SMEM, stream>>>(B, n, s, R, Wpart, rows_per);
            } else {
                KRR_CUDA(cudaFuncSetAttribute(k6t_pass_a_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              int(PassA<8>::SMEM)));
                k6t_pass_a_kernel<8><<<ga, K6T_THREADS, PassA<8>::SMEM, stream>>>(B, n, s, R, Wpart, rows_per);
            }
            KRR_LAUNCH_CHECK();
            reduce_rows_launch(Wpart, nsplit, s * T, W, stream);
        } else {
            KRR_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * size_t(s * T), stream));
        }
    }
    if ((which & 2) && n > 0) {
        const unsigned nb = unsigned((n + B_RB - 1) / B_RB);
        if (T == 16) {
            KRR_CUDA(cudaFuncSetAttribute(k6t_pass_b_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(PassB<16>::SMEM)));
            k6t_pass_b_kernel<16><<<nb, K6T_THREADS, PassB<16>::SMEM, stream>>>(B, n, s, W, R, lambda_p, Z);
        } else {
            KRR_CUDA(cudaFuncSetAttribute(k6t_pass_b_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(PassB<8>::SMEM)));
            k6t_pass_b_kernel<8><<<nb, K6T_THREADS, PassB<8>::SMEM, stream>>>(B, n, s, W, R, lambda_p, Z);
        }
        KRR_LAUNCH_CHECK();
    }
}

}  // namespace krr
