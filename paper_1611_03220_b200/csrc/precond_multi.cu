// K6T — the Woodbury apply for T interleaved right-hand sides (T = 8 or 16), the per-iteration
// preconditioner of the batched PCG (BASELINE config 5: t = 16, s = 16384).
//
// Reference: Preconditioner::apply_columns (precond.cpp:15-18): Z = (R - U^T (U R)) / lambda_p.
// On the device U is stored as B = U^T (n x s row-major, precond.cu), R and Z are n x T
// row-major (interleaved columns), so both passes stream B once:
//   pass 1 (K6T-a):  W (s x T) = B^T R    — 128-feature blocks x row splits, deterministic partials
//   pass 2 (K6T-b):  Z = (R - B W) / lambda_p
// Bound: HBM, 2 x 8 n s bytes per apply (config 5: 2 x 68.7 GB).  At T = 16 every 8-byte element
// of B feeds 16 FMAs, ~70 % of the FP64 pipe at the HBM rate, so the contraction runs on the FP64
// tensor path (DMMA m8n8k4, 256 FMAs per instruction, 8 independent accumulator chains per
// warp).  B tiles are moved by the TMA engine: one 1-D bulk copy per row segment (512 B / 1 KB
// contiguous) into a 4-stage mbarrier ring fed by a producer warp, so each SM keeps ~128 KB of
// loads in flight with a handful of instructions.
#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int NSTAGE = 4;
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
constexpr int NCW = 8;                    // consumer warps
constexpr int NTHREADS = 32 * (NCW + 1);  // + one producer warp

// ---- pass 1: Wpart[split][f][T] = sum_{k in split} B[k][f] R[k][.] for a 128-feature block.
// Consumer warp w owns features f0 + 16w .. + 16 (2 DMMA M tiles) x all T columns; K = rows,
// 32 per stage.  Stage: 32 row segments of 1 KB; the 32 x T block of R is read through L1.
constexpr int A_FB = 128;
constexpr int A_KR = 32;
constexpr int A_LD = A_FB + 8;  // smem row stride (doubles), == 8 mod 32: A-fragment reads conflict-free
template <int T>
struct PassA {
    static constexpr int STAGE = A_KR * A_LD;  // doubles
    static constexpr size_t SMEM = size_t(NSTAGE) * STAGE * 8 + 2 * NSTAGE * 8 + 16;
};

template <int T>
__global__ void __launch_bounds__(NTHREADS, 1) k6t_pass_a_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                                                  const double* __restrict__ R,
                                                                  double* __restrict__ Wpart, int64_t rows_per) {
    extern __shared__ __align__(128) double sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSTAGE * PassA<T>::STAGE);
    uint64_t* empty = full + NSTAGE;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t f0 = int64_t(blockIdx.x) * A_FB;
    const int64_t k0 = int64_t(blockIdx.y) * rows_per;
    const int64_t k1 = min(n, k0 + rows_per);
    const int64_t nchunk = k1 > k0 ? (k1 - k0 + A_KR - 1) / A_KR : 0;
    const int fvalid = int(imin64(A_FB, s - f0));
    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            tc::mbar_init(&full[i], 2);  // the producer's expect-tx arrive + its post-zero-fill arrive
            tc::mbar_init(&empty[i], NCW);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();
    if (warp == NCW) {  // producer
        for (int64_t c = 0; c < nchunk; ++c) {
            const int st = int(c % NSTAGE);
            if (c >= NSTAGE) tc::mbar_wait_sleep(&empty[st], uint32_t((c / NSTAGE - 1) & 1));
            const int64_t kb = k0 + c * A_KR;
            const int rows = int(imin64(A_KR, k1 - kb));
            const uint32_t seg = uint32_t(fvalid) * 8u;
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], seg * uint32_t(rows));
            __syncwarp();
            double* sb = sm + st * PassA<T>::STAGE;
            for (int r = lane; r < rows; r += 32) tc::bulk_g2s(sb + r * A_LD, B + (kb + r) * s + f0, seg, &full[st]);
            // a short last chunk: zero the rows past the split end (generic stores, published by the
            // release of lane 0's arrive below) so the MMA loop needs no per-lane masking
            if (rows < A_KR) {
                for (int e = lane; e < (A_KR - rows) * (A_FB / 2); e += 32) {
                    const int r = rows + e / (A_FB / 2), f = 2 * (e % (A_FB / 2));
                    *reinterpret_cast<double2*>(sb + r * A_LD + f) = make_double2(0.0, 0.0);
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[st]);
        }
        return;
    }
    constexpr int NT = T / 8;
    double acc[2][2][NT][2];  // [K chain][M tile][N tile][2]
#pragma unroll
    for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int j = 0; j < NT; ++j) acc[q][m][j][0] = acc[q][m][j][1] = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) {
        const int st = int(c % NSTAGE);
        tc::mbar_wait(&full[st], uint32_t((c / NSTAGE) & 1));
        const double* sb = sm + st * PassA<T>::STAGE;
        const int64_t kb = k0 + c * A_KR;
        const int rows = int(imin64(A_KR, k1 - kb));
        // the 32 x T block of R straight from global / L1 (every warp reads the same 2-4 KB)
        double bq[A_KR / 4][NT];
#pragma unroll
        for (int q = 0; q < A_KR / 4; ++q) {
            const int rr = 4 * q + t4 < rows ? 4 * q + t4 : 0;  // clamped, then zeroed: no branches
            const double m = 4 * q + t4 < rows ? 1.0 : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) bq[q][j] = m * __ldg(R + (kb + rr) * T + j * 8 + g);
        }
        __syncwarp();  // mma.sync below needs the converged warp
#pragma unroll
        for (int kk = 0; kk < A_KR; kk += 4) {
            const double* b = bq[kk / 4];
            auto& ac = acc[(kk / 4) & 1];
#pragma unroll
            for (int m = 0; m < 2; ++m) {
                const double a = sb[(kk + t4) * A_LD + warp * 16 + m * 8 + g];  // A[g][t4] = B[k][f]
#pragma unroll
                for (int j = 0; j < NT; ++j) dmma884(ac[m][j][0], ac[m][j][1], a, b[j]);
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int m = 0; m < 2; ++m) {
        const int64_t f = f0 + warp * 16 + m * 8 + g;
        if (f < s) {
            double* w = Wpart + (int64_t(blockIdx.y) * s + f) * T;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                w[j * 8 + 2 * t4] = acc[0][m][j][0] + acc[1][m][j][0];
                w[j * 8 + 2 * t4 + 1] = acc[0][m][j][1] + acc[1][m][j][1];
            }
        }
    }
}

// ---- pass 2: Z[k][.] = (R[k][.] - B[k][:] W) / lambda_p for a 64-row block.
// Consumer warp w owns rows r0 + 8w .. + 8 (DMMA M) x all T columns; K = features, 64 per stage.
// Stage: 64 row segments of 512 B + the 64 x T block of W (contiguous).
constexpr int B_RB = 64;
constexpr int B_KF = 64;
constexpr int B_LD = B_KF + 4;  // == 4 mod 32 doubles: A-fragment reads conflict-free
template <int T>
struct PassB {
    static constexpr int STAGE = B_RB * B_LD + B_KF * T;
    static constexpr size_t SMEM = size_t(NSTAGE) * STAGE * 8 + 2 * NSTAGE * 8 + 16;
};

template <int T>
__global__ void __launch_bounds__(NTHREADS, 1) k6t_pass_b_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                                                  const double* __restrict__ W,
                                                                  const double* __restrict__ R, double lambda_p,
                                                                  double* __restrict__ Z) {
    extern __shared__ __align__(128) double sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSTAGE * PassB<T>::STAGE);
    uint64_t* empty = full + NSTAGE;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t r0 = int64_t(blockIdx.x) * B_RB;
    const int rows = int(imin64(B_RB, n - r0));
    const int64_t nchunk = (s + B_KF - 1) / B_KF;
    if (tid == 0) {
        for (int i = 0; i < NSTAGE; ++i) {
            tc::mbar_init(&full[i], 2);  // the producer's expect-tx arrive + its post-zero-fill arrive
            tc::mbar_init(&empty[i], NCW);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();
    if (warp == NCW) {  // producer
        for (int64_t c = 0; c < nchunk; ++c) {
            const int st = int(c % NSTAGE);
            if (c >= NSTAGE) tc::mbar_wait_sleep(&empty[st], uint32_t((c / NSTAGE - 1) & 1));
            const int64_t fb = c * B_KF;
            const int fv = int(imin64(B_KF, s - fb));
            const uint32_t seg = uint32_t(fv) * 8u;
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], seg * uint32_t(rows) + uint32_t(fv * T * 8));
            __syncwarp();
            double* sb = sm + st * PassB<T>::STAGE;
            for (int r = lane; r < rows; r += 32) tc::bulk_g2s(sb + r * B_LD, B + (r0 + r) * s + fb, seg, &full[st]);
            if (lane == 0) tc::bulk_g2s(sb + B_RB * B_LD, W + fb * T, uint32_t(fv * T * 8), &full[st]);
            // the last feature chunk may be short: zero its missing columns of B and rows of W
            // (generic stores published by lane 0's arrive) so the MMA loop needs no masking
            if (fv < B_KF) {
                for (int e = lane; e < rows * (B_KF - fv); e += 32)
                    sb[(e / (B_KF - fv)) * B_LD + fv + e % (B_KF - fv)] = 0.0;
                for (int e = lane; e < (B_KF - fv) * T; e += 32) sb[B_RB * B_LD + fv * T + e] = 0.0;
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[st]);
        }
        return;
    }
    constexpr int NT = T / 8;
    constexpr int KI = 4;
    double acc[KI][NT][2];
#pragma unroll
    for (int q = 0; q < KI; ++q)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[q][j][0] = acc[q][j][1] = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) {
        const int st = int(c % NSTAGE);
        tc::mbar_wait(&full[st], uint32_t((c / NSTAGE) & 1));
        const double* sb = sm + st * PassB<T>::STAGE;
        const double* sw = sb + B_RB * B_LD;
#pragma unroll
        for (int kk = 0; kk < B_KF; kk += 4) {
            const double a = sb[(warp * 8 + g) * B_LD + kk + t4];  // A[g][t4] = B[row][f]
            auto& ac = acc[(kk / 4) % KI];
#pragma unroll
            for (int j = 0; j < NT; ++j) dmma884(ac[j][0], ac[j][1], a, sw[(kk + t4) * T + j * 8 + g]);
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[st]);
    }
    const int64_t row = r0 + warp * 8 + g;
    if (row < n) {
#pragma unroll
        for (int j = 0; j < NT; ++j) {  // precond.cpp:12 divides by lambda_p
            const double y0 = (acc[0][j][0] + acc[1][j][0]) + (acc[2][j][0] + acc[3][j][0]);
            const double y1 = (acc[0][j][1] + acc[1][j][1]) + (acc[2][j][1] + acc[3][j][1]);
            const int64_t o = row * T + j * 8 + 2 * t4;
            Z[o] = (R[o] - y0) / lambda_p;
            Z[o + 1] = (R[o + 1] - y1) / lambda_p;
        }
    }
}

template <int T>
void k6t_run(const double* B, int64_t n, int64_t s, const double* R, double lambda_p, double* Z, double* Wpart,
             int nsplit, double* W, int which, cudaStream_t stream) {
    if (which & 1) {
        if (n > 0) {
            const int64_t rows_per = (n + nsplit - 1) / nsplit;
            dim3 ga(unsigned((s + A_FB - 1) / A_FB), unsigned(nsplit));
            KRR_CUDA(cudaFuncSetAttribute(k6t_pass_a_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(PassA<T>::SMEM)));
            k6t_pass_a_kernel<T><<<ga, NTHREADS, PassA<T>::SMEM, stream>>>(B, n, s, R, Wpart, rows_per);
            KRR_LAUNCH_CHECK();
            reduce_rows_launch(Wpart, nsplit, s * T, W, stream);
        } else {
            KRR_CUDA(cudaMemsetAsync(W, 0, sizeof(double) * size_t(s * T), stream));
        }
    }
    if ((which & 2) && n > 0) {
        KRR_CUDA(cudaFuncSetAttribute(k6t_pass_b_kernel<T>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                      int(PassB<T>::SMEM)));
        k6t_pass_b_kernel<T><<<unsigned((n + B_RB - 1) / B_RB), NTHREADS, PassB<T>::SMEM, stream>>>(B, n, s, W, R,
                                                                                                    lambda_p, Z);
        KRR_LAUNCH_CHECK();
    }
}

}  // namespace

// Row splits of pass 1: enough CTAs for ~8 waves of 148 SMs.
int k6t_splits(int64_t n, int64_t s) {
    const int64_t fblocks = (s + A_FB - 1) / A_FB;
    int64_t splits = std::max<int64_t>(1, (148 * 8 + fblocks - 1) / fblocks);
    splits = std::min<int64_t>(splits, std::max<int64_t>(1, (n + 1023) / 1024));
    return int(splits);
}

bool k6t_supported(int64_t s, const void* B) { return s % 2 == 0 && (reinterpret_cast<uintptr_t>(B) & 15) == 0; }

// pass 1 writes Wpart (nsplit x s x T), reduced in fixed order into W (s x T); pass 2 writes Z
// rows [0, n) (the caller's row shard).  The all-reduce of W (multi-rank) runs between the
// passes, hence `which` (1 = pass 1, 2 = pass 2, 3 = both).  Needs 16-byte aligned row starts
// for the bulk copies (s even): k6t_supported.
void precond_multi_launch(const double* B, int64_t n, int64_t s, const double* R, double lambda_p, double* Z,
                          double* Wpart, int nsplit, double* W, int T, int which, cudaStream_t stream) {
    if (!k6t_supported(s, B)) fail(KRR_ERR_INVALID_ARGUMENT, "K6T: needs an even sketch size s");
    if (T == 16)
        k6t_run<16>(B, n, s, R, lambda_p, Z, Wpart, nsplit, W, which, stream);
    else if (T == 8)
        k6t_run<8>(B, n, s, R, lambda_p, Z, Wpart, nsplit, W, which, stream);
    else
        fail(KRR_ERR_INVALID_ARGUMENT, "K6T: T must be 8 or 16");
}

}  // namespace krr
