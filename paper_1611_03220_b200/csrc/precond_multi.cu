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
// tensor path (DMMA m8n8k4, 256 FMAs per instruction, 8 independent accumulator tiles per
// warp).  B tiles are moved by the TMA engine: one 1-D bulk copy per row segment (1-2 KB
// contiguous: measured, shorter segments cost 2-3x) into a 4-stage mbarrier ring fed by a
// producer warp, so each SM keeps ~128 KB of loads in flight with a handful of instructions.
// Partial tiles are zero-filled by the producer rather than masked per lane: mma.sync must run
// in a converged warp (divergent masking around it hung the kernel).
// Measured at config 5 (n = 524288, s = 16384, t = 16; ncu, round 2 session 4): pass 1 14.2 ms, pass 2
// 14.8 ms = 4.7-4.8 TB/s, 0.72-0.74 of the measured HBM copy rate (round-2 start: 15.0 + 16.4 ms).
// What the probes say (K6T_PROBE, profiles/README.md): pass 1's copy pipeline alone streams U at
// 6.9 TB/s, so pass 1 is bound by its consumers (LDS + DMMA at ~55 % of the FP64 tensor rate with
// 2-4 warps per sub-partition; 16 consumer warps instead of 8: -4 %); pass 2's copy pipeline alone
// ran at 4.3 TB/s with 32-row CTAs because every CTA also pulls the whole W (2 MB) through L2 — a
// third of its ingest — so 64-row CTAs (W re-read half as often, two 84 KB stages): -10 %.  The
// FP64 datapath caps the kernel near 0.8 in any case: at the full copy rate (22 B/clk/SM = 2.8
// elements) 16 FMAs per element need 69 % of the 64 FMA/clk/SM that DMMA and DFMA share.
// Shared-memory strides are == 4 (mod 16) doubles and W carries an XOR column swizzle, so every
// fragment read is conflict-free (ncu before: 2 and 2.7 wavefronts per LDS.64 too many; fixing it
// did not change the time: the LSU pipe was at 25 / 45 %).
#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

#ifndef K6T_PROBE
#define K6T_PROBE 0  // A/B builds only (results invalid): 1 = no DMMA (copy pipeline + operand reads), 2 = no operand reads either
#endif
// W (s x T) is stored with the column XOR-swizzled by the feature row, so that pass 2's DMMA B
// fragments (4 consecutive feature rows x 8 columns per load, rows 8 T bytes apart) read
// conflict-free from the linearly copied chunk: T = 16: col ^ ((f & 3) << 2); T = 8: col ^ ((f & 2) << 1)
template <int T>
__host__ __device__ __forceinline__ int w_swz(int64_t f) {
    return T == 16 ? int((f & 3) << 2) : int((f & 2) << 1);
}
#ifndef K6T_RB
#define K6T_RB 64  // pass-2 rows per CTA: 64 rows x 2 stages re-read W half as often as 32 x 4 (-10 %, same bits)
#endif
#ifndef K6T_NSTB
#define K6T_NSTB 2
#endif
__device__ __forceinline__ void k6t_mma(double& d0, double& d1, double a, double b) {
    if (K6T_PROBE == 0) dmma884(d0, d1, a, b);
    else if (K6T_PROBE == 1) { d0 += a; d1 += b; }
}

constexpr int NSTAGE = 4;
constexpr int A_FB = 256;  // pass-1 feature block: 2 KB row segments (1 KB: 16.9 ms, 2 KB: 15.0 ms, 4 KB: 15.0 ms at config 5)
__host__ __device__ __forceinline__ int64_t imin64(int64_t a, int64_t b) { return a < b ? a : b; }
#ifndef K6T_NCWA
#define K6T_NCWA 16  // pass 1: 16 consumer warps (8: 4 % slower; each warp owns its features, so W does not depend on it)
#endif
constexpr int NCWA = K6T_NCWA;              // pass-1 consumer warps
constexpr int NTHREADS_A = 32 * (NCWA + 1);  // + one producer warp
constexpr int NCW = 8;                      // pass-2 consumer warps (they split K: the count fixes the summation order)
constexpr int NTHREADS = 32 * (NCW + 1);

// ---- pass 1: Wpart[split][f][T] = sum_{k in split} B[k][f] R[k][.] for an FB-feature block.
// Consumer warp w owns features f0 + w FB/8 .. (FB/64 DMMA M tiles) x all T columns; K = rows,
// KR = 4096 / FB per stage.  Stage: KR row segments of 8 FB bytes (32 KB); the KR x T block of R
// is read through L1.
template <int FB>
struct PassA {
    static constexpr int KR = 4096 / FB;
    static constexpr int LD = FB + 4;  // smem row stride (doubles), == 4 mod 16: the 4 feature rows of a half-warp's
                                       // A-fragment read (8 consecutive doubles each) fall in distinct bank groups
    static constexpr int MT = FB / (8 * NCWA);
    static constexpr int STAGE = KR * LD;  // doubles
    static constexpr int NST = 6;          // ring depth: ~192 KB of loads in flight per SM
    static constexpr size_t SMEM = size_t(NST) * STAGE * 8 + 2 * NST * 8 + 16;
};

template <int T, int FB>
__global__ void __launch_bounds__(NTHREADS_A, 1) k6t_pass_a_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                                                  const double* __restrict__ R,
                                                                  double* __restrict__ Wpart, int64_t rows_per) {
    using P = PassA<FB>;
    extern __shared__ __align__(128) double sm[];
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + P::NST * P::STAGE);
    uint64_t* empty = full + P::NST;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t f0 = int64_t(blockIdx.x) * FB;
    const int64_t k0 = int64_t(blockIdx.y) * rows_per;
    const int64_t k1 = min(n, k0 + rows_per);
    const int64_t nchunk = k1 > k0 ? (k1 - k0 + P::KR - 1) / P::KR : 0;
    const int fvalid = int(imin64(FB, s - f0));
    if (tid == 0) {
        for (int i = 0; i < P::NST; ++i) {
            tc::mbar_init(&full[i], 2);  // the producer's expect-tx arrive + its post-zero-fill arrive
            tc::mbar_init(&empty[i], NCWA);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();
    if (warp == NCWA) {  // producer
        for (int64_t c = 0; c < nchunk; ++c) {
            const int st = int(c % P::NST);
            if (c >= P::NST) tc::mbar_wait_sleep(&empty[st], uint32_t((c / P::NST - 1) & 1));
            const int64_t kb = k0 + c * P::KR;
            const int rows = int(imin64(P::KR, k1 - kb));
            const uint32_t seg = uint32_t(fvalid) * 8u;
            if (lane == 0) tc::mbar_arrive_expect_tx(&full[st], seg * uint32_t(rows));
            __syncwarp();
            double* sb = sm + st * P::STAGE;
            for (int r = lane; r < rows; r += 32) tc::bulk_g2s(sb + r * P::LD, B + (kb + r) * s + f0, seg, &full[st]);
            // a short last chunk: zero the rows past the split end (generic stores, published by the
            // release of lane 0's arrive below) so the MMA loop needs no per-lane masking
            if (rows < P::KR) {
                for (int e = lane; e < (P::KR - rows) * (FB / 2); e += 32) {
                    const int r = rows + e / (FB / 2), f = 2 * (e % (FB / 2));
                    *reinterpret_cast<double2*>(sb + r * P::LD + f) = make_double2(0.0, 0.0);
                }
            }
            __syncwarp();
            if (lane == 0) tc::mbar_arrive(&full[st]);
        }
        return;
    }
    constexpr int NT = T / 8;
    constexpr int MT = P::MT;
    double acc[MT][NT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
    for (int64_t c = 0; c < nchunk; ++c) {
        const int st = int(c % P::NST);
        tc::mbar_wait(&full[st], uint32_t((c / P::NST) & 1));
        const double* sb = sm + st * P::STAGE;
        const int64_t kb = k0 + c * P::KR;
        const int rows = int(imin64(P::KR, k1 - kb));
        // the KR x T block of R straight from global / L1 (every warp reads the same 2-4 KB)
        double bq[P::KR / 4][NT];
#pragma unroll
        for (int q = 0; q < P::KR / 4; ++q) {
            const int rr = 4 * q + t4 < rows ? 4 * q + t4 : 0;  // clamped, then zeroed: no branches
            const double m = 4 * q + t4 < rows ? 1.0 : 0.0;
#pragma unroll
            for (int j = 0; j < NT; ++j) bq[q][j] = m * __ldg(R + (kb + rr) * T + j * 8 + g);
        }
        __syncwarp();  // mma.sync below needs the converged warp
#pragma unroll
        for (int kk = 0; kk < P::KR; kk += 4) {
            const double* b = bq[kk / 4];
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const double a = sb[(kk + t4) * P::LD + warp * (FB / NCWA) + m * 8 + g];  // A[g][t4] = B[k][f]
#pragma unroll
                for (int j = 0; j < NT; ++j) k6t_mma(acc[m][j][0], acc[m][j][1], a, b[j]);
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[st]);
    }
#pragma unroll
    for (int m = 0; m < MT; ++m) {
        const int64_t f = f0 + warp * (FB / NCWA) + m * 8 + g;
        if (f < s) {
            double* w = Wpart + (int64_t(blockIdx.y) * s + f) * T;
#pragma unroll
            for (int j = 0; j < NT; ++j) {
                const int col = (j * 8 + 2 * t4) ^ w_swz<T>(f);  // the pair stays adjacent (bits 2-3 flip)
                w[col] = acc[m][j][0];
                w[col + 1] = acc[m][j][1];
            }
        }
    }
}

// ---- pass 2: Z[k][.] = (R[k][.] - B[k][:] W) / lambda_p for a 32-row block.
// The copy shape is pass 1's (32 row segments of 1 KB per stage: few, long bulk copies — 256-B
// segments measured 2-3x slower), plus the 128 x T block of W.  The 8 consumer warps split a
// stage's 128 features (16 each = 4 k-steps) and each accumulates all 4 x T/8 output tiles of
// the block; the partial tiles are summed across warps in fixed order at the end.
constexpr int B_RB = K6T_RB;
constexpr int B_KF = 128;
constexpr int B_LD = B_KF + 4;  // == 4 mod 16 doubles: the 4 rows of a half-warp's A-fragment read fall in distinct bank groups
constexpr int NSTB = K6T_NSTB;  // pass-2 ring stages
template <int T>
struct PassB {
    static constexpr int STAGE = B_RB * B_LD + B_KF * T;
    static_assert(NCW * B_RB * T <= NSTB * STAGE, "cross-warp partials reuse the stage buffers");
    static constexpr size_t SMEM = size_t(NSTB) * STAGE * 8 + 2 * NSTB * 8 + 16;
};

template <int T>
__global__ void __launch_bounds__(NTHREADS, 1) k6t_pass_b_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                                                  const double* __restrict__ W,
                                                                  const double* __restrict__ R, double lambda_p,
                                                                  double* __restrict__ Z) {
    extern __shared__ __align__(128) double sm[];
    double* red = sm;  // after the last stage: the cross-warp partials
    uint64_t* full = reinterpret_cast<uint64_t*>(sm + NSTB * PassB<T>::STAGE);
    uint64_t* empty = full + NSTB;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t r0 = int64_t(blockIdx.x) * B_RB;
    const int rows = int(imin64(B_RB, n - r0));
    const int64_t nchunk = (s + B_KF - 1) / B_KF;
    if (tid == 0) {
        for (int i = 0; i < NSTB; ++i) {
            tc::mbar_init(&full[i], 2);  // the producer's expect-tx arrive + its post-zero-fill arrive
            tc::mbar_init(&empty[i], NCW);
        }
        tc::mbar_fence_init();
    }
    __syncthreads();
    if (warp == NCW) {  // producer
        for (int64_t c = 0; c < nchunk; ++c) {
            const int st = int(c % NSTB);
            if (c >= NSTB) tc::mbar_wait_sleep(&empty[st], uint32_t((c / NSTB - 1) & 1));
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
    constexpr int MT = B_RB / 8;
    double acc[MT][NT][2];
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int j = 0; j < NT; ++j) acc[m][j][0] = acc[m][j][1] = 0.0;
    const int kw = warp * (B_KF / NCW);  // this warp's 16 features of each stage
    for (int64_t c = 0; c < nchunk; ++c) {
        const int st = int(c % NSTB);
        tc::mbar_wait(&full[st], uint32_t((c / NSTB) & 1));
        const double* sb = sm + st * PassB<T>::STAGE;
        const double* sw = sb + B_RB * B_LD;
#pragma unroll
        for (int kk = kw; kk < kw + B_KF / NCW; kk += 4) {
            double b[NT];
#pragma unroll
            for (int j = 0; j < NT; ++j) b[j] = sw[(kk + t4) * T + ((j * 8 + g) ^ w_swz<T>(t4))];  // kk % 4 == 0
#pragma unroll
            for (int m = 0; m < MT; ++m) {
                const double a = sb[(m * 8 + g) * B_LD + kk + t4];  // A[g][t4] = B[row][f]
#pragma unroll
                for (int j = 0; j < NT; ++j) k6t_mma(acc[m][j][0], acc[m][j][1], a, b[j]);
            }
        }
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&empty[st]);
    }
    // cross-warp sum in fixed order (warp 0 + 1 + ... + 7), then the Woodbury finish; the stage
    // buffers are idle once every consumer warp is past its last stage
    asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NCW) : "memory");  // consumer warps only
    double* mine = red + warp * (B_RB * T);
#pragma unroll
    for (int m = 0; m < MT; ++m)
#pragma unroll
        for (int j = 0; j < NT; ++j) {
            mine[(m * 8 + g) * T + j * 8 + 2 * t4] = acc[m][j][0];
            mine[(m * 8 + g) * T + j * 8 + 2 * t4 + 1] = acc[m][j][1];
        }
    asm volatile("bar.sync 1, %0;\n" ::"r"(32 * NCW) : "memory");  // consumer warps only
    for (int e = tid; e < rows * T; e += 32 * NCW) {
        double y = 0.0;
#pragma unroll
        for (int w = 0; w < NCW; ++w) y += red[w * (B_RB * T) + e];
        const int64_t o = r0 * T + e;
        Z[o] = (R[o] - y) / lambda_p;  // precond.cpp:12 divides by lambda_p
    }
}

template <int T>
void k6t_run(const double* B, int64_t n, int64_t s, const double* R, double lambda_p, double* Z, double* Wpart,
             int nsplit, double* W, int which, cudaStream_t stream) {
    if (which & 1) {
        if (n > 0) {
            const int64_t rows_per = (n + nsplit - 1) / nsplit;
            dim3 ga(unsigned((s + A_FB - 1) / A_FB), unsigned(nsplit));
            KRR_CUDA(cudaFuncSetAttribute(k6t_pass_a_kernel<T, A_FB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          int(PassA<A_FB>::SMEM)));
            k6t_pass_a_kernel<T, A_FB><<<ga, NTHREADS_A, PassA<A_FB>::SMEM, stream>>>(B, n, s, R, Wpart, rows_per);
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
