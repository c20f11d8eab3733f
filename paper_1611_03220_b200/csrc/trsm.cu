// K5 — U = L^-1 Z^T in place (build_preconditioner, precond.cpp:38, via numerics::triangular_solve
// numerics.cpp:57-79: Side::Left, lower, no transpose), on the FP64 tensor path.
//
// On the device Z is n x s row-major and the result U^T overwrites it (precond.cu's B = U^T), so
// every data row k solves L u_k = z_k.  Left-looking blocked over 128-feature column blocks
// J = [j0, j0 + 128):
//     Y      = Z[:, J] - Z[:, 0:j0] L[J, 0:j0]^T     (GEMM, K = j0: DMMA m8n8k4)
//     Z[:, J] = forward substitution of each row of Y with the diagonal block L[J, J]
// One launch per column block, one CTA per 64 data rows: 8 warps x (32 rows x 32 columns) of
// DMMA accumulators, operands through a 3-stage cp.async ring of 32-feature stages with one barrier
// per stage (A: 64 rows x 32 features of the already-solved Z, B: the 32 x 128 block of L from L2);
// a stage's refill copies are issued between the first k-steps of the running stage, not as a burst.
// Then the CTA stages Y and L[J, J] in shared memory and each warp carries its 8 rows through the
// block together, lane m holding columns m, m + 32, m + 64, m + 96:
//     x_c = y_c (1 / L_cc), y_m -= L_mc x_c for m > c
// (the reference divides, numerics.cpp:70; the reciprocal, formed once per diagonal entry, costs
// at most one more rounding per step and removes 2 x 128 FP64 divisions per row pair).
// Work: n s^2 / 2 FMAs on the FP64 pipe (config 4: 3.5e13, config 5: 7.0e13); the substitution
// adds n s 64 FMAs (~1 % of the work, ~12 % of the time at config 4).  Measured (round 2, session 4):
// config 4 2.37 s = 0.80 of the live DMMA peak (cuBLAS DTRSM 2.64 s; this kernel before the
// single-barrier ring, the spread refill and the 8-row substitution: 2.97 s, same bits).  L is the column-major lower factor (L(i, k) at L[i + k s]).
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int RB = 64;    // data rows per CTA
constexpr int BW = 128;   // column block width
#ifndef TRSM_KC
#define TRSM_KC 32  // 64-feature stages, double-buffered: equal within 1 % (profiles/README.md, round 2 session 4)
#endif
#ifndef TRSM_NST
#define TRSM_NST 3
#endif
#ifndef TRSM_SPREAD
#define TRSM_SPREAD 4  // k-steps (of 4 features) over which a stage's refill copies are issued; 0: one burst
#endif
constexpr int SPREAD = TRSM_SPREAD;
constexpr int KC = TRSM_KC;    // features of K per stage
constexpr int NST = TRSM_NST;
static_assert(NST >= 2 && KC % 4 == 0 && SPREAD <= KC / 4, "K5: ring depth / stage width / refill spread");
constexpr int LDA = KC + 4;    // doubles; == 4 mod 32: A-fragment reads conflict-free
constexpr int LDB = BW + 4;    // doubles; == 4 mod 32: B-fragment reads conflict-free
constexpr int STAGE = RB * LDA + KC * LDB;
constexpr int LDY = BW + 1;    // Y tile row stride in the epilogue
constexpr size_t SMEM_MAIN = size_t(NST) * STAGE * 8;
constexpr size_t SMEM_EPI = size_t(RB) * LDY * 8 + size_t(BW) * BW * 8;
constexpr size_t SMEM = SMEM_MAIN > SMEM_EPI ? SMEM_MAIN : SMEM_EPI;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async16z(void* smem, const void* gmem, int ndoubles) {
    const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(8 * ndoubles));
}

template <bool V2>
__global__ void __launch_bounds__(256, 1) trsm_block_kernel(double* __restrict__ Z, int64_t n, int64_t s,
                                                            const double* __restrict__ L, int64_t j0, int bw) {
    extern __shared__ __align__(16) double sm[];
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int wr = warp >> 2, wc = warp & 3;  // warp tile: rows 32 wr .., columns 32 wc ..
    const int64_t r0 = int64_t(blockIdx.x) * RB;
    const int nk = int(j0 / KC);

    double acc[4][4][2];
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[m][q][0] = acc[m][q][1] = 0.0;

    auto load = [&](int kc, int st) {
        double* sa = sm + st * STAGE;
        double* sb = sa + RB * LDA;
        const int64_t k0 = int64_t(kc) * KC;
        if constexpr (V2) {  // s even: 16-byte aligned rows of Z and columns of L
            for (int e = tid; e < RB * KC / 2; e += 256) {
                const int r = e / (KC / 2), k = 2 * (e % (KC / 2));
                const bool ok = r0 + r < n;
                cp_async16z(sa + r * LDA + k, ok ? Z + (r0 + r) * s + k0 + k : Z, ok ? 2 : 0);
            }
            for (int e = tid; e < KC * BW / 2; e += 256) {
                const int k = e / (BW / 2), c = 2 * (e % (BW / 2));
                const int cnt = c + 1 < bw ? 2 : (c < bw ? 1 : 0);
                cp_async16z(sb + k * LDB + c, cnt ? L + (j0 + c) + (k0 + k) * s : L, cnt);
            }
        } else {
            for (int e = tid; e < RB * KC; e += 256) {
                const int r = e / KC, k = e % KC;
                const bool ok = r0 + r < n;
                cp_async8(sa + r * LDA + k, ok ? Z + (r0 + r) * s + k0 + k : Z, ok);
            }
            for (int e = tid; e < KC * BW; e += 256) {
                const int k = e / BW, c = e % BW;
                const bool ok = c < bw;
                cp_async8(sb + k * LDB + c, ok ? L + (j0 + c) + (k0 + k) * s : L, ok);
            }
        }
    };
    // the same copies one 256-thread unit at a time (s even): the refill of the next stage is spread
    // over the first SPREAD k-steps of the current one instead of issued as one burst after the
    // barrier (the burst stalled every warp on the load queue while the DMMA pipe idled)
    constexpr int NUA = RB * KC / 2 / 256, NUB = KC * BW / 2 / 256, NU = NUA + NUB;
    auto load_unit = [&](int kc, int st, int u) {
        double* sa = sm + st * STAGE;
        double* sb = sa + RB * LDA;
        const int64_t k0 = int64_t(kc) * KC;
        if (u < NUA) {
            const int e = tid + u * 256;
            const int r = e / (KC / 2), k = 2 * (e % (KC / 2));
            const bool ok = r0 + r < n;
            cp_async16z(sa + r * LDA + k, ok ? Z + (r0 + r) * s + k0 + k : Z, ok ? 2 : 0);
        } else {
            const int e = tid + (u - NUA) * 256;
            const int k = e / (BW / 2), c = 2 * (e % (BW / 2));
            const int cnt = c + 1 < bw ? 2 : (c < bw ? 1 : 0);
            cp_async16z(sb + k * LDB + c, cnt ? L + (j0 + c) + (k0 + k) * s : L, cnt);
        }
    };
#pragma unroll
    for (int st = 0; st < NST - 1; ++st) {
        if (st < nk) load(st, st);
        cp_async_commit();
    }
    // one barrier per stage: it publishes stage kc and retires stage kc - 1, which the refill
    // issued right after it overwrites
    for (int kc = 0; kc < nk; ++kc) {
        cp_async_wait<NST - 2>();
        __syncthreads();
        const bool refill = kc + NST - 1 < nk;
        const int rst = (kc + NST - 1) % NST;
        if (!(V2 && SPREAD > 0)) {
            if (refill) load(kc + NST - 1, rst);
            cp_async_commit();
        }
        const double* sa = sm + (kc % NST) * STAGE;
        const double* sb = sa + RB * LDA;
#pragma unroll
        for (int kk = 0; kk < KC; kk += 4) {
            if constexpr (V2 && SPREAD > 0) {
                constexpr int PER = (NU + SPREAD - 1) / (SPREAD > 0 ? SPREAD : 1);
                const int t = kk / 4;
                if (t < SPREAD && refill) {
#pragma unroll
                    for (int u = t * PER; u < (t + 1) * PER && u < NU; ++u) load_unit(kc + NST - 1, rst, u);
                }
                if (t == SPREAD - 1) cp_async_commit();
            }
            double a[4], b[4];
#pragma unroll
            for (int m = 0; m < 4; ++m) a[m] = sa[(wr * 32 + m * 8 + g) * LDA + kk + t4];  // A[g][t4] = Z[row][k]
#pragma unroll
            for (int q = 0; q < 4; ++q) b[q] = sb[(kk + t4) * LDB + wc * 32 + q * 8 + g];  // B[t4][g] = L[J+col][k]
#pragma unroll
            for (int m = 0; m < 4; ++m)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma884(acc[m][q][0], acc[m][q][1], a[m], b[q]);
        }
    }
    cp_async_wait<0>();
    __syncthreads();

    // Y = Z[rows, J] - acc into shared memory; L[J, J] (lower, column-major c * BW + m) beside it
    double* Y = sm;
    double* LJ = sm + RB * LDY;
#pragma unroll
    for (int m = 0; m < 4; ++m)
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int r = wr * 32 + m * 8 + g, c = wc * 32 + q * 8 + 2 * t4 + e;
                const int64_t row = r0 + r;
                const double z = (row < n && c < bw) ? Z[row * s + j0 + c] : 0.0;
                Y[r * LDY + c] = z - acc[m][q][e];
            }
    for (int e = tid; e < BW * BW; e += 256) {
        const int c = e / BW, m = e % BW;
        LJ[e] = (c < bw && m < bw && m >= c) ? L[(j0 + m) + (j0 + c) * s] : (m == c ? 1.0 : 0.0);
    }
    __syncthreads();
    if (tid < BW) LJ[tid * BW + tid] = 1.0 / LJ[tid * BW + tid];  // the diagonal holds 1 / L_cc
    __syncthreads();

    // forward substitution: each warp carries its 8 rows through the 128 columns together (8
    // independent dependency chains per step; every row sees the same operations in the same
    // order as a row-at-a-time substitution, so the result does not depend on the grouping)
    constexpr int RW = RB / 8;
    const int rw0 = warp * RW;
    double y[RW][4];
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) y[r][q] = Y[(rw0 + r) * LDY + lane + 32 * q];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        for (int cl = 0; cl < 32; ++cl) {
            const int c = 32 * q + cl;
            if (c >= bw) break;
            const double rcc = LJ[c * BW + c];
            double x[RW];
#pragma unroll
            for (int r = 0; r < RW; ++r) {
                x[r] = __shfl_sync(0xffffffffu, y[r][q], cl) * rcc;
                if (lane == cl) y[r][q] = x[r];
            }
#pragma unroll
            for (int q2 = q; q2 < 4; ++q2) {
                const int m = lane + 32 * q2;
                if (m > c) {
                    const double l = LJ[c * BW + m];
#pragma unroll
                    for (int r = 0; r < RW; ++r) y[r][q2] = fma(-l, x[r], y[r][q2]);
                }
            }
        }
    }
#pragma unroll
    for (int r = 0; r < RW; ++r)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int c = lane + 32 * q;
            if (c < bw && r0 + rw0 + r < n) Z[(r0 + rw0 + r) * s + j0 + c] = y[r][q];
        }
}

}  // namespace

// U^T (n x s row-major, in place over Z) = Z L^-T, i.e. U = L^-1 Z^T; L column-major lower s x s.
void trsm_lower_launch(double* Z, int64_t n, int64_t s, const double* L, cudaStream_t stream) {
    if (n <= 0 || s <= 0) return;
    const bool v2 = s % 2 == 0 && (reinterpret_cast<uintptr_t>(Z) & 15) == 0 && (reinterpret_cast<uintptr_t>(L) & 15) == 0;
    auto kern = v2 ? trsm_block_kernel<true> : trsm_block_kernel<false>;
    KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM)));
    const unsigned grid = unsigned((n + RB - 1) / RB);
    for (int64_t j0 = 0; j0 < s; j0 += BW) {
        const int bw = int(std::min<int64_t>(BW, s - j0));
        kern<<<grid, 256, SMEM, stream>>>(Z, n, s, L, j0, bw);
        KRR_LAUNCH_CHECK();
    }
}

}  // namespace krr
