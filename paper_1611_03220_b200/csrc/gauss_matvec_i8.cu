// K1-I8 — the fused symmetric Gaussian mat-vec with the dot products on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators), exact to
// fp64 level via an Ozaki-style slice decomposition.
//
// Why: on B200 the FP64 tensor path (DMMA) and DFMA share one FP64 datapath
// (37 TFLOP/s), and the d-long dot product is ~90 % of K1's FP64 work.  INT8 tensor
// throughput is ~120x larger, and integer MMA accumulates exactly.
//
// Decomposition (per row i, e_i = ilogb(max_k |x_ik|) + 1, u_i = x_i 2^-e_i in (-1, 1)):
//     u_i = sum_{p<8} A_i^(p) 2^(-7(p+1)) + r_i,   A^(p) in [-127, 127],  |r_i| < 2^-56
// (truncation, all steps exact in fp64).  Then
//     x_i . x_j = 2^(e_i + e_j) sum_{p,q} 2^(-7(p+q+2)) (A_i^(p) . A_j^(q))
// keeping p + q <= 7: 36 int8 GEMM products accumulated exactly in int32 into 8 TMEM
// groups c = p + q.  The epilogue recombines the groups in fp64 (pairs fused in int32,
// 4 exact int->fp64 conversions, 3 FMAs), forms d2 = |x_i|^2 + |x_j|^2 - 2 x_i.x_j,
// and continues exactly like K1 (table exp, row sums, column sums).  Dot-product error
// <= ~2^-52 * d * 2^(e_i + e_j), the same order as an fp64 dot product's bound.
//
// Structure (one CTA per symmetric super-tile, 10 warps):
//   warp 0     producer: 1-D bulk async copies (TMA engine) of the slice tiles into
//              shared memory — the I tile (128 rows x 8 slices, resident per I) and a
//              3-stage ring of J tiles (32 rows x 8 slices) — on mbarrier tx counts;
//   warp 1     MMA issuer: one thread issues 36 x (kp/32) tcgen05.mma (M = 128, N = 32,
//              K = 32) per 128 x 32 tile into one of two TMEM accumulator buffers
//              (2 x 8 groups x 32 columns = all 512 columns) and commits to mbarriers;
//   warps 2-9  epilogue: each thread owns one row (its TMEM lane) and 16 of the 32
//              columns; tcgen05.ld of the 8 groups, fp64 recombination + exp, row sums
//              in registers, column sums by a deterministic butterfly + fixed-order
//              shared-memory reduction.  Tile q's epilogue overlaps tile q+1's MMAs.
// Slots in `part` follow exactly the K1 rules (gauss_matvec.cu), so the finish kernel
// is shared.  Operand layout in global memory: slice p, 8-row group, 16-byte K chunk
// ([p][n_pad/8][kp/16][8][16]), so any 8-aligned row range is one contiguous block that
// is directly the canonical no-swizzle K-major UMMA layout (LBO = 128 B, SBO = 8 kp B).
#include "common.cuh"
#include "gauss_exp.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int P = 8;      // slices
constexpr int NGRP = 8;   // groups c = p + q in [0, 7]
constexpr int TI = 128;   // I tile rows (MMA M)
constexpr int TJ = 32;    // J tile columns (MMA N)
constexpr int NST = 3;    // J-tile stages
constexpr int NEPI = 8;   // epilogue warps
constexpr int NTHR = 32 * (2 + NEPI);
constexpr uint32_t TMEM_COLS = 512;
constexpr int KP_MAX = 96;

struct I8Args {
    const uint8_t* __restrict__ S;
    const int* __restrict__ ex;
    const double* __restrict__ sq;
    const double* __restrict__ v;
    double* __restrict__ part;
    const int2* __restrict__ tiles;
    const double* __restrict__ exp_tab;
    int64_t n_pad;
    int kp;
    int st;
    ExpConsts ec;
};

__device__ __forceinline__ double i2d_exact(int32_t b) {
    // 1.5 * 2^52 + (b + 2^31) built bitwise, minus the same constant: exact for all int32
    return __hiloint2double(0x43380000, int(uint32_t(b) ^ 0x80000000u)) - 6755401588539392.0;
}

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory"); }

size_t i8_smem_bytes(int kp, int st) {
    return size_t(P) * TI * kp + size_t(NST) * P * TJ * kp + sizeof(double) * (size_t(st) + 2 * TI + 2 * 2 * 4 * 16 + 64) +
           sizeof(uint64_t) * 16 + 16;
}

template <int KPT>
__global__ void __launch_bounds__(NTHR, 1) gauss_matvec_i8_kernel(const I8Args A) {
    extern __shared__ __align__(1024) uint8_t smem[];
    constexpr int kp = KPT;
    uint8_t* sA = smem;
    uint8_t* sB = sA + P * TI * kp;
    double* colacc = reinterpret_cast<double*>(sB + NST * P * TJ * kp);
    double* rowbuf = colacc + A.st;
    double* colscr = rowbuf + 2 * TI;        // [2 buffers][2 halves][4 quarters][16]
    double* tab = colscr + 2 * 2 * 4 * 16;  // 64
    uint64_t* bars = reinterpret_cast<uint64_t*>(tab + 64);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 1;
    uint64_t* b_full = bars + 2;
    uint64_t* b_empty = b_full + NST;
    uint64_t* t_full = b_empty + NST;
    uint64_t* t_empty = t_full + 2;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int2 tile = A.tiles[blockIdx.x];
    const int sa = tile.x, sb = tile.y;
    const bool diag = (sa == sb);
    const int nTI = A.st / TI, nTJ = A.st / TJ;
    const int64_t rowBase = int64_t(sa) * A.st;
    const int64_t colBase = int64_t(sb) * A.st;
    constexpr int ksteps = kp / 32;
    constexpr uint32_t sbo = uint32_t(kp) * 8;  // bytes between 8-row groups

    if (tid == 0) {
        tc::mbar_init(a_full, 1);
        tc::mbar_init(a_empty, 1);
        for (int s = 0; s < NST; ++s) {
            tc::mbar_init(b_full + s, 1);
            tc::mbar_init(b_empty + s, 1);
        }
        for (int b = 0; b < 2; ++b) {
            tc::mbar_init(t_full + b, 1);
            tc::mbar_init(t_empty + b, NEPI);
        }
        tc::mbar_fence_init();
    }
    for (int i = tid; i < A.st; i += NTHR) colacc[i] = 0.0;
    if (tid < 64) tab[tid] = A.exp_tab[tid];
    if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int bq = 0;
            for (int it = 0; it < nTI; ++it) {
                if (it > 0) tc::mbar_wait(a_empty, uint32_t((it - 1) & 1));
                tc::mbar_arrive_expect_tx(a_full, uint32_t(P * TI * kp));
                const int64_t r0 = rowBase + int64_t(it) * TI;
                for (int p = 0; p < P; ++p)
                    tc::bulk_g2s(sA + p * TI * kp, A.S + int64_t(p) * A.n_pad * kp + r0 * kp, uint32_t(TI * kp), a_full);
                for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                    const int s = bq % NST;
                    if (bq >= NST) tc::mbar_wait(b_empty + s, uint32_t(((bq / NST) - 1) & 1));
                    tc::mbar_arrive_expect_tx(b_full + s, uint32_t(P * TJ * kp));
                    const int64_t c0 = colBase + int64_t(jt) * TJ;
                    for (int q = 0; q < P; ++q)
                        tc::bulk_g2s(sB + (s * P + q) * TJ * kp, A.S + int64_t(q) * A.n_pad * kp + c0 * kp,
                                     uint32_t(TJ * kp), b_full + s);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        if (lane == 0) {
            const uint32_t idesc = tc::idesc_i8(TI, TJ);
            const uint32_t aBase = tc::smem_u32(sA);
            int bq = 0, tq = 0;
            for (int it = 0; it < nTI; ++it) {
                tc::mbar_wait(a_full, uint32_t(it & 1));
                tc::fence_after();
                for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq, ++tq) {
                    const int s = bq % NST, buf = tq & 1;
                    if (tq >= 2) tc::mbar_wait(t_empty + buf, uint32_t(((tq >> 1) - 1) & 1));
                    tc::mbar_wait(b_full + s, uint32_t((bq / NST) & 1));
                    tc::fence_after();
                    // Descriptors differ only in the start-address field (16-byte units):
                    // build the two bases once and add compile-time offsets, so the
                    // fully unrolled 36 x ksteps issue sequence is pure uniform adds.
                    const uint64_t dA0 = tc::smem_desc(aBase, 128, sbo);
                    const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sB + s * P * TJ * kp), 128, sbo);
                    const uint32_t dcol0 = tmem_base + uint32_t(buf * NGRP * TJ);
#pragma unroll
                    for (int p = 0; p < P; ++p)
#pragma unroll
                        for (int q = 0; q + p < NGRP; ++q)
#pragma unroll
                            for (int ks = 0; ks < ksteps; ++ks)
                                tc::mma_i8(dcol0 + uint32_t((p + q) * TJ),
                                           dA0 + uint64_t((p * TI * kp + ks * 256) >> 4),
                                           dB0 + uint64_t((q * TJ * kp + ks * 256) >> 4), idesc,
                                           (p == 0 && ks == 0) ? 0u : 1u);
                    tc::mma_commit(b_empty + s);
                    tc::mma_commit(t_full + buf);
                }
                tc::mma_commit(a_empty);
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp - 2;            // 0..7
        const int quarter = warp & 3;       // TMEM lane quarter this warp may access
        const int half = ew >> 2;           // which 16 of the 32 columns
        const int etid = ew * 32 + lane;    // 0..255
        const int row = quarter * 32 + lane;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        int tq = 0;
        for (int it = 0; it < nTI; ++it) {
            const int64_t gi = rowBase + int64_t(it) * TI + row;
            const int ei = A.ex[gi];
            const double sqi = A.sq[gi];
            const double vi = A.v[gi];
            double rowacc = 0.0;
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++tq) {
                const int buf = tq & 1;
                const bool dmask = diag && jt < (it + 1) * (TI / TJ);
                tc::mbar_wait(t_full + buf, uint32_t((tq >> 1) & 1));
                tc::fence_after();
                const int64_t jbase = colBase + int64_t(jt) * TJ + half * 16;
                double colv[16];
#pragma unroll
                for (int hb = 0; hb < 2; ++hb) {
                    uint32_t acc[NGRP][8];
#pragma unroll
                    for (int c = 0; c < NGRP; ++c)
                        tc::tmem_ld8(tmem_base + lane_addr + uint32_t(buf * NGRP * TJ + c * TJ + half * 16 + hb * 8),
                                     acc[c]);
                    tc::tmem_wait_ld();
                    if (hb == 1) {
                        // both halves of this thread's columns are in registers: release TMEM
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) tc::mbar_arrive(t_empty + buf);
                    }
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        const int64_t j = jbase + hb * 8 + jj;
                        const int32_t b0 = int32_t(acc[0][jj]) * 128 + int32_t(acc[1][jj]);
                        const int32_t b1 = int32_t(acc[2][jj]) * 128 + int32_t(acc[3][jj]);
                        const int32_t b2 = int32_t(acc[4][jj]) * 128 + int32_t(acc[5][jj]);
                        const int32_t b3 = int32_t(acc[6][jj]) * 128 + int32_t(acc[7][jj]);
                        double t = i2d_exact(b3);
                        t = fma(t, 0x1p-14, i2d_exact(b2));
                        t = fma(t, 0x1p-14, i2d_exact(b1));
                        t = fma(t, 0x1p-14, i2d_exact(b0));
                        // -2 x_i.x_j = t * (-2^(e_i + e_j - 20))
                        const int be = ei + A.ex[j] + (1023 - 20);
                        const double nscale = __hiloint2double(int(0x80000000u | (uint32_t(be) << 20)), 0);
                        const double d2 = fma(t, nscale, sqi + A.sq[j]);
                        double e = gauss_exp_table(d2, A.ec, tab);
                        if (dmask && j <= gi) e = 0.0;
                        rowacc = fma(e, A.v[j], rowacc);
                        colv[hb * 8 + jj] = e * vi;
                    }
                }
                // column sums over the warp's 32 rows: butterfly reduce-scatter, then lanes
                // (2c, 2c+1) hold column c's sum.
                double w8[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const double mine = (lane & 16) ? colv[8 + k] : colv[k];
                    const double other = (lane & 16) ? colv[k] : colv[8 + k];
                    w8[k] = mine + __shfl_xor_sync(0xffffffffu, other, 16);
                }
                double w4[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double mine = (lane & 8) ? w8[4 + k] : w8[k];
                    const double other = (lane & 8) ? w8[k] : w8[4 + k];
                    w4[k] = mine + __shfl_xor_sync(0xffffffffu, other, 8);
                }
                double w2[2];
#pragma unroll
                for (int k = 0; k < 2; ++k) {
                    const double mine = (lane & 4) ? w4[2 + k] : w4[k];
                    const double other = (lane & 4) ? w4[k] : w4[2 + k];
                    w2[k] = mine + __shfl_xor_sync(0xffffffffu, other, 4);
                }
                double w1;
                {
                    const double mine = (lane & 2) ? w2[1] : w2[0];
                    const double other = (lane & 2) ? w2[0] : w2[1];
                    w1 = mine + __shfl_xor_sync(0xffffffffu, other, 2);
                }
                w1 += __shfl_xor_sync(0xffffffffu, w1, 1);
                const int cb = tq & 1;
                if ((lane & 1) == 0) colscr[((cb * 2 + half) * 4 + quarter) * 16 + (lane >> 1)] = w1;
                epi_bar();
                if (etid < TJ) {
                    const int h = etid >> 4, c16 = etid & 15;
                    const double* cs = colscr + (cb * 2 + h) * 4 * 16 + c16;
                    colacc[jt * TJ + etid] += ((cs[0] + cs[16]) + cs[32]) + cs[48];
                }
            }
            // row partials of this I tile: combine the two column halves in fixed order
            rowbuf[half * TI + row] = rowacc;
            epi_bar();
            if (etid < TI) {
                const double r = rowbuf[etid] + rowbuf[TI + etid];
                if (diag) {
                    colacc[it * TI + etid] += r;
                } else {
                    A.part[int64_t(sb) * A.n_pad + rowBase + int64_t(it) * TI + etid] = r;
                }
            }
            epi_bar();
        }
    }

    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    // column sums (diag: combined row + column sums) -> this CTA's slot
    double* dst = A.part + int64_t(sa) * A.n_pad + (diag ? rowBase : colBase);
    for (int i = tid; i < A.st; i += NTHR) dst[i] = colacc[i];
    if (warp == 1) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

// ---- operand preparation
__global__ void row_exponent_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad,
                                    int* __restrict__ ex) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_pad; i += warps) {
        double m = 0.0;
        if (i < n)
            for (int64_t k = lane; k < d; k += 32) m = fmax(m, fabs(X[i * d + k]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) ex[i] = m > 0.0 ? ilogb(m) + 1 : 0;
    }
}

__global__ void slice_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, int kp,
                             const int* __restrict__ ex, uint8_t* __restrict__ S) {
    const int64_t total = n_pad * kp;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = idx / kp;
        const int k = int(idx % kp);
        const double x = (row < n && k < d) ? X[row * d + k] : 0.0;
        double w = scalbn(x, 7 - ex[row]);  // u * 2^7, |u| < 1
        const int64_t off = (row >> 3) * int64_t(kp) * 8 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            const double a = trunc(w);
            S[int64_t(p) * n_pad * kp + off] = uint8_t(int8_t(int(a)));
            w = (w - a) * 128.0;
        }
    }
}

__global__ void copy_sq_kernel(const double* __restrict__ L, int64_t n_pad, int dp, int d, double* __restrict__ sq) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad; i += int64_t(gridDim.x) * blockDim.x)
        sq[i] = L[i * dp + d];
}

}  // namespace

bool i8_supported(int64_t d, int st) {
    const int kp = int((d + 31) / 32 * 32);
    return kp <= KP_MAX && st % TI == 0 && i8_smem_bytes(kp, st) <= 227 * 1024;
}

int i8_kp(int64_t d) { return int((d + 31) / 32 * 32); }

void i8_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp, uint8_t* S,
                       int* ex, double* sq, cudaStream_t stream) {
    const int kp = i8_kp(d);
    const unsigned wblocks = unsigned(std::min<int64_t>((n_pad + 7) / 8, 148 * 16));
    row_exponent_kernel<<<wblocks, 256, 0, stream>>>(X, n, d, n_pad, ex);
    KRR_LAUNCH_CHECK();
    const int64_t total = n_pad * kp;
    slice_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, stream>>>(X, n, d, n_pad, kp,
                                                                                                 ex, S);
    KRR_LAUNCH_CHECK();
    copy_sq_kernel<<<unsigned(std::min<int64_t>((n_pad + 255) / 256, 148 * 8)), 256, 0, stream>>>(L, n_pad, dp,
                                                                                                  int(d), sq);
    KRR_LAUNCH_CHECK();
}

void gauss_matvec_i8_launch(const GaussMatvecPlan& p, const uint8_t* S, const int* ex, const double* sq,
                            const double* v, double* part, int kp, cudaStream_t stream) {
    if (p.num_tiles == 0) return;
    I8Args a;
    a.S = S;
    a.ex = ex;
    a.sq = sq;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.exp_tab = p.exp_tab;
    a.n_pad = p.n_pad;
    a.kp = kp;
    a.st = p.st;
    a.ec = p.ec;
    const size_t smem = i8_smem_bytes(kp, p.st);
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<unsigned(p.num_tiles), NTHR, smem, stream>>>(a);
    };
    if (kp == 32) run(gauss_matvec_i8_kernel<32>);
    else if (kp == 64) run(gauss_matvec_i8_kernel<64>);
    else if (kp == 96) run(gauss_matvec_i8_kernel<96>);
    else fail(KRR_ERR_INVALID_ARGUMENT, "K1-I8: kp must be 32, 64 or 96");
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
