// K3-I8 — the Gram matrix of the sketch, G = Z^T Z (build_preconditioner, precond.cpp:23), on the
// 5th-generation tensor cores: tcgen05.mma kind::i8 with TMEM accumulators, exact to better than
// fp64 level through the same Ozaki slice decomposition as K1-I8 (gauss_matvec_i8.cu).
//
// Decomposition (per feature column j, e_j = ilogb(max_k |z_kj|) + 1, u = z 2^-e_j in (-1, 1)):
//     u_kj = sum_{p<8} A_kj^(p) 2^(-7(p+1)) + r,   A^(p) in [-127, 127],  |r| < 2^-56
//     G_ij = sum_k z_ki z_kj = 2^(e_i + e_j - 14) sum_c 2^(-7c) sum_{p+q=c} sum_k A_ki^(p) A_kj^(q)
// keeping c <= 7 (36 int8 products per 32-row chunk, accumulated exactly in int32 in 8 TMEM
// groups).  Truncation error per entry <= ~2^-55 n 2^(e_i + e_j): below an fp64 SYRK's own
// rounding bound (n eps |z_i||z_j|), so the Cholesky sees fp64-quality G.  int32 exactness
// bounds one accumulation to 16384 rows (8 x 127^2 x 16384 < 2^31): rows are processed in
// units of 16384, each unit's tile converted to fp64 and added into G (one writer per element,
// fixed unit order: deterministic).
//
// Layout: the rows of one unit are sliced into S[p][kc][s_pad/8][2][8][16] (kc = 32-row chunk),
// so any 8-aligned run of features of one chunk is one contiguous block in the canonical
// no-swizzle K-major UMMA layout (LBO = 128 B between the two 16-byte K halves, SBO = 256 B
// between 8-row groups) — a 128-feature A tile is one 4 KB bulk copy, a 64-feature B tile 2 KB.
// One CTA per lower 128 x 64 tile of G (M = 128 features of I, N = 64 of J), 6 warps:
//   warp 0   producer: 16 bulk copies (TMA engine) per chunk into a 4-stage ring (48 KB each)
//   warp 1   MMA issuer: 36 tcgen05.mma per chunk, group c = 7 .. 0 into TMEM columns 64 c
//   warps 2-5 epilogue: drain the 8 groups once per unit (tcgen05.ld), combine in int64,
//            convert, scale by 2^(e_i + e_j - 35) and add into G (column-major lower triangle,
//            the layout the Cholesky reads: element (i >= j) at G[j s + i], coalesced in i).
// Bound: the tensor core.  Per unit and tile, 512 chunks x 36 MMAs of 128 x 64 x 32 B at the
// N = 64 rate (~45-48 clk, shared-memory operand reads), i.e. (n s^2 / 2) x 36 int8 MACs per
// Gram: config 4 (n = 2^20, s = 8192) 1.3e15 MACs, config 5 (2^19, 16384) 2.5e15.
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int P = 8;       // slices
constexpr int NGRP = 8;    // groups c = p + q in [0, 7]
constexpr int TI = 128;    // G tile rows (features of I; MMA M, TMEM lanes)
constexpr int TJ = 64;     // G tile columns (features of J; MMA N)
constexpr int NSTG = 4;    // chunk ring stages
constexpr int A_CH = P * TI * 32;  // 32 KB of A slices per chunk
constexpr int B_CH = P * TJ * 32;  // 16 KB of B slices per chunk
constexpr int STG = A_CH + B_CH;
constexpr int NTHR = 32 * 6;
constexpr uint32_t TMEM_COLS = 512;
constexpr size_t SMEM = size_t(NSTG) * STG + 1024;

struct GramArgs {
    const uint8_t* __restrict__ S;  // slices of the unit
    const int* __restrict__ ex;     // e_j per feature (s_pad)
    const int2* __restrict__ tiles; // (I block, J block) of each lower tile
    double* __restrict__ G;         // s x s, column-major lower triangle accumulated
    int64_t s, s_pad;
    int kchunks;                    // 32-row chunks in this unit (<= 512)
};

// exact int64 combination of one column's 8 group sums -> 2^21 sum_c 2^-7c G_c (one rounding
// in each conversion): b_k = 128 G_2k + G_2k+1, H = 2^14 b_0 + b_1, Lo = 2^14 b_2 + b_3
__device__ __forceinline__ double combine(const int32_t (&gc)[NGRP]) {
    const int64_t b0 = int64_t(gc[0]) * 128 + gc[1];
    const int64_t b1 = int64_t(gc[2]) * 128 + gc[3];
    const int64_t b2 = int64_t(gc[4]) * 128 + gc[5];
    const int64_t b3 = int64_t(gc[6]) * 128 + gc[7];
    const int64_t H = b0 * 16384 + b1;
    const int64_t Lo = b2 * 16384 + b3;
    return fma(double(Lo), 0x1p-28, double(H));
}

__global__ void __launch_bounds__(NTHR, 1) gram_i8_kernel(const GramArgs A) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sStg = smem;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + size_t(NSTG) * STG);
    uint64_t* s_full = bars;
    uint64_t* s_empty = bars + NSTG;
    uint64_t* done = bars + 2 * NSTG;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * NSTG + 1);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int2 tile = A.tiles[blockIdx.x];
    const int64_t I0 = int64_t(tile.x) * TI, J0 = int64_t(tile.y) * TJ;
    const int64_t g8 = A.s_pad / 8;

    if (tid == 0) {
        for (int s = 0; s < NSTG; ++s) {
            tc::mbar_init(s_full + s, 1);
            tc::mbar_init(s_empty + s, 1);
        }
        tc::mbar_init(done, 1);
        tc::mbar_fence_init();
    }
    if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            for (int kc = 0; kc < A.kchunks; ++kc) {
                const int s = kc % NSTG;
                if (kc >= NSTG) tc::mbar_wait_sleep(s_empty + s, uint32_t((kc / NSTG - 1) & 1));
                tc::mbar_arrive_expect_tx(s_full + s, uint32_t(STG));
                uint8_t* st = sStg + s * STG;
                for (int p = 0; p < P; ++p) {
                    const uint8_t* base = A.S + (int64_t(p) * A.kchunks + kc) * g8 * 256;
                    tc::bulk_g2s(st + p * (TI * 32), base + (I0 >> 3) * 256, uint32_t(TI * 32), s_full + s);
                    tc::bulk_g2s(st + A_CH + p * (TJ * 32), base + (J0 >> 3) * 256, uint32_t(TJ * 32), s_full + s);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer (converged warp,
        // elect.sync lane: no per-MMA waterfall loop, gauss_matvec_i8.cu)
        const uint32_t idesc = tc::idesc_i8(TI, TJ);
        for (int kc = 0; kc < A.kchunks; ++kc) {
            const int s = kc % NSTG;
            tc::mbar_wait_sleep(s_full + s, uint32_t((kc / NSTG) & 1));
            tc::fence_after();
            const uint32_t sbase = tc::smem_u32(sStg + s * STG);
            const uint64_t dA0 = tc::smem_desc(sbase, 128, 256);
            const uint64_t dB0 = tc::smem_desc(sbase + A_CH, 128, 256);
            if (tc::elect_one()) {
#pragma unroll
                for (int c = NGRP - 1; c >= 0; --c) {
#pragma unroll
                    for (int p = 0; p <= c; ++p)
                        tc::mma_i8(tmem_base + uint32_t(c * TJ), dA0 + uint64_t((p * TI * 32) >> 4),
                                   dB0 + uint64_t(((c - p) * TJ * 32) >> 4), idesc, (kc == 0 && p == 0) ? 0u : 1u);
                }
                tc::mma_commit(s_empty + s);
                if (kc == A.kchunks - 1) tc::mma_commit(done);
            }
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue: 4 warps, one per
        // TMEM lane quarter; thread = one feature i of the I tile, 8 columns at a time
        const int quarter = warp & 3;
        const int64_t i = I0 + quarter * 32 + lane;
        const int ei = A.ex[i];
        tc::mbar_wait_sleep(done, 0);
        tc::fence_after();
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16);
#pragma unroll 1
        for (int cb = 0; cb < TJ; cb += 8) {
            uint32_t r[NGRP][8];
#pragma unroll
            for (int c = 0; c < NGRP; ++c) tc::tmem_ld8(taddr + uint32_t(c * TJ + cb), r[c]);
            tc::tmem_wait_ld();
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int64_t j = J0 + cb + k;
                if (i >= j && i < A.s) {
                    int32_t gc[NGRP];
#pragma unroll
                    for (int c = 0; c < NGRP; ++c) gc[c] = int32_t(r[c][k]);
                    const double v = ldexp(combine(gc), ei + A.ex[j] - 35);
                    double* dst = A.G + j * A.s + i;
                    *dst += v;
                }
            }
        }
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

// max |z| per feature column (bit pattern of a non-negative double: integer max == double max)
// and a non-finite flag
__global__ void colmax_kernel(const double* __restrict__ Z, int64_t rows, int64_t s, int64_t rows_per,
                              unsigned long long* __restrict__ maxbits, int* __restrict__ bad) {
    const int64_t j = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (j >= s) return;
    const int64_t k0 = int64_t(blockIdx.y) * rows_per;
    const int64_t k1 = min(rows, k0 + rows_per);
    double m = 0.0;
    bool nf = false;
    for (int64_t k = k0; k < k1; ++k) {
        const double z = Z[k * s + j];
        nf |= !isfinite(z);
        m = fmax(m, fabs(z));
    }
    if (nf) atomicOr(bad, 1);
    if (m > 0.0) atomicMax(maxbits + j, static_cast<unsigned long long>(__double_as_longlong(m)));
}

__global__ void exponent_kernel(const unsigned long long* __restrict__ maxbits, int64_t s_pad, int* __restrict__ ex) {
    for (int64_t j = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; j < s_pad; j += int64_t(gridDim.x) * blockDim.x) {
        const double m = __longlong_as_double(static_cast<long long>(maxbits[j]));
        ex[j] = (m > 0.0 && isfinite(m)) ? ilogb(m) + 1 : 0;
    }
}

// Slices of rows [r0, r0 + kchunks * 32) (rows >= `rows` are zero): one thread per (feature j,
// 16-row half of a chunk); 16 values -> 8 slices x 16 bytes (one 16-byte store each).
__global__ void gram_slice_kernel(const double* __restrict__ Z, int64_t rows, int64_t s, int64_t s_pad, int64_t r0,
                                  int kchunks, const int* __restrict__ ex, uint8_t* __restrict__ S) {
    const int64_t total = int64_t(kchunks) * 2 * s_pad;
    const int64_t g8 = s_pad / 8;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t j = idx % s_pad;
        const int64_t h = idx / s_pad;  // 16-row half index within the unit
        const int kc = int(h >> 1), hb = int(h & 1);
        const int sh = 7 - ex[j];
        uint32_t dig[P][4] = {};
#pragma unroll
        for (int rr = 0; rr < 16; ++rr) {
            const int64_t k = r0 + h * 16 + rr;
            double w = (j < s && k < rows) ? scalbn(Z[k * s + j], sh) : 0.0;  // u * 2^7, |u| < 1
#pragma unroll
            for (int p = 0; p < P; ++p) {
                const double a = trunc(w);
                dig[p][rr >> 2] |= uint32_t(uint8_t(int8_t(int(a)))) << (8 * (rr & 3));
                w = (w - a) * 128.0;
            }
        }
        const int64_t off = (int64_t(kc) * g8 + (j >> 3)) * 256 + hb * 128 + (j & 7) * 16;
#pragma unroll
        for (int p = 0; p < P; ++p)
            *reinterpret_cast<uint4*>(S + int64_t(p) * kchunks * g8 * 256 + off) =
                make_uint4(dig[p][0], dig[p][1], dig[p][2], dig[p][3]);
    }
}

__global__ void fill_nan_kernel(double* G, int64_t count) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < count; k += int64_t(gridDim.x) * blockDim.x)
        G[k] = __longlong_as_double(0x7FF8000000000000LL);
}

}  // namespace

constexpr int64_t kGramUnitRows = 16384;  // int32-exact accumulation bound (8 x 127^2 x 16384 < 2^31)

int64_t gram_i8_spad(int64_t s) { return (s + TI - 1) / TI * TI; }

size_t gram_i8_scratch_bytes(int64_t rows, int64_t s) {
    const int64_t unit = std::min<int64_t>(kGramUnitRows, (std::max<int64_t>(1, rows) + 31) / 32 * 32);
    return size_t(P) * size_t(unit) * size_t(gram_i8_spad(s));
}

// G (s x s column-major; lower triangle incl. diagonal written, upper untouched) = Z^T Z over the
// `rows` x s row-major Z.  scratch: gram_i8_scratch_bytes; ex: s_pad ints; maxbits: s_pad u64;
// bad: one int; tiles: (s_pad/128) * (s_pad/64) int2.  Returns nothing; a non-finite Z makes G NaN
// (the caller's Cholesky then fails, as LLT does on the reference's non-finite G).
void gram_i8_launch(const double* Z, int64_t rows, int64_t s, double* G, uint8_t* scratch, int* ex,
                    unsigned long long* maxbits, int* bad, int2* tiles, cudaStream_t stream) {
    const int64_t s_pad = gram_i8_spad(s);
    KRR_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * size_t(s * s), stream));
    if (rows <= 0) return;
    KRR_CUDA(cudaMemsetAsync(maxbits, 0, sizeof(unsigned long long) * size_t(s_pad), stream));
    KRR_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), stream));
    {
        const unsigned bx = unsigned((s + 255) / 256);
        const int64_t ry = std::max<int64_t>(1, std::min<int64_t>(int64_t(148 * 8) / bx + 1, (rows + 255) / 256));
        const int64_t rows_per = (rows + ry - 1) / ry;
        colmax_kernel<<<dim3(bx, unsigned(ry)), 256, 0, stream>>>(Z, rows, s, rows_per, maxbits, bad);
        KRR_LAUNCH_CHECK();
        exponent_kernel<<<unsigned(std::min<int64_t>((s_pad + 255) / 256, 148 * 4)), 256, 0, stream>>>(maxbits, s_pad, ex);
        KRR_LAUNCH_CHECK();
    }
    // lower tiles (I block of 128, J block of 64 with J start < I end), heaviest rows first
    const int nbi = int(s_pad / TI);
    std::vector<int2> h;
    for (int bi = nbi - 1; bi >= 0; --bi)
        for (int bj = 0; bj < 2 * (bi + 1); ++bj) h.push_back(make_int2(bi, bj));
    KRR_CUDA(cudaMemcpyAsync(tiles, h.data(), sizeof(int2) * h.size(), cudaMemcpyHostToDevice, stream));
    KRR_CUDA(cudaFuncSetAttribute(gram_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM)));
    for (int64_t r0 = 0; r0 < rows; r0 += kGramUnitRows) {
        const int64_t ur = std::min<int64_t>(kGramUnitRows, rows - r0);
        const int kchunks = int((ur + 31) / 32);
        const int64_t work = int64_t(kchunks) * 2 * s_pad;
        gram_slice_kernel<<<unsigned(std::min<int64_t>((work + 255) / 256, 148 * 16)), 256, 0, stream>>>(
            Z, rows, s, s_pad, r0, kchunks, ex, scratch);
        KRR_LAUNCH_CHECK();
        GramArgs a;
        a.S = scratch;
        a.ex = ex;
        a.tiles = tiles;
        a.G = G;
        a.s = s;
        a.s_pad = s_pad;
        a.kchunks = kchunks;
        gram_i8_kernel<<<unsigned(h.size()), NTHR, SMEM, stream>>>(a);
        KRR_LAUNCH_CHECK();
    }
    int hbad = 0;
    KRR_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    if (hbad) {
        fill_nan_kernel<<<unsigned(std::min<int64_t>((s * s + 255) / 256, 148 * 8)), 256, 0, stream>>>(G, s * s);
        KRR_LAUNCH_CHECK();
    }
}

}  // namespace krr
