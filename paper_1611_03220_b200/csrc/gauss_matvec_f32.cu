// K1-F32 — the optional fp32-accuracy mode of the fused symmetric Gaussian mat-vec
// (BASELINE north_star: "an optional fp32/3xTF32 mode is reported separately with its
// residual history"; SURVEY.md §8b krr_set_precision).  The PCG around it stays fp64.
//
// Dot products on the 5th-generation tensor cores: each x_ik is split into three bf16
// parts (round to nearest: b0 = bf16(x), b1 = bf16(x - b0), b2 = bf16(x - b0 - b1); 24
// significant bits), and x_i.x_j = sum_{p+q<=2} b_i^(p) . b_j^(q) — six bf16 products, exact
// in fp32, accumulated by tcgen05.mma kind::f16 into ONE fp32 TMEM accumulator (the dropped
// products are ~2^-24 relative: fp32 level).  One accumulator per tile means four TMEM
// buffers (4 x 64 of the 512 columns), so the MMAs of the next tiles run while the epilogue
// drains this one.  The epilogue is fp32: y = log2(e) * (-scale d2) = s_i + s_j + 2c D with
// s = -c |x|^2, c = scale log2(e), clamped at 0, e = ex2.approx(y) on the SFU; per-tile row
// and column sums in fp32, accumulated across tiles in fp64.  Relative error of K v: ~1e-6.
//
// Structure mirrors K1-I8 (gauss_matvec_i8.cu): one CTA per symmetric super-tile, warp 0
// producer (1-D bulk async copies of the resident I tile, a ring of J tiles and of the
// per-column data), warp 1 MMA issuer, 16 epilogue warps (4 per TMEM lane quarter, one row
// x 16 columns each), deterministic slots in `part` (one writer per slot and index).
// Operand layout: part p, 8-row group, 16-byte K chunk ([p][n_pad/8][kb/16][8][16], kb =
// 2 * kpe bytes per row, kpe = d rounded up to 16 elements) — the canonical no-swizzle
// K-major UMMA layout (LBO = 128 B, SBO = 8 kb B), byte-identical in structure to K1-I8's.
#include <cuda_bf16.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int NPART = 3;  // bf16 parts
constexpr int TI = 128;   // I tile rows (MMA M)
constexpr int TJ = 64;    // J tile columns (MMA N)
constexpr int NACC = 4;   // TMEM accumulator buffers
constexpr int NCD = 4;    // column-data stages
constexpr int NEPI = 16;  // epilogue warps
constexpr int CPT = 16;   // columns per epilogue thread per tile
constexpr int CPP = 2 * CPT;  // per tile pair (the epilogue consumes two tiles per step)
constexpr int NTHR = 32 * (2 + NEPI);
constexpr uint32_t TMEM_COLS = 256;
constexpr int SCR_LD = 33;
constexpr int CD_BYTES = TJ * 4 * 2;  // s (fp32), v (fp32)
constexpr int KB_MAX = 256;           // bytes per row per part (d <= 128)

template <int KB>
struct CfgF {
    static constexpr size_t A_BYTES = size_t(NPART) * TI * KB;
    static constexpr size_t B_BYTES = size_t(NPART) * TJ * KB;
    static constexpr size_t SCR_BYTES = size_t(NEPI) * CPP * SCR_LD * 4;
    static constexpr size_t FIXED = NCD * CD_BYTES + SCR_BYTES + 2 * 4 * 2 * TJ * 4 + 512;
    static constexpr size_t FIT = (232448 - A_BYTES - FIXED) / B_BYTES;
    static constexpr int NSTB = FIT >= 3 ? 3 : int(FIT);  // J-tile stages that fit
    static_assert(NSTB >= 1, "K1-F32: operand tiles do not fit");
    static constexpr size_t OFF_B = A_BYTES;
    static constexpr size_t OFF_CD = OFF_B + NSTB * B_BYTES;
    static constexpr size_t OFF_SCR = OFF_CD + NCD * CD_BYTES;
    static constexpr size_t OFF_COLSCR = OFF_SCR + (SCR_BYTES > 4 * TI * 8 ? SCR_BYTES : 4 * TI * 8);
    static constexpr size_t OFF_BARS = OFF_COLSCR + 2 * 4 * 2 * TJ * 4;
    static constexpr int NBARS = 2 + 2 * NSTB + 2 * NCD + 2 * NACC;
    static constexpr size_t SMEM = OFF_BARS + NBARS * 8 + 16;
};

struct F32Args {
    const uint8_t* __restrict__ S;  // bf16 parts
    const float* __restrict__ s;    // -c |x|^2
    const float* __restrict__ v;    // v as fp32
    double* __restrict__ part;
    const int2* __restrict__ tiles;
    int64_t n_pad;
    int st;
    float c2;  // 2 c = 2 scale log2(e)
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory"); }

__device__ __forceinline__ float ex2_approx(float y) {
    float r;
    asm("ex2.approx.ftz.f32 %0, %1;\n" : "=f"(r) : "f"(y));
    return r;
}

template <int KB>
__global__ void __launch_bounds__(NTHR, 1) gauss_matvec_f32_kernel(const F32Args A) {
    using C = CfgF<KB>;
    constexpr int NSTB = C::NSTB;
    constexpr int ksteps = KB / 32;
    constexpr uint32_t sbo = uint32_t(KB) * 8;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::OFF_B;
    uint8_t* sCD = smem + C::OFF_CD;
    float* scr_all = reinterpret_cast<float*>(smem + C::OFF_SCR);
    double* rowbuf = reinterpret_cast<double*>(smem + C::OFF_SCR);  // pass ends only
    float* colscr = reinterpret_cast<float*>(smem + C::OFF_COLSCR);  // [2][4 quarters][64]
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BARS);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 1;
    uint64_t* b_full = bars + 2;
    uint64_t* b_empty = b_full + NSTB;
    uint64_t* cd_full = b_empty + NSTB;
    uint64_t* cd_empty = cd_full + NCD;
    uint64_t* t_full = cd_empty + NCD;
    uint64_t* t_empty = t_full + NACC;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + NACC);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int2 tile = A.tiles[blockIdx.x];
    const int sa = tile.x, sb = tile.y;
    const bool diag = (sa == sb);
    const int nTI = A.st / TI, nTJ = A.st / TJ;
    const int64_t rowBase = int64_t(sa) * A.st;
    const int64_t colBase = int64_t(sb) * A.st;

    if (tid == 0) {
        tc::mbar_init(a_full, 1);
        tc::mbar_init(a_empty, 1);
        for (int s = 0; s < NSTB; ++s) {
            tc::mbar_init(b_full + s, 1);
            tc::mbar_init(b_empty + s, 1);
        }
        for (int s = 0; s < NCD; ++s) {
            tc::mbar_init(cd_full + s, 1);
            tc::mbar_init(cd_empty + s, NEPI);
        }
        for (int b = 0; b < NACC; ++b) {
            tc::mbar_init(t_full + b, 1);
            tc::mbar_init(t_empty + b, NEPI);
        }
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
            int bq = 0;
            for (int it = 0; it < nTI; ++it) {
                if (it > 0) tc::mbar_wait_sleep(a_empty, uint32_t((it - 1) & 1));
                tc::mbar_arrive_expect_tx(a_full, uint32_t(C::A_BYTES));
                const int64_t r0 = rowBase + int64_t(it) * TI;
                for (int p = 0; p < NPART; ++p)
                    tc::bulk_g2s(sA + p * TI * KB, A.S + int64_t(p) * A.n_pad * KB + r0 * KB, uint32_t(TI * KB), a_full);
                for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                    const int s = bq % NSTB;
                    if (bq >= NSTB) tc::mbar_wait_sleep(b_empty + s, uint32_t(((bq / NSTB) - 1) & 1));
                    tc::mbar_arrive_expect_tx(b_full + s, uint32_t(C::B_BYTES));
                    const int64_t c0 = colBase + int64_t(jt) * TJ;
                    for (int q = 0; q < NPART; ++q)
                        tc::bulk_g2s(sB + s * C::B_BYTES + q * TJ * KB, A.S + int64_t(q) * A.n_pad * KB + c0 * KB,
                                     uint32_t(TJ * KB), b_full + s);
                    const int cs = bq % NCD;
                    if (bq >= NCD) tc::mbar_wait_sleep(cd_empty + cs, uint32_t(((bq / NCD) - 1) & 1));
                    tc::mbar_arrive_expect_tx(cd_full + cs, uint32_t(CD_BYTES));
                    uint8_t* cd = sCD + cs * CD_BYTES;
                    tc::bulk_g2s(cd, A.s + c0, TJ * 4, cd_full + cs);
                    tc::bulk_g2s(cd + TJ * 4, A.v + c0, TJ * 4, cd_full + cs);
                }
            }
        }
    } else if (warp == 1) {
        // ------------------------------------------------------------ MMA issuer
        // converged warp, one elect.sync lane issues (no per-MMA ELECT/R2UR waterfall loop; the
        // same change made K1-I8 3 % faster, gauss_matvec_i8.cu)
        constexpr uint32_t idesc = tc::idesc_bf16(TI, TJ);
        const uint32_t aBase = tc::smem_u32(sA);
        int bq = 0;
        for (int it = 0; it < nTI; ++it) {
            tc::mbar_wait_sleep(a_full, uint32_t(it & 1));
            tc::fence_after();
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                const int s = bq % NSTB, buf = bq % NACC;
                if (bq >= NACC) tc::mbar_wait_sleep(t_empty + buf, uint32_t(((bq / NACC) - 1) & 1));
                tc::mbar_wait_sleep(b_full + s, uint32_t((bq / NSTB) & 1));
                tc::fence_after();
                const uint64_t dA0 = tc::smem_desc(aBase, 128, sbo);
                const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sB + s * C::B_BYTES), 128, sbo);
                const uint32_t d = tmem_base + uint32_t(buf * TJ);
                // small products first (fp32 accumulation), then the leading one
                constexpr int PP[6] = {2, 1, 0, 1, 0, 0};
                constexpr int QQ[6] = {0, 1, 2, 0, 1, 0};
                if (tc::elect_one()) {
#pragma unroll
                    for (int m = 0; m < 6; ++m)
#pragma unroll
                        for (int ks = 0; ks < ksteps; ++ks)
                            tc::mma_f16(d, dA0 + uint64_t((PP[m] * TI * KB + ks * 256) >> 4),
                                        dB0 + uint64_t((QQ[m] * TJ * KB + ks * 256) >> 4), idesc,
                                        (m == 0 && ks == 0) ? 0u : 1u);
                    tc::mma_commit(b_empty + s);
                    tc::mma_commit(t_full + buf);
                }
                __syncwarp();
            }
            if (tc::elect_one()) tc::mma_commit(a_empty);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue
        // Two consecutive 64-column tiles per step (every pass has an even tile count):
        // one barrier, one transpose and one owner update per 128 columns.
        const int ew = warp - 2;
        const int quarter = warp & 3;
        const int part = ew >> 2;  // which 16 of each tile's 64 columns
        const int etid = ew * 32 + lane;
        const int row = quarter * 32 + lane;
        const int colOff = part * CPT;
        const uint32_t lane_addr = uint32_t(quarter * 32) << 16;
        float* scr = scr_all + ew * CPP * SCR_LD;
        int tq = 0;
        for (int it = 0; it < nTI; ++it) {
            const int64_t gi = rowBase + int64_t(it) * TI + row;
            const float s_i = A.s[gi];
            const float v_i = A.v[gi];
            double rowacc = 0.0;
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; jt += 2, tq += 2) {
                // owner thread of pair column etid (< 128): the same thread every pass
                double* cdst = A.part + int64_t(sa) * A.n_pad + colBase + int64_t(jt) * TJ + etid;
                double cprev = 0.0;
                if (etid < 2 * TJ && it > 0) cprev = *cdst;
                uint32_t dr[CPP];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int buf = (tq + h) % NACC;
                    tc::mbar_wait(t_full + buf, uint32_t(((tq + h) / NACC) & 1));
                }
                tc::fence_after();
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    uint32_t(&d16)[CPT] = *reinterpret_cast<uint32_t(*)[CPT]>(dr + h * CPT);
                    tc::tmem_ld16(tmem_base + lane_addr + uint32_t(((tq + h) % NACC) * TJ + colOff), d16);
                }
                tc::tmem_wait_ld();
                tc::fence_before();
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(t_empty + tq % NACC);
                    tc::mbar_arrive(t_empty + (tq + 1) % NACC);
                }
                const float* cds[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int cs = (tq + h) % NCD;
                    tc::mbar_wait(cd_full + cs, uint32_t(((tq + h) / NCD) & 1));
                    cds[h] = reinterpret_cast<const float*>(sCD + cs * CD_BYTES);
                }
                // the pair (2it, 2it+1) of a diagonal super-tile is the diagonal block: keep
                // pair column > row
                const bool masked = diag && jt == it * (TI / TJ);
                float rt0 = 0.f, rt1 = 0.f;
                auto exp_cols = [&](auto mask_tag) {
                    constexpr bool MASK = decltype(mask_tag)::value;
#pragma unroll
                    for (int k = 0; k < CPP; ++k) {
                        const int h = k / CPT, cl = colOff + (k % CPT);
                        // y = log2(e) (-scale) d2 = s_i + s_j + 2c x_i.x_j, clamped at 0 (d2 >= 0)
                        const float y = fminf(fmaf(__uint_as_float(dr[k]), A.c2, s_i + cds[h][cl]), 0.f);
                        float e = ex2_approx(y);
                        if constexpr (MASK) e = (h * TJ + cl > row) ? e : 0.f;
                        if (k & 1) rt1 = fmaf(e, cds[h][TJ + cl], rt1);
                        else rt0 = fmaf(e, cds[h][TJ + cl], rt0);
                        scr[k * SCR_LD + lane] = e * v_i;
                    }
                };
                if (masked) exp_cols(std::true_type{});
                else exp_cols(std::false_type{});
                rowacc += double(rt0 + rt1);
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(cd_empty + tq % NCD);
                    tc::mbar_arrive(cd_empty + (tq + 1) % NCD);
                }
                // column sums over the warp's 32 rows: lane k sums its column over all 32 rows
                {
                    const float* src = scr + lane * SCR_LD;
                    float a0 = 0.f, a1 = 0.f, a2 = 0.f, a3 = 0.f;
#pragma unroll
                    for (int r = 0; r < 32; r += 4) {
                        a0 += src[r];
                        a1 += src[r + 1];
                        a2 += src[r + 2];
                        a3 += src[r + 3];
                    }
                    const int pc = (lane / CPT) * TJ + colOff + (lane % CPT);  // pair column
                    colscr[((tq >> 1) & 1) * 4 * 2 * TJ + quarter * 2 * TJ + pc] = (a0 + a1) + (a2 + a3);
                }
                __syncwarp();
                epi_bar();
                if (etid < 2 * TJ) {
                    const float* q4 = colscr + ((tq >> 1) & 1) * 4 * 2 * TJ + etid;
                    *cdst = cprev + double((q4[0] + q4[2 * TJ]) + (q4[4 * TJ] + q4[6 * TJ]));
                }
            }
            // pass end: row partials, 4 column parts combined in fixed order; the pair-column
            // owner (index mod 128) adds on diagonal super-tiles
            rowbuf[part * TI + row] = rowacc;
            epi_bar();
            if (etid < TI) {
                const double rs = ((rowbuf[etid] + rowbuf[TI + etid]) + rowbuf[2 * TI + etid]) + rowbuf[3 * TI + etid];
                if (diag) {
                    double* dst = A.part + int64_t(sa) * A.n_pad + rowBase + int64_t(it) * TI + etid;
                    *dst = *dst + rs;
                } else {
                    A.part[int64_t(sb) * A.n_pad + rowBase + int64_t(it) * TI + etid] = rs;
                }
            }
            epi_bar();
        }
    }

    tc::fence_before();
    __syncthreads();
    if (warp == 1) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

// ---- operand preparation: three bf16 parts per element, s = -c |x|^2 in fp32
__global__ void bf16_split_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, int kb,
                                  uint8_t* __restrict__ S) {
    const int kpe = kb / 2;
    const int64_t total = n_pad * kpe;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = idx / kpe;
        const int k = int(idx % kpe);
        double x = (row < n && k < d) ? X[row * d + k] : 0.0;
        const int kbyte = 2 * k;
        const int64_t off = (row >> 3) * int64_t(kb) * 8 + (kbyte >> 4) * 128 + (row & 7) * 16 + (kbyte & 15);
#pragma unroll
        for (int p = 0; p < NPART; ++p) {
            const __nv_bfloat16 b = __float2bfloat16_rn(float(x));  // x -> fp32 -> bf16 (nearest)
            *reinterpret_cast<__nv_bfloat16*>(S + int64_t(p) * n_pad * kb + off) = b;
            x -= double(__bfloat162float(b));  // exact residual in fp64
        }
    }
}

__global__ void f32_side_kernel(const double* __restrict__ L, int64_t n_pad, int dp, int d, double c,
                                float* __restrict__ s) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad; i += int64_t(gridDim.x) * blockDim.x)
        s[i] = float(-c * L[i * dp + d]);
}

__global__ void to_f32_kernel(const double* __restrict__ v, int64_t n, float* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n; i += int64_t(gridDim.x) * blockDim.x)
        out[i] = float(v[i]);
}

template <int KB>
void launch_kb(const F32Args& a, int64_t num_tiles, cudaStream_t stream) {
    constexpr size_t smem = CfgF<KB>::SMEM;
    static_assert(smem <= 227 * 1024, "K1-F32 shared memory");
    KRR_CUDA(cudaFuncSetAttribute(gauss_matvec_f32_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    gauss_matvec_f32_kernel<KB><<<unsigned(num_tiles), NTHR, smem, stream>>>(a);
}

}  // namespace

bool f32_supported(int64_t d, int st) { return d <= KB_MAX / 2 && st % TI == 0 && st >= TI; }

int f32_kb(int64_t d) { return int((d + 15) / 16 * 16) * 2; }

void f32_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp, double scale,
                        uint8_t* S, float* s, cudaStream_t stream) {
    const int kb = f32_kb(d);
    const int64_t total = n_pad * (kb / 2);
    bf16_split_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, stream>>>(X, n, d, n_pad,
                                                                                                      kb, S);
    KRR_LAUNCH_CHECK();
    const double c = scale * 1.4426950408889634;  // scale log2(e)
    f32_side_kernel<<<unsigned(std::min<int64_t>((n_pad + 255) / 256, 148 * 8)), 256, 0, stream>>>(L, n_pad, dp,
                                                                                                    int(d), c, s);
    KRR_LAUNCH_CHECK();
}

void gauss_matvec_f32_launch(const GaussMatvecPlan& p, const uint8_t* S, const float* s, const double* v,
                             float* v32, double* part, int kb, double scale, cudaStream_t stream) {
    if (p.num_tiles == 0) return;
    to_f32_kernel<<<unsigned(std::min<int64_t>((p.n_pad + 255) / 256, 148 * 8)), 256, 0, stream>>>(v, p.n_pad, v32);
    KRR_LAUNCH_CHECK();
    F32Args a;
    a.S = S;
    a.s = s;
    a.v = v32;
    a.part = part;
    a.tiles = p.tiles;
    a.n_pad = p.n_pad;
    a.st = p.st;
    a.c2 = float(2.0 * scale * 1.4426950408889634);
    if (kb == 32) launch_kb<32>(a, p.num_tiles, stream);
    else if (kb == 64) launch_kb<64>(a, p.num_tiles, stream);
    else if (kb == 96) launch_kb<96>(a, p.num_tiles, stream);
    else if (kb == 128) launch_kb<128>(a, p.num_tiles, stream);
    else if (kb == 160) launch_kb<160>(a, p.num_tiles, stream);
    else if (kb == 192) launch_kb<192>(a, p.num_tiles, stream);
    else if (kb == 224) launch_kb<224>(a, p.num_tiles, stream);
    else if (kb == 256) launch_kb<256>(a, p.num_tiles, stream);
    else fail(KRR_ERR_INVALID_ARGUMENT, "K1-F32: unsupported row width");
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
