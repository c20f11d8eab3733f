// K1T-I8 — fused symmetric Gaussian mat-mat  OUT = (K + lambda I) V  for T = 16 interleaved
// right-hand sides (BASELINE config 5: n = 524288, d = 440, t = 16 one-vs-all RLSC targets),
// K never stored.  The dot products run on the 5th-generation tensor cores exactly as in
// K1-I8 (gauss_matvec_i8.cu: tcgen05.mma kind::i8 on 7 Ozaki slices of balanced 8-bit digits, 28
// products in 7 TMEM groups, the same integer drain and table exp), so every K_ij is K1-I8's bit pattern;
// the E . V contractions run on the FP64 tensor path (DMMA m8n8k4):
//     rows:     O_I (128 x 16) += E (128 x 64)   . V_J (64 x 16)    (accumulated over a pass)
//     columns:  O_J (64 x 16)   = E^T (64 x 128) . V_I (128 x 16)   (one J tile)
//
// Differences from K1-I8, both forced by d = 440:
//  * K-streamed operands.  The I tile's slices (7 x 128 x 448 B = 392 KB) cannot stay
//    resident, so both operands stream through a 2-stage ring of 32-byte K chunks
//    (7 slices x (128 + 64) rows x 32 B = 42 KB per stage), one bulk copy (TMA engine) per
//    slice and operand.  The MMAs are then shared-memory-bandwidth bound: (128 + 64) x 32 B
//    of SS operand reads per MMA plus the TMA fills, ~57 clk per MMA (a 3rd stage and an
//    L2 prefetch one tile ahead were measured slower, profiles/README.md).  The slices use a K-chunk-major global layout
//    [p][kp/32][n_pad/8][2][8][16] so that a chunk of any 128 (64) consecutive rows is one
//    contiguous 4 KB (2 KB) block in the canonical no-swizzle K-major UMMA layout
//    (LBO = 128 B between the two 16-byte K halves, SBO = 256 B between 8-row groups).
//  * T = 16 right-hand sides.  The exp phase writes E (masked on the diagonal blocks) to a
//    shared-memory tile (row stride 68 doubles, column XOR-swizzled by row / 4, so both the
//    row-per-lane stores and the DMMA fragment reads of E and E^T are bank-conflict free);
//    warps 0-7 of the epilogue then contract rows (2 m8 blocks each, C fragments kept in
//    registers for the whole 128-row pass), warps 8-15 columns (one 8-column block each,
//    K = 128).  V tiles are stored with the column XOR-swizzled by (row % 4) * 4.
//
// Unlike K1-I8, the FP64 phase (exp + DMMA) of a tile overlaps the next tile's MMAs: with
// the tensor core at ~60 % duty (shared-memory bound) the FP64 throttling under INT8 MMAs
// costs less than serialising (config 5: 2.84 s vs 3.17 s per pass; MI8_TMUX=1 restores
// K1-I8's time-multiplexing).
//
// Reductions are deterministic and atomic-free with the K1 / K1T slot rules (part is
// NS x n_pad x T, element (slot, i, c) at (slot * n_pad + i) * T + c): rows of super-row a
// -> slot b, columns of super-column b -> slot a; on a diagonal super-tile both go to slot a
// and the column owner thread adds the rows at the end of each pass.  matmat_finish_launch
// (gauss_matvec_multi.cu) sums the slots, adds K_ii v_i = v_i and lambda v.
#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gauss_exp.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int P = 7;       // slices (balanced 8-bit digits, tc_i8.cuh:balanced_digits8)
constexpr int NGRP = 7;    // groups c = p + q in [0, 6]
constexpr int TI = 128;    // I tile rows (MMA M, TMEM lanes)
constexpr int TJ = 64;     // J tile columns (MMA N)
constexpr int TR = 16;     // right-hand sides
constexpr int NEPI = 16;   // epilogue warps (4 per TMEM lane quarter)
constexpr int CPT = 16;    // columns per epilogue thread
constexpr int NTHR = 32 * (2 + NEPI);
#ifndef MI8_MMA_LAST
#define MI8_MMA_LAST 0  // 1: control warps last (epilogue 0-15, producer 16, MMA 17): the issue arbiter prefers
                        // high warp ids, and here the epilogue's exp / DMMA work runs beside the MMAs
#endif
constexpr int WARP_PROD = MI8_MMA_LAST ? NEPI : 0, WARP_MMA = MI8_MMA_LAST ? NEPI + 1 : 1;
constexpr uint32_t TMEM_COLS = 512;
#ifndef MI8_NSTG
#define MI8_NSTG 2  // K-chunk ring stages (3 needs MI8_TAB_REP = 8 to fit the 227 KB)
#endif
#ifndef MI8_TAB_REP
#define MI8_TAB_REP 16
#endif
constexpr int NSTG = MI8_NSTG;          // K-chunk ring stages
constexpr int A_CH = P * TI * 32;       // 28 KB
constexpr int B_CH = P * TJ * 32;       // 14 KB
constexpr int STG_BYTES = A_CH + B_CH;  // 42 KB
constexpr int ELD = 68;                 // E tile row stride (doubles), = 4 (mod 16)
constexpr int NCD = 2;                  // column-data stages (sq', e_j << 20)
constexpr int CD_BYTES = TJ * 8 + TJ * 4;
constexpr int TAB = 64;
constexpr int TAB_REP = MI8_TAB_REP;
constexpr int YMIN_K = -1022 * TAB;
constexpr int KP_MAX = 448;
#ifndef MI8_BW
#define MI8_BW 2  // columns per exp batch
#endif
#ifndef MI8_TS
#define MI8_TS 4  // A slices 0 .. MI8_TS-1 of each K chunk copied to TMEM (tcgen05.cp) and used in TS
                  // mode: the 64 TMEM columns the 7 accumulator groups leave free hold two chunks x 4
                  // slices; 22 of the 28 MMAs then read only B from shared memory
#endif
#ifndef MI8_PROFILE
#define MI8_PROFILE 0  // 1: compile the profiling modes (debug bits 1 / 2 / 8; A/B builds only: they cost ~6 % in the hot loops)
#endif
#ifndef MI8_SLICEBAR
#define MI8_SLICEBAR 0  // 1: per-slice ring barriers: slice q of a stage is refilled as soon as group q (its last reader) completes
#endif
#ifndef MI8_BIGCOPY
#define MI8_BIGCOPY 0  // 1: two copies of the slices laid out so one ring stage is 2 bulk copies (A 28 KB, B 14 KB)
#endif
#ifndef MI8_TMUX
#define MI8_TMUX 0  // time-multiplex the tensor core with the FP64 phase (1), overlap them (0), or run the
                    // DMMA contraction of tile t after tile t+1's MMAs, exp still overlapped (2)
#endif

constexpr size_t OFF_E = size_t(NSTG) * STG_BYTES;
constexpr size_t OFF_VI = OFF_E + size_t(TI) * ELD * 8;
constexpr size_t OFF_VJ = OFF_VI + size_t(TI) * TR * 8;
constexpr size_t OFF_CD = OFF_VJ + size_t(TJ) * TR * 8;
constexpr size_t OFF_TAB = OFF_CD + size_t(NCD) * CD_BYTES;
constexpr size_t OFF_BARS = OFF_TAB + size_t(TAB) * TAB_REP * 8;
constexpr int NBARS = 2 * NSTG * P + 2 * NCD + 2 * NGRP + 1;
constexpr size_t SMEM = OFF_BARS + NBARS * 8 + 16;
static_assert(SMEM <= 227 * 1024, "K1T-I8 shared memory");
static_assert(NGRP * TJ + 2 * MI8_TS * 8 <= TMEM_COLS, "K1T-I8 TMEM: accumulators + TS operand buffers");

// profiling trace (debug bit 2): clock64 stamps of CTA 0, 16 per tile, first 32 tiles
constexpr int MTRACE_TILES = 32;
__device__ long long g_mtrace[MTRACE_TILES * 16];
#define MI8_TRACE(cond, tile, slot)                                                         \
    do {                                                                                    \
        if ((A.debug & 4) && blockIdx.x == 0 && (cond) && (tile) < MTRACE_TILES)            \
            g_mtrace[(tile) * 16 + (slot)] = clock64();                                     \
    } while (0)

struct MI8Args {
    const uint8_t* __restrict__ S;   // K-chunk-major slices
    const int* __restrict__ ex;      // e_i
    const int* __restrict__ ejs;     // e_j << 20
    const double* __restrict__ sqs;  // kscale |x_j|^2
    const double* __restrict__ v;    // n_pad x 16
    double* __restrict__ part;       // NS x n_pad x 16
    const int2* __restrict__ tiles;
    const double* __restrict__ tab64;
    int64_t n_pad;
    int st;
    int ks;  // kp / 32
    int debug;  // bit 2: trace; with MI8_PROFILE (results invalid): 1 no MMAs, 2 no exp arithmetic, 8 no DMMA
    double kabs;
    double a1, a2, a3, a4, a5;
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory"); }

// a * b + c with a 32 x 32 -> 64-bit signed product (mad.wide.s32)
__device__ __forceinline__ int64_t mad_wide(int32_t a, int32_t b, int64_t c) {
    int64_t d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}
// K1-I8's drain (gauss_matvec_i8.cu), with int64 partials throughout: at kp = 448 a group sum
// reaches 7 x 128^2 x 448 = 5.1e7, so 2^8 G_1 + G_2 no longer fits in int32 here.  MAGIC + V is
// the double 1.5 * 2^52 + V (|V| < 2^51); M2 = 1.5 * 2^52 (1 + 2^-24).
constexpr int64_t MAGIC = 0x4338000000000000LL;
constexpr double M2 = 6755399441055744.0 + 402653184.0;

// swizzled shared-memory indices
__device__ __forceinline__ int e_idx(int r, int c) { return r * ELD + (c ^ ((r >> 2) & 3)); }
__device__ __forceinline__ int v_idx(int r, int t) { return r * TR + (t ^ ((r & 3) << 2)); }

__global__ void __launch_bounds__(NTHR, 1) gauss_matmat_i8_kernel(const MI8Args A) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sStg = smem;
    double* sE = reinterpret_cast<double*>(smem + OFF_E);
    double* sVI = reinterpret_cast<double*>(smem + OFF_VI);
    double* sVJ = reinterpret_cast<double*>(smem + OFF_VJ);
    uint8_t* sCD = smem + OFF_CD;
    double* tab = reinterpret_cast<double*>(smem + OFF_TAB);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + OFF_BARS);
    uint64_t* s_full = bars;              // [NSTG][P] (MI8_SLICEBAR) or [NSTG]
    uint64_t* s_empty = s_full + NSTG * P;
    uint64_t* cd_full = s_empty + NSTG * P;
    uint64_t* cd_empty = cd_full + NCD;
    uint64_t* g_full = cd_empty + NCD;
    uint64_t* g_empty = g_full + NGRP;
    uint64_t* epi_done = g_empty + NGRP;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);

    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int2 tile = A.tiles[blockIdx.x];
    const int sa = tile.x, sb = tile.y;
    const bool diag = (sa == sb);
    const int nTI = A.st / TI, nTJ = A.st / TJ;
    const int64_t rowBase = int64_t(sa) * A.st;
    const int64_t colBase = int64_t(sb) * A.st;
    const int KS = A.ks;
    const int64_t g8 = A.n_pad / 8;  // 8-row groups per K chunk

    if (tid == 0) {
        for (int s = 0; s < NSTG * P; ++s) {
            tc::mbar_init(s_full + s, 1);
            tc::mbar_init(s_empty + s, 1);
        }
        for (int s = 0; s < NCD; ++s) {
            tc::mbar_init(cd_full + s, 1);
            tc::mbar_init(cd_empty + s, NEPI);
        }
        for (int g = 0; g < NGRP; ++g) {
            tc::mbar_init(g_full + g, 1);
            tc::mbar_init(g_empty + g, NEPI);
        }
        tc::mbar_init(epi_done, NEPI);
        tc::mbar_fence_init();
    }
    for (int i = tid; i < TAB * TAB_REP; i += NTHR) {  // entry j carries hi(2^(j/64)) - (j << 14) (K1-I8's table)
        const double t = A.tab64[i / TAB_REP];
        tab[i] = __hiloint2double(__double2hiint(t) - (i / TAB_REP) * (1 << 14), __double2loint(t));
    }
    if (warp == WARP_MMA) tc::tmem_alloc(tmem_slot, TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == WARP_PROD) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int bq = 0, cc = 0;  // cc: running K-chunk count (ring position)
            int uses[NSTG] = {};
            for (int it = 0; it < nTI; ++it) {
                const int64_t r0 = rowBase + int64_t(it) * TI;
                for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                    const int64_t c0 = colBase + int64_t(jt) * TJ;
                    const int cs = bq % NCD;
                    if (bq >= NCD) tc::mbar_wait_sleep(cd_empty + cs, uint32_t(((bq / NCD) - 1) & 1));
                    tc::mbar_arrive_expect_tx(cd_full + cs, uint32_t(CD_BYTES));
                    uint8_t* cd = sCD + cs * CD_BYTES;
                    tc::bulk_g2s(cd, A.sqs + c0, TJ * 8, cd_full + cs);
                    tc::bulk_g2s(cd + TJ * 8, A.ejs + c0, TJ * 4, cd_full + cs);
                    for (int ks = 0; ks < KS; ++ks, ++cc) {
                        const int s = cc % NSTG;
                        if (ks == 0) MI8_TRACE(true, bq, 12);
                        uint8_t* st = sStg + s * STG_BYTES;
                        if (MI8_SLICEBAR && !MI8_BIGCOPY) {
                            // slice q (A and B) as soon as the previous chunk in this stage released it
                            for (int q = P - 1; q >= 0; --q) {
                                uint64_t* full = s_full + s * P + q;
                                if (uses[s] > 0) tc::mbar_wait_sleep(s_empty + s * P + q, uint32_t((uses[s] - 1) & 1));
                                tc::mbar_arrive_expect_tx(full, uint32_t((TI + TJ) * 32));
                                const uint8_t* base = A.S + (int64_t(q) * KS + ks) * g8 * 256;
                                tc::bulk_g2s(st + q * (TI * 32), base + (r0 >> 3) * 256, uint32_t(TI * 32), full);
                                tc::bulk_g2s(st + A_CH + q * (TJ * 32), base + (c0 >> 3) * 256, uint32_t(TJ * 32), full);
                            }
                            ++uses[s];
                            continue;
                        }
                        if (uses[s] > 0) tc::mbar_wait_sleep(s_empty + s, uint32_t((uses[s] - 1) & 1));
                        ++uses[s];
                        tc::mbar_arrive_expect_tx(s_full + s, uint32_t(STG_BYTES));
                        if (MI8_BIGCOPY) {
                            // [ks][n_pad/128][p][128 x 32 B] and [ks][n_pad/64][p][64 x 32 B] copies
                            const uint8_t* sa = A.S + (int64_t(ks) * (A.n_pad / TI) + (r0 / TI)) * A_CH;
                            const uint8_t* sb = A.S + int64_t(KS) * A.n_pad * P * 32 +
                                                (int64_t(ks) * (A.n_pad / TJ) + (c0 / TJ)) * B_CH;
                            tc::bulk_g2s(st, sa, uint32_t(A_CH), s_full + s);
                            tc::bulk_g2s(st + A_CH, sb, uint32_t(B_CH), s_full + s);
                        } else {
                            for (int p = 0; p < P; ++p) {
                                const uint8_t* base = A.S + (int64_t(p) * KS + ks) * g8 * 256;
                                tc::bulk_g2s(st + p * (TI * 32), base + (r0 >> 3) * 256, uint32_t(TI * 32), s_full + s);
                                tc::bulk_g2s(st + A_CH + p * (TJ * 32), base + (c0 >> 3) * 256, uint32_t(TJ * 32),
                                             s_full + s);
                            }
                        }
                    }
                }
            }
        }
    } else if (warp == WARP_MMA) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = tc::idesc_i8(TI, TJ);
        int bq = 0, cc = 0;
        int uses[NSTG] = {};
        for (int it = 0; it < nTI; ++it) {
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                // time-multiplexed with the previous tile's FP64 phase (exp + DMMA)
                if (MI8_TMUX == 1 && bq > 0) tc::mbar_wait_sleep(epi_done, uint32_t((bq - 1) & 1));
                MI8_TRACE(lane == 0, bq, 8);
                for (int ks = 0; ks < KS; ++ks, ++cc) {
                    const int s = cc % NSTG;
                    constexpr bool SB = MI8_SLICEBAR && !MI8_BIGCOPY;
                    const uint32_t ph = uint32_t(uses[s] & 1);
                    if (!SB) tc::mbar_wait_sleep(s_full + s, ph);
                    ++uses[s];
                    if (ks == 0 || ks == KS / 2 || ks == KS - 1) MI8_TRACE(lane == 0, bq, ks == 0 ? 9 : (ks == KS - 1 ? 11 : 10));
                    tc::fence_after();
                    const uint32_t sbase = tc::smem_u32(sStg + s * STG_BYTES);
                    const uint64_t dA0 = tc::smem_desc(sbase, 128, 256);
                    const uint64_t dB0 = tc::smem_desc(sbase + A_CH, 128, 256);
                    const bool last = (ks == KS - 1);
                    // TS operands of this chunk into one of two TMEM buffers, free once the chunk two back
                    // completed: with a 2-stage ring the stage's own refill implies that; a deeper ring
                    // waits for that chunk's s_empty commit here (mma -> cp is not a pipelined tcgen05 pair)
                    const uint32_t abuf = tmem_base + uint32_t(NGRP * TJ) + uint32_t((cc & 1) * MI8_TS * 8);
                    if (!SB && MI8_TS > 0) {
                        if (NSTG > 2 && cc >= 2) {
                            tc::mbar_wait_sleep(s_empty + (cc - 2) % NSTG, uint32_t(((cc - 2) / NSTG) & 1));
                            tc::fence_after();
                        }
                        if (tc::elect_one())
#pragma unroll
                            for (int p = 0; p < MI8_TS; ++p)
                                tc::tmem_cp_128x256b(abuf + uint32_t(p * 8), dA0 + uint64_t((p * TI * 32) >> 4));
                        __syncwarp();
                    }
#pragma unroll
                    for (int c = NGRP - 1; c >= 0; --c) {
                        if (ks == 0 && bq > 0) {
                            tc::mbar_wait_sleep(g_empty + c, uint32_t((bq - 1) & 1));
                            tc::fence_after();
                        }
                        if (SB && c == NGRP - 1) {
                            // the first group reads every slice of the chunk: wait for each pair (p, 7 - p)
#pragma unroll
                            for (int p = 0; p <= c; ++p) {
                                if (p < 4) {
                                    tc::mbar_wait_sleep(s_full + s * P + p, ph);
                                    tc::mbar_wait_sleep(s_full + s * P + (c - p), ph);
                                    tc::fence_after();
                                }
                                if (tc::elect_one() && !(MI8_PROFILE && (A.debug & 1)))
                                    tc::mma_i8(tmem_base + uint32_t(c * TJ), dA0 + uint64_t((p * TI * 32) >> 4),
                                               dB0 + uint64_t(((c - p) * TJ * 32) >> 4), idesc,
                                               (ks == 0 && p == 0) ? 0u : 1u);
                                __syncwarp();
                            }
                            if (tc::elect_one()) {
                                if (last) tc::mma_commit(g_full + c);
                                tc::mma_commit(s_empty + s * P + c);  // group c: last reader of slice c
                            }
                            __syncwarp();
                            continue;
                        }
                        if (tc::elect_one()) {
#pragma unroll
                            for (int p = 0; p <= c; ++p) {
                                if (MI8_PROFILE && (A.debug & 1)) continue;
                                const uint64_t db = dB0 + uint64_t(((c - p) * TJ * 32) >> 4);
                                if (!SB && p < MI8_TS)
                                    tc::mma_i8_ts(tmem_base + uint32_t(c * TJ), abuf + uint32_t(p * 8), db, idesc,
                                                  (ks == 0 && p == 0) ? 0u : 1u);
                                else
                                    tc::mma_i8(tmem_base + uint32_t(c * TJ), dA0 + uint64_t((p * TI * 32) >> 4), db, idesc,
                                               (ks == 0 && p == 0) ? 0u : 1u);
                            }
                            if (last) tc::mma_commit(g_full + c);
                            if (SB) tc::mma_commit(s_empty + s * P + c);  // group c: last reader of slice c
                        }
                        __syncwarp();
                    }
                    if (!SB) {
                        if (tc::elect_one()) tc::mma_commit(s_empty + s);
                        __syncwarp();
                    }
                }
            }
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = MI8_MMA_LAST ? warp : warp - 2;  // 0..15
        const int quarter = warp & 3;  // TMEM lane quarter
        const int half = ew >> 2;      // which 16 of the 64 columns (exp phase)
        const double* tab_l = tab + (lane & (TAB_REP - 1));  // this lane's table replica
        const int etid = ew * 32 + lane;
        const int row = quarter * 32 + lane;
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(half * CPT);
        const int kabs_hi = __double2hiint(A.kabs), kabs_lo = __double2loint(A.kabs);
        const double shifter = 6755399441055744.0;  // 1.5 * 2^52
        const int g = lane >> 2, t4 = lane & 3;      // DMMA fragment coordinates
        const bool rows_role = ew < 8;              // warps 0-7: E . V_J; 8-15: E^T . V_I
        const int jb = ew - 8;                       // column role: 8-column block of the tile
        int tq = 0;
        int ntiles_cta = 0;  // tiles of this CTA (the MMA warp's order)
        for (int it2 = 0; it2 < nTI; ++it2) ntiles_cta += nTJ - (diag ? it2 * (TI / TJ) : 0);
        for (int it = 0; it < nTI; ++it) {
            const int64_t i0 = rowBase + int64_t(it) * TI;
            const int64_t gi = i0 + row;
            const double sqs_i = A.sqs[gi];
            const int nsi_hi = kabs_hi + (A.ex[gi] - 39) * (1 << 20);  // -2 x.x = -2^(e_i+e_j-39) T
            // V_I of the pass (swizzled; the previous pass's readers are past the tile barrier)
            for (int k = etid; k < TI * TR / 2; k += NEPI * 32) {
                const int r = (2 * k) / TR, t = (2 * k) % TR;
                const double2 vv = *reinterpret_cast<const double2*>(A.v + (i0 + r) * TR + t);
                *reinterpret_cast<double2*>(sVI + v_idx(r, t)) = vv;
            }
            double racc[2][2][2] = {};  // rows role: [m block][n block][pair]
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++tq) {
                const uint32_t ph = uint32_t(tq & 1);
                const int64_t j0 = colBase + int64_t(jt) * TJ;
                // prefetch: this tile's V_J (2 doubles per thread) and the column owners' running sums
                const double2 vj = *reinterpret_cast<const double2*>(A.v + j0 * TR + 2 * etid);
                double cprev[2][2] = {};
                const int64_t cidx = j0 + jb * 8 + g;  // column role: this lane's column
                if (!rows_role && it > 0) {
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) {
                        const double2 pv = *reinterpret_cast<const double2*>(
                            A.part + (int64_t(sa) * A.n_pad + cidx) * TR + nb * 8 + 2 * t4);
                        cprev[nb][0] = pv.x;
                        cprev[nb][1] = pv.y;
                    }
                }

                MI8_TRACE(etid == 0, tq, 0);
                // ---- drain the 7 groups as (6, 5), (4, 3), (2, 1), (0) (K1-I8's integer combination:
                // T = H + 2^-24 L, H = 2^24 G_0 + 2^16 G_1 + 2^8 G_2, L = 2^24 G_3 + 2^16 G_4 + 2^8 G_5 + G_6)
                // in two 8-column halves, each through all four stages: the int64 partials of one half
                // only stay live (register pressure); the groups are released after the second
                int64_t acc[CPT / 2];
                double lo[CPT / 2], T[CPT];
                auto stage = [&](int ca, int cb, int h, auto&& fn) {  // groups ca (completes first), cb = ca - 1 or none
                    if (h == 0) {
                        tc::mbar_wait_sleep(g_full + ca, ph);
                        if (cb >= 0) tc::mbar_wait_sleep(g_full + cb, ph);
                        tc::fence_after();
                    }
                    uint32_t ga[CPT / 2], gb[CPT / 2];
                    tc::tmem_ld8(taddr + uint32_t(ca * TJ + h * (CPT / 2)), ga);
                    if (cb >= 0) tc::tmem_ld8(taddr + uint32_t(cb * TJ + h * (CPT / 2)), gb);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < CPT / 2; ++k) fn(k, int32_t(ga[k]), int32_t(gb[k]));
                    if (h == 1) {
                        tc::fence_before();
                        __syncwarp();
                        if (lane == 0) {
                            tc::mbar_arrive(g_empty + ca);
                            if (cb >= 0) tc::mbar_arrive(g_empty + cb);
                        }
                    }
                };
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    stage(6, 5, h, [&](int k, int32_t g6, int32_t g5) { acc[k] = mad_wide(g5, 256, int64_t(g6)); });
                    if (h == 0) MI8_TRACE(etid == 0, tq, 1);
                    stage(4, 3, h, [&](int k, int32_t g4, int32_t g3) {
                        lo[k] = __longlong_as_double(mad_wide(g3, 1 << 24, mad_wide(g4, 65536, acc[k] + MAGIC)));
                    });
                    stage(2, 1, h, [&](int k, int32_t g2, int32_t g1) { acc[k] = mad_wide(g1, 256, int64_t(g2)); });
                    stage(0, -1, h, [&](int k, int32_t g0, int32_t) {
                        T[h * (CPT / 2) + k] = fma(lo[k], 0x1p-24, __longlong_as_double(mad_wide(g0, 1 << 24, acc[k] * 256 + MAGIC)) - M2);
                    });
                }

                MI8_TRACE(etid == 0, tq, 2);
                // ---- exp phase: E tile (masked on the diagonal blocks) into shared memory
                const int cs = tq % NCD;
                tc::mbar_wait(cd_full + cs, uint32_t((tq / NCD) & 1));
                const double* cd_sq = reinterpret_cast<const double*>(sCD + cs * CD_BYTES);
                const int* cd_e = reinterpret_cast<const int*>(sCD + cs * CD_BYTES + TJ * 8);
                const int colOff = half * CPT;
                const bool masked = diag && jt < (it + 1) * (TI / TJ);
                const int mask_row = row - (jt - it * (TI / TJ)) * TJ;
                if (MI8_PROFILE && (A.debug & 2)) {  // profiling: no exp arithmetic (results invalid)
#pragma unroll
                    for (int k = 0; k < CPT; ++k) sE[e_idx(row, colOff + k)] = T[k];
                } else
#pragma unroll
                for (int k0 = 0; k0 < CPT; k0 += MI8_BW) {
                    double y[MI8_BW], t2[MI8_BW], f[MI8_BW], q[MI8_BW];
                    int kk[MI8_BW];
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) {
                        const int cl = colOff + k0 + b;
                        const double nscale = __hiloint2double(nsi_hi + cd_e[cl], kabs_lo);
                        y[b] = fma(T[k0 + b], nscale, sqs_i + cd_sq[cl]);
                        y[b] = __hiloint2double(min(__double2hiint(y[b]), 0), __double2loint(y[b]));
                    }
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) t2[b] = y[b] + shifter;
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) f[b] = y[b] - (t2[b] - shifter);
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) q[b] = fma(f[b], A.a5, A.a4);
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) q[b] = fma(q[b], f[b], A.a3);
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) q[b] = fma(q[b], f[b], A.a2);
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) q[b] = fma(q[b], f[b], A.a1);
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) {
                        q[b] = q[b] * f[b];
                        kk[b] = max(__double2loint(t2[b]), YMIN_K);
                    }
#pragma unroll
                    for (int b = 0; b < MI8_BW; ++b) {
                        // K1-I8's lookup: byte offset (k << 7) & 0x1F80 in this lane's replica, k << 14 on the high word
                        const double tj = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab_l) +
                                                                           ((kk[b] * (TAB_REP * 8)) & ((TAB - 1) * TAB_REP * 8)));
                        const double ts = __hiloint2double(__double2hiint(tj) + kk[b] * (1 << 14), __double2loint(tj));
                        double e = fma(ts, q[b], ts);
                        const int cl = colOff + k0 + b;
                        if (masked) e = (cl > mask_row) ? e : 0.0;
                        sE[e_idx(row, cl)] = e;
                    }
                }
                {
                    const int r = (2 * etid) / TR, t = (2 * etid) % TR;
                    *reinterpret_cast<double2*>(sVJ + v_idx(r, t)) = vj;
                }
                __syncwarp();
                MI8_TRACE(etid == 0, tq, 3);
                if (lane == 0) tc::mbar_arrive(cd_empty + cs);
                epi_bar();  // E and V_J complete
                MI8_TRACE(etid == 0, tq, 4);

                // ---- FP64 tensor phase
                if (MI8_TMUX == 2 && tq + 1 < ntiles_cta) tc::mbar_wait(g_full + 0, uint32_t((tq + 1) & 1));
                if (rows_role) {
                    // O_I rows 16 ew .. 16 ew + 15 (+)= E . V_J
#pragma unroll 4
                    for (int kk = 0; kk < ((MI8_PROFILE && (A.debug & 8)) ? 0 : TJ / 4); ++kk) {
                        const int k0 = kk * 4;
                        double af[2], bf[2];
#pragma unroll
                        for (int mb = 0; mb < 2; ++mb) af[mb] = sE[e_idx(ew * 16 + mb * 8 + g, k0 + t4)];
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) bf[nb] = sVJ[v_idx(k0 + t4, nb * 8 + g)];
#pragma unroll
                        for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                            for (int nb = 0; nb < 2; ++nb)
                                dmma884(racc[mb][nb][0], racc[mb][nb][1], af[mb], bf[nb]);
                    }
                    __syncwarp();
                    MI8_TRACE(etid == 0, tq, 5);
                    if (lane == 0) tc::mbar_arrive(epi_done);
                } else {
                    // O_J (columns jb*8 .. +7) = E^T . V_I over the tile's 128 rows
                    double cacc[2][2] = {};
#pragma unroll 4
                    for (int kk = 0; kk < ((MI8_PROFILE && (A.debug & 8)) ? 0 : TI / 4); ++kk) {
                        const int r0 = kk * 4;
                        const double a = sE[e_idx(r0 + t4, jb * 8 + g)];
                        double bf[2];
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) bf[nb] = sVI[v_idx(r0 + t4, nb * 8 + g)];
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) dmma884(cacc[nb][0], cacc[nb][1], a, bf[nb]);
                    }
                    __syncwarp();
                    MI8_TRACE(etid == 8 * 32, tq, 6);
                    if (lane == 0) tc::mbar_arrive(epi_done);
#pragma unroll
                    for (int nb = 0; nb < 2; ++nb) {
                        double2 o;
                        o.x = cprev[nb][0] + cacc[nb][0];
                        o.y = cprev[nb][1] + cacc[nb][1];
                        *reinterpret_cast<double2*>(A.part + (int64_t(sa) * A.n_pad + cidx) * TR + nb * 8 + 2 * t4) = o;
                    }
                }
                epi_bar();  // E / V_J readers done before the next tile overwrites them
                MI8_TRACE(etid == 0, tq, 7);
            }
            // ---- rows of this pass
            if (!diag) {
                if (rows_role) {
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) {
                            const int64_t r = i0 + ew * 16 + mb * 8 + g;
                            double2 o;
                            o.x = racc[mb][nb][0];
                            o.y = racc[mb][nb][1];
                            *reinterpret_cast<double2*>(A.part + (int64_t(sb) * A.n_pad + r) * TR + nb * 8 + 2 * t4) = o;
                        }
                }
            } else {
                // same slot as the columns: stage the rows in shared memory (the V_I tile: its last
                // readers are past the tile barrier, and it is reloaded by the next pass; the E
                // region may already hold the next tile's K chunks), and the column owner of each
                // index adds them (one writer per element, program order)
                double* rowbuf = sVI;  // [128][16], plain layout
                if (rows_role) {
#pragma unroll
                    for (int mb = 0; mb < 2; ++mb)
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) {
                            const int r = ew * 16 + mb * 8 + g;
                            rowbuf[r * TR + nb * 8 + 2 * t4] = racc[mb][nb][0];
                            rowbuf[r * TR + nb * 8 + 2 * t4 + 1] = racc[mb][nb][1];
                        }
                }
                epi_bar();
                if (!rows_role) {
#pragma unroll
                    for (int h = 0; h < TI / TJ; ++h) {
                        const int r = h * TJ + jb * 8 + g;
#pragma unroll
                        for (int nb = 0; nb < 2; ++nb) {
                            double2* dst = reinterpret_cast<double2*>(A.part + (int64_t(sa) * A.n_pad + i0 + r) * TR +
                                                                      nb * 8 + 2 * t4);
                            double2 o = *dst;
                            o.x += rowbuf[r * TR + nb * 8 + 2 * t4];
                            o.y += rowbuf[r * TR + nb * 8 + 2 * t4 + 1];
                            *dst = o;
                        }
                    }
                }
                epi_bar();  // rowbuf (V_I) is reloaded by the next pass
            }
        }
    }

    tc::fence_before();
    __syncthreads();
    if (warp == WARP_MMA) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

// ---- operand preparation: the K-chunk-major slices [p][kp/32][n_pad/8][2][8][16]
__global__ void row_exponent_s_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad,
                                      int* __restrict__ ex, int* __restrict__ ejs) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_pad; i += warps) {
        double m = 0.0;
        if (i < n)
            for (int64_t k = lane; k < d; k += 32) m = fmax(m, fabs(X[i * d + k]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane == 0) {
            // |x_ik| 2^-e <= 0.498: the range of 7 balanced 8-bit digits (as K1-I8)
            int e = m > 0.0 ? ilogb(m) + 2 : 0;
            if (m > 0.0 && scalbn(m, -e) > 0.498) ++e;
            ex[i] = e;
            ejs[i] = e * (1 << 20);
        }
    }
}

__global__ void slice_s_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, int kp,
                               const int* __restrict__ ex, uint8_t* __restrict__ S) {
    const int64_t total = n_pad * kp;
    const int ks_n = kp / 32;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = idx / kp;
        const int k = int(idx % kp);
        const double x = (row < n && k < d) ? X[row * d + k] : 0.0;
        int a[P];
        tc::balanced_digits8(x, ex[row], a);  // as K1-I8
        const int64_t off =
            (int64_t(k >> 5) * (n_pad >> 3) + (row >> 3)) * 256 + ((k >> 4) & 1) * 128 + (row & 7) * 16 + (k & 15);
        // MI8_BIGCOPY: A copy [ks][n_pad/128][p][16][2][8][16], B copy [ks][n_pad/64][p][8][2][8][16]
        const int64_t in_a = (int64_t(k >> 5) * (n_pad / TI) + row / TI) * (P * TI * 32) + ((row % TI) >> 3) * 256 +
                             ((k >> 4) & 1) * 128 + (row & 7) * 16 + (k & 15);
        const int64_t in_b = int64_t(ks_n) * n_pad * P * 32 +
                             (int64_t(k >> 5) * (n_pad / TJ) + row / TJ) * (P * TJ * 32) + ((row % TJ) >> 3) * 256 +
                             ((k >> 4) & 1) * 128 + (row & 7) * 16 + (k & 15);
#pragma unroll
        for (int p = 0; p < P; ++p) {
            if (MI8_BIGCOPY) {
                S[in_a + p * (TI * 32)] = uint8_t(int8_t(a[p]));
                S[in_b + p * (TJ * 32)] = uint8_t(int8_t(a[p]));
            } else {
                S[int64_t(p) * ks_n * n_pad * 32 + off] = uint8_t(int8_t(a[p]));
            }
        }
    }
}

__global__ void scaled_sq_s_kernel(const double* __restrict__ L, int64_t n_pad, int dp, int d, double kscale,
                                   double* __restrict__ sqs) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad; i += int64_t(gridDim.x) * blockDim.x)
        sqs[i] = kscale * L[i * dp + d];
}

}  // namespace

void i8s_read_trace(long long* out, int count) {
    count = std::min(count, MTRACE_TILES * 16);
    KRR_CUDA(cudaMemcpyFromSymbol(out, g_mtrace, sizeof(long long) * size_t(count)));
}

int i8s_kp(int64_t d) { return int((d + 31) / 32 * 32); }

size_t i8s_slice_bytes(int64_t n_pad, int64_t d) { return size_t(MI8_BIGCOPY ? 16 : 8) * size_t(n_pad) * size_t(i8s_kp(d)); }

bool i8s_supported(int64_t d, int st) { return i8s_kp(d) <= KP_MAX && st % TI == 0 && st >= TI; }

bool i8s_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp, double kscale,
                        uint8_t* S, int* ex, int* ejs, double* sqs, cudaStream_t stream) {
    const int kp = i8s_kp(d);
    const unsigned wblocks = unsigned(std::min<int64_t>((n_pad + 7) / 8, 148 * 16));
    row_exponent_s_kernel<<<wblocks, 256, 0, stream>>>(X, n, d, n_pad, ex, ejs);
    KRR_LAUNCH_CHECK();
    const int64_t total = n_pad * kp;
    slice_s_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, stream>>>(X, n, d, n_pad, kp,
                                                                                                   ex, S);
    KRR_LAUNCH_CHECK();
    scaled_sq_s_kernel<<<unsigned(std::min<int64_t>((n_pad + 255) / 256, 148 * 8)), 256, 0, stream>>>(L, n_pad, dp,
                                                                                                     int(d), kscale, sqs);
    KRR_LAUNCH_CHECK();
    // the exponent range K1-I8 requires (gauss_matvec_i8.cu, i8_prepare_launch)
    std::vector<int> h(static_cast<size_t>(n_pad));
    KRR_CUDA(cudaMemcpyAsync(h.data(), ex, sizeof(int) * size_t(n_pad), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    int lo = 0, hi = 0;
    for (int e : h) {
        lo = std::min(lo, e);
        hi = std::max(hi, e);
    }
    const int ek = std::ilogb(-kscale);
    const double ymax = -kscale * 4.0 * double(d) * std::ldexp(1.0, 2 * hi);
    return ek + 2 * lo - 39 > -1000 && ek + 2 * hi - 39 < 1000 && ymax < std::ldexp(1.0, 50);
}

void gauss_matmat_i8_launch(const GaussMatvecPlan& p, const uint8_t* S, const int* ex, const int* ejs,
                            const double* sqs, const double* v, double* part, int kp, cudaStream_t stream,
                            int debug) {
    if (p.num_tiles == 0) return;
    if (kp % 32 != 0 || kp > KP_MAX) fail(KRR_ERR_INVALID_ARGUMENT, "K1T-I8: kp must be a multiple of 32, <= 448");
    MI8Args a;
    a.S = S;
    a.ex = ex;
    a.ejs = ejs;
    a.sqs = sqs;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.tab64 = p.exp_tab;
    a.n_pad = p.n_pad;
    a.st = p.st;
    a.ks = kp / 32;
    a.debug = debug;
    const long double ln2 = 0.693147180559945309417232121458176568L;
    const long double l = ln2 / TAB;
    a.kabs = -p.ec.kscale;
    long double term = 1.0L;
    double c[6];
    for (int m = 1; m <= 5; ++m) {
        term = term * l / (long double)m;
        c[m] = double(term);
    }
    a.a1 = c[1];
    a.a2 = c[2];
    a.a3 = c[3];
    a.a4 = c[4];
    a.a5 = c[5];
    KRR_CUDA(cudaFuncSetAttribute(gauss_matmat_i8_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM)));
    gauss_matmat_i8_kernel<<<unsigned(p.num_tiles), NTHR, SMEM, stream>>>(a);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
