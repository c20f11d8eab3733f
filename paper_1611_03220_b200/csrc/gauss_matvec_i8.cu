// K1-I8 — the fused symmetric Gaussian mat-vec with the dot products on the
// 5th-generation tensor cores (tcgen05.mma kind::i8, TMEM accumulators), exact to
// fp64 level via an Ozaki-style slice decomposition.
//
// Why: the d-long dot product is ~90 % of K1's FP64 work, and integer MMA accumulates
// exactly.  Measured on B200 (tools/mma_rate.py, profiles/): the FP64 pipe, DMMA and the
// INT8 tensor path share one execution resource — DFMA / DADD drop from 61 to 16
// lane-ops / clk / SM while tcgen05 INT8 MMAs run — so K1-I8's cost is MMA time + FP64
// time, and the design minimises both: one MMA per 128 x 64 x 32-byte block (~50 clk),
// and 15 FP64 operations per pair in the epilogue (vs 92 + 12 per pair for the DMMA K1
// at d = 90).
//
// Decomposition (per row i, e_i = ilogb(max_k |x_ik|) + 2, u_i = x_i 2^-e_i in (-1/2, 1/2)):
//     U_i = rint(u_i 2^56) (int64),  u_i = sum_{p<7} A_i^(p) 2^(-8(p+1)) + r_i,  A^(p) in [-128, 127],  |r_i| <= 2^-57
// (the balanced bytes of U_i, tc_i8.cuh:balanced_digits8).  Then
//     x_i . x_j = 2^(e_i + e_j - 16) sum_c 2^(-8c) G_c,   G_c = sum_{p+q=c} A_i^(p) . A_j^(q)
// keeping c = p + q <= 6: 28 int8 products accumulated exactly in int32 into 7 TMEM groups (the
// dropped c >= 7 terms are zero-mean, |A| <= 128: the dot product stays at fp64 level, as with the
// round-1 scheme of 8 truncated 7-bit digits and 36 products).  The drain fuses the groups in
// integer arithmetic, straight into the mantissa field of 1.5 * 2^52 (mad.wide), and converts once:
//     Hi = 2^24 G_0 + 2^16 G_1 + 2^8 G_2 + G_3,  Lo = 2^16 G_4 + 2^8 G_5 + G_6   (int64, exact)
//     T = Hi + 2^-24 Lo  (one DADD + one DFMA, one rounding)  =  2^40 u_i . u_j
// so -2 x_i.x_j = -2^(e_i + e_j - 39) T.  The exp argument is formed directly in units of 1/64
// octave,
//     y = kscale d2 = sq'_i + sq'_j + |kscale| 2^(e_i - 39) 2^(e_j) T,   sq' = kscale |x|^2,
// with kscale = -scale 64 / ln2 (the per-column power of two is an integer add on the high
// word), and e = 2^(k/64) (1 + q(f)), k = round(y), f = y - k, from the K1 64-entry table
// (replicated 16x in shared memory so a warp's lookups are bank-conflict free) and a
// degree-5 polynomial.  Dot-product error <= ~2^-52 * d * 2^(e_i + e_j), the order of an fp64 dot product's own bound.
//
// Structure (one CTA per symmetric super-tile, 10 warps, tiles of M = 128 rows x N = 64
// columns):
//   warp 0     producer: 1-D bulk async copies (TMA engine) of the I tile (128 rows x 8
//              slices, resident for a pass), a ring of J tiles (64 rows x 7 slices) and a
//              ring of per-column data (sq', v, e_j << 20);
//   warp 1     MMA issuer: one thread issues the 28 x (kp/32) tcgen05.mma of a tile group by
//              group, c = 6 down to 0, each group into its own 64 TMEM columns (7 x 64 = 448 of
//              the 512 allocated), committing one mbarrier per group;
//   warps 2-9  epilogue: each thread owns one row (its TMEM lane) and 32 of the 64 columns.
//              It drains the groups in completion order (tcgen05.ld) and releases each pair
//              at once, so the next tile's MMAs start while this tile is still converting.
//              Row sums stay in registers; every e v_i goes straight to a per-warp
//              shared-memory transpose (one sync per tile), then each lane sums one column
//              and the four lane quarters combine in fixed order.
// The J-tile ring has one stage at kp = 96: the next tile's load overlaps this tile's FP64
// epilogue, which cannot overlap the MMAs anyway (shared execution resource, above).  Slots in `part` follow exactly the K1 rules
// (gauss_matvec.cu) — one writer per (slot, index) — so the finish kernel is shared; column
// sums accumulate in the CTA's own slot in global memory (one owner thread per column,
// program order).  Everything is deterministic.
// Operand layout in global memory: slice p, 8-row group, 16-byte K chunk
// ([p][n_pad/8][kp/16][8][16]), so any 8-aligned row range is one contiguous block that
// is directly the canonical no-swizzle K-major UMMA layout (LBO = 128 B, SBO = 8 kp B).
#include <cmath>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "gauss_exp.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int P = 7;      // slices (balanced 8-bit digits)
constexpr int NGRP = 7;   // groups c = p + q in [0, 6]
constexpr int TI = 128;   // I tile rows (MMA M)
constexpr int TJ = 64;    // J tile columns (MMA N)
constexpr int NCD = 3;    // column-data stages
constexpr int NEPI = 16;  // epilogue warps (4 per TMEM lane quarter)
constexpr int CPT = 16;   // columns per epilogue thread (one tcgen05.ld x16 per group)
constexpr int NTHR = 32 * (2 + NEPI);
#ifndef I8_PROFILE
#define I8_PROFILE 0  // 1: compile in the profiling modes (debug bits 1, 2, 16, 32; the trace is always there);
                      // build them with tools/build_variant.py ... -DI8_PROFILE=1 (the lean build is 1-2 % faster)
#endif
#ifndef I8_TS
#define I8_TS 1  // A slices 0 .. nts-1 of the resident I tile copied to the 64 TMEM columns the 7
                 // accumulator groups leave free (tcgen05.cp, once per pass) and used in TS mode
#endif
#ifndef I8_REUSE
#define I8_REUSE 1  // 1: 5 accumulator slots (groups 6..2; groups 1 / 0 reuse the slots of 6 / 5 once the
                    // epilogue has drained those), so all 7 A slices fit in TMEM (TS mode for every MMA):
                    // +6 % (the MMA phase is no longer bound by shared-memory operand reads), bitwise unchanged
#endif
#ifndef I8_LATE_DRAIN
#define I8_LATE_DRAIN 0  // 1: drain only after the tile's last group (no TMEM loads while the MMAs run)
#endif
#ifndef I8_MMA_LAST
#define I8_MMA_LAST 1  // control warps last (epilogue 0-15, producer 16, MMA 17): the issue arbiter
                       // prefers high warp ids, so the MMA warp is not starved by the epilogue on its SMSP
#endif
constexpr int WARP_PROD = I8_MMA_LAST ? NEPI : 0, WARP_MMA = I8_MMA_LAST ? NEPI + 1 : 1;
static_assert(!(I8_REUSE && I8_LATE_DRAIN), "groups 1 / 0 wait for the drain of groups 6 / 5");
// TMEM column slot of accumulator group c
constexpr int NSLOT = I8_REUSE ? 5 : 7;
__host__ __device__ constexpr int gslot(int c) { return I8_REUSE ? (c >= 2 ? c - 2 : c + 3) : c; }
#ifndef I8_BW
#define I8_BW 8      // columns per exp batch: with the int64 tail, 4 beat 2 by 2.5 %; with all A slices in TMEM and
                     // the lean build, 8 beats 4 by 1-2 % (4 row-sum chains either way: bitwise the same K v)
#endif
#ifndef I8_EARLY_DONE
#define I8_EARLY_DONE 1  // arrive on epi_done after the exp element loop (1) or after the column sums (0).  With 4-column
                         // batches and the int64 tail, releasing the tensor core before the column-sum transposes is
                         // 2.5 % faster again (it was 3 % slower with 2-column batches); releasing it inside the
                         // element loop (after 8 or 12 of the 16 columns) is 17 % slower: FP64 under the MMAs
#endif
constexpr uint32_t TMEM_COLS = 512;
constexpr int KP_MAX = 96;
constexpr int SCR_LD = 33;  // transpose scratch row stride (doubles): conflict-free both ways
constexpr int CD_BYTES = TJ * 8 * 2 + TJ * 4;  // sq', v, e_j << 20
constexpr int TAB = 64;    // 2^(j/64), replicated per lane pair: conflict-free lookups
constexpr int TAB_REP = 16;
constexpr int YMIN_K = -1022 * TAB;  // 2^(k/64) stays normal

__device__ double g_tab64[TAB];
// profiling trace (i8_debug bit 2): clock64 stamps of CTA 0, 16 per tile, first 64 tiles
constexpr int TRACE_TILES = 64;
__device__ long long g_trace[TRACE_TILES * 16];
#define I8_TRACE(cond, tile, slot)                                                          \
    do {                                                                                    \
        if ((A.debug & 4) && blockIdx.x == 0 && (cond) && (tile) < TRACE_TILES)             \
            g_trace[(tile) * 16 + (slot)] = clock64();                                      \
    } while (0)

template <int KPT>
struct Cfg {
    static constexpr int NSTB = KPT >= 96 ? 1 : (KPT >= 64 ? 2 : 3);  // J-tile stages
    static constexpr size_t A_BYTES = size_t(P) * TI * KPT;
    static constexpr size_t B_BYTES = size_t(P) * TJ * KPT;
    static constexpr size_t OFF_B = A_BYTES;
    static constexpr size_t OFF_CD = OFF_B + NSTB * B_BYTES;
    static constexpr size_t OFF_SCR = OFF_CD + NCD * CD_BYTES;
    static constexpr size_t OFF_COLSCR = OFF_SCR + size_t(NEPI) * CPT * SCR_LD * 8;
    static constexpr size_t OFF_TAB = OFF_COLSCR + 2 * 4 * TJ * 8;
    static constexpr size_t OFF_BARS = OFF_TAB + TAB * TAB_REP * 8;
    static constexpr int NBARS = 2 + 2 * NSTB + 2 * NCD + 2 * NGRP + 1;
    static constexpr size_t SMEM = OFF_BARS + NBARS * 8 + 16;
};

struct I8Consts {
    double kabs;                // |kscale| = scale 64 / ln2 (polynomial kernel: gamma)
    double a1, a2, a3, a4, a5;  // (ln2/64)^m / m!      (polynomial kernel: a1 = offset c)
    int degree;                 // polynomial kernel only
    int pad_;
};

struct I8Args {
    const uint8_t* __restrict__ S;
    const int* __restrict__ ex;      // e_i
    const int* __restrict__ ejs;     // e_j << 20
    const double* __restrict__ sqs;  // kscale |x_j|^2
    const double* __restrict__ v;
    double* __restrict__ part;
    const int2* __restrict__ tiles;
    int64_t n_pad;
    int st;
    int debug;  // profiling only: bit 0 skips the MMAs, bit 1 the exp phase (results invalid),
                // bit 2 records a clock64 trace of CTA 0 (i8_read_trace), bit 4 drops the exp
                // polynomial (4 FP64 ops / pair fewer; results invalid); bit 5 = overlap mode
                // (valid results: a tile's MMAs may run during the previous tile's exp phase)
    I8Consts ec;
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory"); }

// a * b + c with a 32 x 32 -> 64-bit signed product (mad.wide.s32)
__device__ __forceinline__ int64_t mad_wide(int32_t a, int32_t b, int64_t c) {
    int64_t d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}
// the bits of 1.5 * 2^52: MAGIC + V is the double 1.5 * 2^52 + V for |V| < 2^51
constexpr int64_t MAGIC = 0x4338000000000000LL;
// 1.5 * 2^52 (1 + 2^-24): (1.5 2^52 + Hi) + (1.5 2^52 + Lo) 2^-24 - M2 = Hi + 2^-24 Lo, exact integers
constexpr double M2 = 6755399441055744.0 + 402653184.0;

template <bool MASK, bool CHEAP = false, bool POLY = false>
__device__ __forceinline__ void exp_phase(const double (&T)[CPT], const I8Consts& ec, const double* __restrict__ tab,
                                          const double* __restrict__ cd_sq, const double* __restrict__ cd_v,
                                          const int* __restrict__ cd_e, double* __restrict__ scr,
                                          double* __restrict__ colscr_q, long long* __restrict__ tr,
                                          int nsi_hi, int nsi_lo, double sqs_i,
                                          double v_i, double& rowacc, int lane, int colOff, int mask_row,
                                          uint64_t* fp64_done) {
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52
    double racc[4] = {0.0, 0.0, 0.0, 0.0};
    // four columns at a time, each step applied across the batch: independent chains
    // side by side for the scheduler (the per-pair chain is ~16 dependent FP64 ops)
    constexpr int BW = I8_BW;
    auto tval = [&](int k) { return T[k]; };
#pragma unroll
    for (int k0 = 0; k0 < CPT; k0 += BW) {
        double y[BW], t2[BW], f[BW], q[BW], e[BW];
        int kk[BW];
        if constexpr (POLY) {
            // polynomial kernel: p = gamma x_i.x_j + c = fma(T, gamma 2^(e_i+e_j-35), c),
            // then ipow(p, q) as r = p, r *= p (kernels.cpp:10-14), degree-outer across the batch
#pragma unroll
            for (int b = 0; b < BW; ++b) {
                const int cl = colOff + k0 + b;
                const double nscale = __hiloint2double(nsi_hi + cd_e[cl], nsi_lo);
                y[b] = fma(tval(k0 + b), nscale, ec.a1);
                e[b] = y[b];
            }
            for (int r = 1; r < ec.degree; ++r)
#pragma unroll
                for (int b = 0; b < BW; ++b) e[b] = __dmul_rn(e[b], y[b]);
#pragma unroll
            for (int b = 0; b < BW; ++b) {
                if constexpr (MASK) e[b] = (colOff + k0 + b > mask_row) ? e[b] : 0.0;
                racc[b & 3] = fma(e[b], cd_v[colOff + k0 + b], racc[b & 3]);
                scr[(k0 + b) * SCR_LD + lane] = e[b] * v_i;
            }
            continue;
        }
#pragma unroll
        for (int b = 0; b < BW; ++b) {
            const int cl = colOff + k0 + b;
            const double nscale = __hiloint2double(nsi_hi + cd_e[cl], nsi_lo);
            y[b] = fma(tval(k0 + b), nscale, sqs_i + cd_sq[cl]);
            // y <= 0 (d2 >= 0): y > 0 (rounding, near-duplicate rows) has a non-negative high
            // word; clamping it to 0 leaves a positive denormal, whose exp is 1 exactly.
            y[b] = __hiloint2double(min(__double2hiint(y[b]), 0), __double2loint(y[b]));
        }
#pragma unroll
        for (int b = 0; b < BW; ++b) t2[b] = y[b] + shifter;
#pragma unroll
        for (int b = 0; b < BW; ++b) f[b] = y[b] - (t2[b] - shifter);
        if constexpr (CHEAP) {  // profiling only (i8_debug 16): 4 fewer FP64 ops, wrong values
#pragma unroll
            for (int b = 0; b < BW; ++b) q[b] = ec.a1;
        } else {
#pragma unroll
            for (int b = 0; b < BW; ++b) q[b] = fma(f[b], ec.a5, ec.a4);
#pragma unroll
            for (int b = 0; b < BW; ++b) q[b] = fma(q[b], f[b], ec.a3);
#pragma unroll
            for (int b = 0; b < BW; ++b) q[b] = fma(q[b], f[b], ec.a2);
#pragma unroll
            for (int b = 0; b < BW; ++b) q[b] = fma(q[b], f[b], ec.a1);
        }
#pragma unroll
        for (int b = 0; b < BW; ++b) {
            q[b] = q[b] * f[b];
            // k >= -1022 * 64 keeps 2^(k/64) normal (e >= ~2^-1022 instead of underflowing)
            kk[b] = max(__double2loint(t2[b]), YMIN_K);
        }
#pragma unroll
        for (int b = 0; b < BW; ++b) {
            // 2^(k/64) = 2^(k >> 6) 2^((k & 63)/64): entry j = k & 63 of this lane's replica is at byte offset
            // (k << 7) & 0x1F80 and carries hi(2^(j/64)) - (j << 14), so adding k << 14 = ((k >> 6) << 20) +
            // (j << 14) to its high word applies the power of two (two integer ops per pair fewer: +1 %)
            const double tj = *reinterpret_cast<const double*>(reinterpret_cast<const char*>(tab) + ((kk[b] << 7) & 0x1F80));
            const double ts = __hiloint2double(__double2hiint(tj) + kk[b] * (1 << 14), __double2loint(tj));
            e[b] = fma(ts, q[b], ts);
            if constexpr (MASK) e[b] = (colOff + k0 + b > mask_row) ? e[b] : 0.0;
        }
#pragma unroll
        for (int b = 0; b < BW; ++b) {
            racc[b & 3] = fma(e[b], cd_v[colOff + k0 + b], racc[b & 3]);
            scr[(k0 + b) * SCR_LD + lane] = e[b] * v_i;  // column k, row `lane`
        }
    }
    if (tr) tr[13] = clock64();  // profiling trace: element loop done
    rowacc += (racc[0] + racc[1]) + (racc[2] + racc[3]);
    // The FP64-heavy part of the tile is over: release the tensor core now, so the next tile's
    // first MMA groups overlap the column-sum transposes below (shared-memory traffic and one
    // DADD per pair) instead of waiting for them.
    if (fp64_done) {
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(fp64_done);
    }
    // column sums over the warp's 32 rows: lane L sums column L % CPT over rows
    // (L / CPT) * RPL .. + RPL in 4 chains, then a butterfly over the row blocks (fixed order)
    __syncwarp();
    constexpr int RPL = 32 * CPT / 32;  // rows per lane
    const double* src = scr + (lane % CPT) * SCR_LD + (lane / CPT) * RPL;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int r = 0; r < RPL; r += 4) {
        a0 += src[r];
        a1 += src[r + 1];
        a2 += src[r + 2];
        a3 += src[r + 3];
    }
    double acc = (a0 + a1) + (a2 + a3);
#pragma unroll
    for (int o = CPT; o < 32; o <<= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (tr) tr[14] = clock64();  // column sums done
    if (lane < CPT) colscr_q[colOff + lane] = acc;
    __syncwarp();
}

template <int KPT, bool POLY>
__global__ void __launch_bounds__(NTHR, 1) gauss_matvec_i8_kernel(const I8Args A) {
    using C = Cfg<KPT>;
    constexpr int kp = KPT;
    constexpr int NSTB = C::NSTB;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::OFF_B;
    uint8_t* sCD = smem + C::OFF_CD;
    double* scr_all = reinterpret_cast<double*>(smem + C::OFF_SCR);
    double* colscr = reinterpret_cast<double*>(smem + C::OFF_COLSCR);  // [2][4 quarters][64]
    double* rowbuf = scr_all;  // [NEPI/4 parts][128], only at pass ends (scratch idle)
    double* tab = reinterpret_cast<double*>(smem + C::OFF_TAB);
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BARS);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 1;
    uint64_t* b_full = bars + 2;
    uint64_t* b_empty = b_full + NSTB;
    uint64_t* cd_full = b_empty + NSTB;
    uint64_t* cd_empty = cd_full + NCD;
    uint64_t* g_full = cd_empty + NCD;
    uint64_t* g_empty = g_full + NGRP;
    uint64_t* epi_done = g_empty + NGRP;  // the exp phase of a tile is over (MMA time-multiplexing)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(epi_done + 1);

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
        for (int s = 0; s < NSTB; ++s) {
            tc::mbar_init(b_full + s, 1);
            tc::mbar_init(b_empty + s, 1);
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
    for (int i = tid; i < TAB * TAB_REP; i += NTHR) {
        const double t = g_tab64[i / TAB_REP];
        tab[i] = __hiloint2double(__double2hiint(t) - (i / TAB_REP) * (1 << 14), __double2loint(t));  // see exp_phase
    }
    if (warp == WARP_MMA) tc::tmem_alloc(tmem_slot, TMEM_COLS);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == WARP_PROD) {
        // ------------------------------------------------------------ producer
        if (lane == 0) {
            int bq = 0;
            for (int it = 0; it < nTI; ++it) {
                if (it > 0) tc::mbar_wait_sleep(a_empty, uint32_t((it - 1) & 1));
                tc::mbar_arrive_expect_tx(a_full, uint32_t(C::A_BYTES));
                const int64_t r0 = rowBase + int64_t(it) * TI;
                for (int p = 0; p < P; ++p)
                    tc::bulk_g2s(sA + p * TI * kp, A.S + int64_t(p) * A.n_pad * kp + r0 * kp, uint32_t(TI * kp), a_full);
                for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                    const int s = bq % NSTB;
                    if (bq >= NSTB) tc::mbar_wait_sleep(b_empty + s, uint32_t(((bq / NSTB) - 1) & 1));
                    tc::mbar_arrive_expect_tx(b_full + s, uint32_t(C::B_BYTES));
                    const int64_t c0 = colBase + int64_t(jt) * TJ;
                    for (int q = 0; q < P; ++q)
                        tc::bulk_g2s(sB + s * C::B_BYTES + q * TJ * kp, A.S + int64_t(q) * A.n_pad * kp + c0 * kp,
                                     uint32_t(TJ * kp), b_full + s);
                    const int cs = bq % NCD;
                    if (bq >= NCD) tc::mbar_wait_sleep(cd_empty + cs, uint32_t(((bq / NCD) - 1) & 1));
                    tc::mbar_arrive_expect_tx(cd_full + cs, uint32_t(CD_BYTES));
                    uint8_t* cd = sCD + cs * CD_BYTES;
                    tc::bulk_g2s(cd, A.sqs + c0, TJ * 8, cd_full + cs);
                    tc::bulk_g2s(cd + TJ * 8, A.v + c0, TJ * 8, cd_full + cs);
                    tc::bulk_g2s(cd + TJ * 16, A.ejs + c0, TJ * 4, cd_full + cs);
                }
            }
        }
    } else if (warp == WARP_MMA) {
        // ------------------------------------------------------------ MMA issuer
        // The whole warp runs the (warp-uniform) schedule and waits, so the descriptors stay in
        // uniform registers; one elected lane issues each group's MMAs and their commits.  (A
        // single-thread `if (lane == 0)` region made ptxas wrap every tcgen05.mma in an
        // ELECT / R2UR waterfall loop of ~10 dependent instructions.)
        const uint32_t idesc = tc::idesc_i8(TI, TJ);
        const uint32_t aBase = tc::smem_u32(sA);
        int bq = 0;
        // TS operands: A slices p < NTS (kp / 4 TMEM columns each) after the accumulator slots
        constexpr int COLS_A = kp / 4;
        constexpr int NTS = I8_TS ? ((TMEM_COLS - NSLOT * TJ) / COLS_A < P ? (TMEM_COLS - NSLOT * TJ) / COLS_A : P) : 0;
        const uint32_t tA = tmem_base + uint32_t(NSLOT * TJ);
        for (int it = 0; it < nTI; ++it) {
            tc::mbar_wait_sleep(a_full, uint32_t(it & 1));
            tc::fence_after();
            if (NTS > 0) {
                // the previous pass's MMAs are complete (the producer reloaded A after a_empty), so the
                // columns are free; tcgen05 ops of one thread run in order, so the MMAs below see the copy
                const uint64_t dAc = tc::smem_desc(aBase, 128, sbo);
                if (tc::elect_one())
#pragma unroll
                    for (int p = 0; p < NTS; ++p)
#pragma unroll
                        for (int ks = 0; ks < ksteps; ++ks)
                            tc::tmem_cp_128x256b(tA + uint32_t(p * COLS_A + ks * 8),
                                                 dAc + uint64_t((p * TI * kp + ks * 256) >> 4));
                __syncwarp();
            }
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                const int s = bq % NSTB;
                tc::mbar_wait_sleep(b_full + s, uint32_t((bq / NSTB) & 1));
                tc::fence_after();
                I8_TRACE(lane == 0, bq, 9);
                // Descriptors differ only in the start-address field (16-byte units):
                // two bases plus compile-time offsets in the fully unrolled sequence.
                const uint64_t dA0 = tc::smem_desc(aBase, 128, sbo);
                const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sB + s * C::B_BYTES), 128, sbo);
                // Time-multiplexed with the epilogue: no MMA of this tile while the epilogue's
                // FP64 exp phase of the previous tile runs.  Measured: INT8 MMAs throttle the
                // FP64 pipe ~4x (probe) to ~8x (in situ), so FP64 work overlapped with MMAs is
                // nearly wasted; serialising the exp phase is 6 % faster (d = 54 and 90).  The
                // drain (TMEM loads, integer combination) still overlaps the MMAs.
                if (!(I8_PROFILE && (A.debug & 32)) && bq > 0) {
                    tc::mbar_wait_sleep(epi_done, uint32_t((bq - 1) & 1));
                }
                I8_TRACE(lane == 0, bq, 8);  // the previous tile's epilogue has released the tensor core
#pragma unroll
                for (int c = NGRP - 1; c >= 0; --c) {
                    if (I8_REUSE && c < 2) {
                        // slot of group 6 / 5 of this tile: wait for the epilogue's drain of it
                        tc::mbar_wait_sleep(g_empty + (c == 1 ? 6 : 5), uint32_t(bq & 1));
                        tc::fence_after();
                    } else if (bq > 0) {
                        // the previous tile's drain of the group that last used this slot
                        const int prev = I8_REUSE ? (c == 6 ? 1 : (c == 5 ? 0 : c)) : c;
                        tc::mbar_wait_sleep(g_empty + prev, uint32_t((bq - 1) & 1));
                        tc::fence_after();
                    }
                    if (c == NGRP - 1 || c == 4 || c == 0) I8_TRACE(lane == 0, bq, c == NGRP - 1 ? 10 : (c == 4 ? 11 : 12));
                    if (tc::elect_one()) {
                        if (!(I8_PROFILE && (A.debug & 1)))
#pragma unroll
                            for (int p = 0; p <= c; ++p)
#pragma unroll
                                for (int ks = 0; ks < ksteps; ++ks) {
                                    const uint64_t db = dB0 + uint64_t(((c - p) * TJ * kp + ks * 256) >> 4);
                                    if (p < NTS)
                                        tc::mma_i8_ts(tmem_base + uint32_t(gslot(c) * TJ), tA + uint32_t(p * COLS_A + ks * 8), db,
                                                      idesc, (p == 0 && ks == 0) ? 0u : 1u);
                                    else
                                        tc::mma_i8(tmem_base + uint32_t(gslot(c) * TJ), dA0 + uint64_t((p * TI * kp + ks * 256) >> 4),
                                                   db, idesc, (p == 0 && ks == 0) ? 0u : 1u);
                                }
                        tc::mma_commit(g_full + c);
                    }
                    __syncwarp();
                }
                if (tc::elect_one()) tc::mma_commit(b_empty + s);
                __syncwarp();
            }
            if (tc::elect_one()) tc::mma_commit(a_empty);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = I8_MMA_LAST ? warp : warp - 2;  // 0..NEPI-1
        const int quarter = warp & 3;       // TMEM lane quarter this warp may access
        const int half = ew >> 2;           // which CPT of the 64 columns
        const int etid = ew * 32 + lane;
        const int row = quarter * 32 + lane;
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(half * CPT);
        double* scr = scr_all + ew * CPT * SCR_LD;
        const double* tab_l = tab + (lane & (TAB_REP - 1));  // this lane's table replica (conflict-free lookups)
        const int kabs_hi = __double2hiint(A.ec.kabs), kabs_lo = __double2loint(A.ec.kabs);
        int tq = 0;
        for (int it = 0; it < nTI; ++it) {
            const int64_t gi = rowBase + int64_t(it) * TI + row;
            const double sqs_i = A.sqs[gi];
            const double v_i = A.v[gi];
            // |kscale| 2^(e_i - 39) (Gaussian: -2 x.x = -2^(e_i+e_j-39) T) | gamma 2^(e_i - 40) (polynomial)
            const int nsi_hi = kabs_hi + (A.ex[gi] - (POLY ? 40 : 39)) * (1 << 20);
            double rowacc = 0.0;
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++tq) {
                const uint32_t ph = uint32_t(tq & 1);
                I8_TRACE(etid == 0, tq, 0);

                // ---- drain the 8 groups in MMA completion order (7 -> 0) two at a time,
                // 16 columns per tcgen05.ld (register pressure), releasing each pair at once
                // Completion order 6 -> 0, drained as (6, 5), (4, 3), (2, 1), (0).  W = sum_c 2^(8(6-c)) G_c
                // = 2^24 H + L with
                //   L = 2^24 G_3 + 2^16 G_4 + 2^8 G_5 + G_6   (|L| < 2^47),
                //   H = 2^24 G_0 + 2^16 G_1 + 2^8 G_2         (|H| < 2^45),
                // each built as int64 straight into the mantissa field of 1.5 * 2^52 (mad.wide), then
                // T = H + 2^-24 L = 2^-24 W with one DADD + one DFMA (one rounding).  Live partials: one
                // int64 (2^8 G_5 + G_6 can exceed int32 for all-128 digits), then the double L, then
                // 1.5 2^52 + 2^16 G_1 + 2^8 G_2 as int64.  (Pairing (6), (5, 4), (3, 2), (1, 0) measured 3 % slower.)
                int64_t acc[CPT], hp[CPT];
                double lo[CPT], T[CPT];
                auto stage = [&](int ca, int cb, auto&& fn) {  // groups ca (completes first) and cb = ca - 1 (or none)
                    // both loads in flight before one wait (TMEM load latency under load ~250 clk)
                    uint32_t ga[CPT], gb[CPT];
                    tc::mbar_wait_sleep(g_full + ca, ph);
                    tc::fence_after();
                    if (ca == 0) I8_TRACE(etid == 0, tq, 15);  // the tile's last MMA group is complete
                    tc::tmem_ld16(taddr + uint32_t(gslot(ca) * TJ), ga);
                    if (cb >= 0) {
                        tc::mbar_wait_sleep(g_full + cb, ph);
                        tc::fence_after();
                        tc::tmem_ld16(taddr + uint32_t(gslot(cb) * TJ), gb);
                    }
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < CPT; ++k) fn(k, int32_t(ga[k]), int32_t(gb[k]));
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        tc::mbar_arrive(g_empty + ca);
                        if (cb >= 0) tc::mbar_arrive(g_empty + cb);
                    }
                };
                if (I8_LATE_DRAIN) tc::mbar_wait_sleep(g_full + 0, ph);
                stage(6, 5, [&](int k, int32_t g6, int32_t g5) { acc[k] = mad_wide(g5, 256, int64_t(g6)); });
                I8_TRACE(etid == 0, tq, 1);
                stage(4, 3, [&](int k, int32_t g4, int32_t g3) {
                    lo[k] = __longlong_as_double(mad_wide(g3, 1 << 24, mad_wide(g4, 65536, acc[k] + MAGIC)));  // 1.5 2^52 + L
                });
                I8_TRACE(etid == 0, tq, 2);
                // 1.5 2^52 + 2^16 G_1 + 2^8 G_2 (|256 G_1 + G_2| < 2^30), so the tail adds 2^24 G_0 only (+2 %)
                stage(2, 1, [&](int k, int32_t g2, int32_t g1) { hp[k] = mad_wide(g1 * 256 + g2, 256, MAGIC); });
                I8_TRACE(etid == 0, tq, 3);
                stage(0, -1, [&](int k, int32_t g0, int32_t) {
#if I8_PROBE_NOFP64_T  // profiling only (wrong values): the last drain stage without its two FP64 ops
                    T[k] = __longlong_as_double((hp[k] + (int64_t(g0) << 24)) ^ __double_as_longlong(lo[k]));
#else
                    T[k] = fma(lo[k], 0x1p-24, __longlong_as_double(hp[k] + (int64_t(g0) << 24)) - M2);
#endif
                });

                // ---- exp, row sums, column sums
                I8_TRACE(etid == 0, tq, 4);
                const int cs = tq % NCD;
                tc::mbar_wait(cd_full + cs, uint32_t((tq / NCD) & 1));
                I8_TRACE(etid == 0, tq, 5);
                const uint8_t* cd = sCD + cs * CD_BYTES;
                const double* cd_sq = reinterpret_cast<const double*>(cd);
                const double* cd_v = reinterpret_cast<const double*>(cd + TJ * 8);
                const int* cd_e = reinterpret_cast<const int*>(cd + TJ * 16);
                double* colscr_q = colscr + ((tq & 1) * 4 + quarter) * TJ;
                const int colOff = half * CPT;
                const bool masked = diag && jt < (it + 1) * (TI / TJ);
                long long* trp = ((A.debug & 4) && blockIdx.x == 0 && etid == 0 && tq < TRACE_TILES)
                                     ? g_trace + tq * 16 : nullptr;
                // epi_done is arrived inside exp_phase (after its FP64 element loop) unless the
                // exp phase is skipped (profiling) or I8_EARLY_DONE = 0
                uint64_t* early = (I8_EARLY_DONE && !(I8_PROFILE && (A.debug & 2))) ? epi_done : nullptr;
                if (I8_PROFILE && (A.debug & 2)) {
                    double z = 0.0;
#pragma unroll
                    for (int k = 0; k < CPT; ++k) z += T[k];
                    rowacc += z;
                } else if (masked) {
                    // diagonal block: keep j > i (local column index vs local row index)
                    const int mask_row = row - (jt - it * (TI / TJ)) * TJ;
                    exp_phase<true, false, POLY>(T, A.ec, tab_l, cd_sq, cd_v, cd_e, scr, colscr_q, trp, nsi_hi, kabs_lo, sqs_i, v_i,
                                         rowacc, lane, colOff, mask_row, early);
                } else if (I8_PROFILE && (A.debug & 16)) {
                    exp_phase<false, true>(T, A.ec, tab_l, cd_sq, cd_v, cd_e, scr, colscr_q, trp, nsi_hi, kabs_lo, sqs_i,
                                           v_i, rowacc, lane, colOff, 0, early);
                } else {
                    exp_phase<false, false, POLY>(T, A.ec, tab_l, cd_sq, cd_v, cd_e, scr, colscr_q, trp, nsi_hi, kabs_lo, sqs_i, v_i,
                                          rowacc, lane, colOff, 0, early);
                }
                I8_TRACE(etid == 0, tq, 6);
                __syncwarp();
                if (lane == 0) {
                    tc::mbar_arrive(cd_empty + cs);
                    if (!early) tc::mbar_arrive(epi_done);
                }
                epi_bar();
                I8_TRACE(etid == 0, tq, 7);
                if (etid < TJ) {
                    double* cdst = A.part + int64_t(sa) * A.n_pad + colBase + int64_t(jt) * TJ + etid;
                    // the column's running sum (owner thread, same thread every pass), read here rather
                    // than prefetched before the drain: a shorter live range (fewer spills, +0.8 %)
                    const double cprev = it > 0 ? *cdst : 0.0;
                    const double* q4 = colscr + (tq & 1) * 4 * TJ + etid;
                    const double s4 = ((q4[0] + q4[TJ]) + q4[2 * TJ]) + q4[3 * TJ];
                    *cdst = cprev + s4;
                }
            }
            // row partials of this I tile: combine the column parts in fixed order
            rowbuf[half * TI + row] = rowacc;
            epi_bar();
            if (diag) {
                // same slot and index range as the column sums: the column owner adds
                if (etid < TJ) {
#pragma unroll
                    for (int h = 0; h < TI / TJ; ++h) {
                        const int r = h * TJ + etid;
                        double* dst = A.part + int64_t(sa) * A.n_pad + rowBase + int64_t(it) * TI + r;
                        double rs = rowbuf[r];
#pragma unroll
                        for (int h2 = 1; h2 < NEPI / 4; ++h2) rs += rowbuf[h2 * TI + r];
                        *dst = *dst + rs;
                    }
                }
            } else if (etid < TI) {
                double rs = rowbuf[etid];
#pragma unroll
                for (int h2 = 1; h2 < NEPI / 4; ++h2) rs += rowbuf[h2 * TI + etid];
                A.part[int64_t(sb) * A.n_pad + rowBase + int64_t(it) * TI + etid] = rs;
            }
            epi_bar();  // the scratch (row buffer) is reused by the next pass
        }
    }

    tc::fence_before();
    __syncthreads();
    if (warp == WARP_MMA) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

// ---- operand preparation
__global__ void row_exponent_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad,
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
            // |x_ik| 2^-e <= 127/255 - 2^-56: the range of 7 balanced 8-bit digits (tc_i8.cuh)
            int e = m > 0.0 ? ilogb(m) + 2 : 0;
            if (m > 0.0 && scalbn(m, -e) > 0.498) ++e;
            ex[i] = e;
            ejs[i] = e * (1 << 20);
        }
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
        int a[P];
        tc::balanced_digits8(x, ex[row], a);
        const int64_t off = (row >> 3) * int64_t(kp) * 8 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
#pragma unroll
        for (int p = 0; p < P; ++p) S[int64_t(p) * n_pad * kp + off] = uint8_t(int8_t(a[p]));
    }
}

// sq'_i = kscale |x_i|^2 (|x_i|^2 from the L operand's column d)
__global__ void scaled_sq_kernel(const double* __restrict__ L, int64_t n_pad, int dp, int d, double kscale,
                                 double* __restrict__ sqs) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad; i += int64_t(gridDim.x) * blockDim.x)
        sqs[i] = kscale * L[i * dp + d];
}

template <int KPT, bool POLY>
void launch_kp(const I8Args& a, int64_t num_tiles, cudaStream_t stream) {
    constexpr size_t smem = Cfg<KPT>::SMEM;
    static_assert(smem <= 227 * 1024, "K1-I8 shared memory");
    KRR_CUDA(cudaFuncSetAttribute(gauss_matvec_i8_kernel<KPT, POLY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    gauss_matvec_i8_kernel<KPT, POLY><<<unsigned(num_tiles), NTHR, smem, stream>>>(a);
}

// kscale of the 1/64-octave table exp (the K1 constant, -scale 64 / ln2)
double i8_kscale(double kscale64) { return kscale64; }

void ensure_table(cudaStream_t stream) {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    KRR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && done[dev]) return;
    double t[TAB];
    make_exp_table(t);  // 2^(j/64), correctly rounded (the K1 table)
    KRR_CUDA(cudaMemcpyToSymbolAsync(g_tab64, t, sizeof(t), 0, cudaMemcpyHostToDevice, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    if (dev < 64) done[dev] = true;
}

}  // namespace

void i8_read_trace(long long* out, int count) {
    count = std::min(count, TRACE_TILES * 16);
    KRR_CUDA(cudaMemcpyFromSymbol(out, g_trace, sizeof(long long) * size_t(count)));
}

bool i8_supported(int64_t d, int st) {
    const int kp = int((d + 31) / 32 * 32);
    return kp <= KP_MAX && st % TI == 0 && st >= TI;
}

int i8_kp(int64_t d) { return int((d + 31) / 32 * 32); }

bool i8_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, const double* L, int dp,
                       double kscale, uint8_t* S, int* ex, int* ejs, double* sqs, cudaStream_t stream,
                       double poly_gamma) {
    ensure_table(stream);  // here (it synchronises once) so graph-captured launches never need to
    const int kp = i8_kp(d);
    const double ks = i8_kscale(kscale);
    const unsigned wblocks = unsigned(std::min<int64_t>((n_pad + 7) / 8, 148 * 16));
    row_exponent_kernel<<<wblocks, 256, 0, stream>>>(X, n, d, n_pad, ex, ejs);
    KRR_LAUNCH_CHECK();
    const int64_t total = n_pad * kp;
    slice_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 32)), 256, 0, stream>>>(X, n, d, n_pad, kp,
                                                                                                 ex, S);
    KRR_LAUNCH_CHECK();
    scaled_sq_kernel<<<unsigned(std::min<int64_t>((n_pad + 255) / 256, 148 * 8)), 256, 0, stream>>>(
        L, n_pad, dp, int(d), ks, sqs);
    KRR_LAUNCH_CHECK();
    // exponent range: (1) |kscale| 2^(e_i + e_j - 39) stays a normal double;
    // (2) |y| = |kscale| d2 <= |kscale| 4 d 2^(2 e_max) < 2^50 (the 1.5 * 2^52 rounding shifter)
    std::vector<int> h(static_cast<size_t>(n_pad));
    KRR_CUDA(cudaMemcpyAsync(h.data(), ex, sizeof(int) * size_t(n_pad), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    int lo = 0, hi = 0;
    for (int e : h) {
        lo = std::min(lo, e);
        hi = std::max(hi, e);
    }
    if (poly_gamma > 0.0) {  // polynomial kernel: gamma 2^(e_i + e_j - 40) must be a normal double
        const int eg = std::ilogb(poly_gamma);
        return eg + 2 * lo - 40 > -1000 && eg + 2 * hi - 40 < 1000;
    }
    const int ek = std::ilogb(-ks);
    const double ymax = -ks * 4.0 * double(d) * std::ldexp(1.0, 2 * hi);
    return ek + 2 * lo - 39 > -1000 && ek + 2 * hi - 39 < 1000 && ymax < std::ldexp(1.0, 50);
}

void gauss_matvec_i8_launch(const GaussMatvecPlan& p, const uint8_t* S, const int* ex, const int* ejs,
                            const double* sqs, const double* v, double* part, int kp, cudaStream_t stream,
                            int debug, int poly_degree, double poly_gamma, double poly_offset) {
    if (p.num_tiles == 0) return;
    ensure_table(stream);
    I8Args a;
    a.S = S;
    a.ex = ex;
    a.ejs = ejs;
    a.sqs = sqs;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.n_pad = p.n_pad;
    a.st = p.st;
    a.debug = debug;
    const long double ln2 = 0.693147180559945309417232121458176568L;
    const long double l = ln2 / TAB;
    a.ec.kabs = -i8_kscale(p.ec.kscale);
    long double term = 1.0L;
    double c[6];
    for (int m = 1; m <= 5; ++m) {
        term = term * l / (long double)m;
        c[m] = double(term);
    }
    a.ec.a1 = c[1];
    a.ec.a2 = c[2];
    a.ec.a3 = c[3];
    a.ec.a4 = c[4];
    a.ec.a5 = c[5];
    a.ec.degree = 0;
    a.ec.pad_ = 0;
    const bool poly = poly_degree > 0;
    if (poly) {  // polynomial kernel: gamma, offset, degree in the constants (8f4)
        a.ec.kabs = poly_gamma;
        a.ec.a1 = poly_offset;
        a.ec.degree = poly_degree;
    }
    if (kp == 32) poly ? launch_kp<32, true>(a, p.num_tiles, stream) : launch_kp<32, false>(a, p.num_tiles, stream);
    else if (kp == 64) poly ? launch_kp<64, true>(a, p.num_tiles, stream) : launch_kp<64, false>(a, p.num_tiles, stream);
    else if (kp == 96) poly ? launch_kp<96, true>(a, p.num_tiles, stream) : launch_kp<96, false>(a, p.num_tiles, stream);
    else fail(KRR_ERR_INVALID_ARGUMENT, "K1-I8: kp must be 32, 64 or 96");
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
