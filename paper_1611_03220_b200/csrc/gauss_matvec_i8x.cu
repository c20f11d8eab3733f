// K1-I8X — the fused symmetric Gaussian mat-vec on the 5th-generation INT8 tensor cores with
// an INTEGER exp epilogue, so the epilogue of one tile runs under the next tile's MMAs.
//
// Why a second I8 kernel.  K1-I8 (gauss_matvec_i8.cu) evaluates ~15 FP64 operations per pair,
// and on B200 the INT8 tensor path throttles the FP64 pipe ~4x (DFMA 61 -> 16 lane-ops / clk /
// SM beside back-to-back kind::i8 MMAs, profiles/r1_tcgen05_contention.log), so K1-I8 must
// time-multiplex each SM: MMA phase, then FP64 exp phase (~8.1k + ~3.0k clk per 128 x 64 tile
// at d = 90).  The FP32 and integer pipes are not throttled (IMAD 314 -> 283).  K1-I8X moves the
// whole exp argument and the exp itself to 32/64-bit integer arithmetic; the FP64 pipe keeps 4
// operations per pair (one DFMA assembling e, the row DFMA, e v_i, the column DADD), and the
// MMAs of tile t+1 run while tile t's epilogue works.
//
// Arithmetic (restated bit for bit by paper_1611_03220_b200/intexp.py, checked on the CPU in
// tests/test_intexp.py).  z = sqrt(2 scale) x (fp64), one global exponent E (|z_ik| < 2^E,
// 1 <= E <= 8), 8 signed digits per element (round to nearest, exact in fp64).  Then with
// G = 55 - 2E fraction bits:
//     W_ij = sum_{c<=7} 2^(49-7c) G_c                     (G_c: tensor-core int32 sums, exact)
//     P_ij = floor(W_ij / 2^8)   = z_i.z_j 2^G
//     SQ_i = |z~_i|^2/2 2^G (floor)                       (prepared per row: every product of the digits)
//     u    = SQ_i + SQ_j - P_ij  = scale |x_i - x_j|^2 2^G  (int64; the cancellation is exact)
// The reference forms d2 = max(0, sq_i + sq_j - 2 p_ij) in fp64 (kernels.cpp:79-84), with
// rounding ~2^-53 (|x_i|^2 + |x_j|^2) scale; here only the slice truncation (~2^-55 |z|^2) enters.
// exp(-u) = 2^(-k/64) exp(s), k = round(u 64/ln2) (32-bit multiply of u's top bits), s = k ln2/64
// - u exactly mod 2^64 in units 2^-69 (|s| <= ln2/128), exp(s) - 1 = Q 2^-53 from s, s^2/2 (a
// two-limb square) and s^3 D(s) (32-bit Horner, mul.hi), all integer; then
//     e = fma(T_j 2^-53, X, T_j/4) 2^-m,   X = the double with bits 0x4338... + Q = 1.5 2^52 + Q,
// k = 64 m + j, T_j = 2^(-j/64) from a 64-entry table (T_j/4 is exact, so the one DFMA rounds
// once).  Error <= 2 ulp against exp of the exact fixed-point argument (tests/test_intexp.py).
//
// Structure: one CTA per symmetric super-tile, 18 warps, tiles M = 128 rows x N = 64 columns
// (the K1-I8 operand layout, tile order and part-slot rules; its finish kernel).
//   warps 0-15 epilogue (4 per TMEM lane quarter): drain the 8 groups (tcgen05.ld) in pairs,
//              combine into P (int64) and release each pair at once; integer exp; row sums in
//              registers, column sums through a per-warp shared-memory transpose;
//   warp 16    producer: I tile (resident for a 128-row pass), J tiles slice by slice (one
//              stage with per-slice barriers: slice q of tile t+1 is loaded as soon as tile t's
//              group q — the last one reading it — completes), per-column data (SQ_j, v_j);
//   warp 17    MMA issuer, the highest warp id on its SM sub-partition (the issue arbiter
//              prefers high warp ids, so the busy epilogue warps there cannot starve it).
// No epi_done hand-off: the tensor core runs as far ahead as TMEM (one tile) allows.
#include <cmath>
#include <cstring>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "kernels.cuh"
#include "tc_i8.cuh"

namespace krr {

namespace {

constexpr int P = 8;      // slices
constexpr int NGRP = 8;   // groups c = p + q in [0, 7]
constexpr int TI = 128;   // I tile rows (MMA M)
constexpr int TJ = 64;    // J tile columns (MMA N)
#ifndef I8X_QA
#define I8X_QA 0   // 1: exp(s) - 1 in integers in phase A; 0: k and s in phase A, the polynomial in FP64 in phase B
#endif
#ifndef I8X_BBW
#define I8X_BBW 1  // columns per phase-B batch (1, 2, 4, 8 measured equal: profiles/README.md)
#endif
#ifndef I8X_PRE6
#define I8X_PRE6 1  // load the next tile's groups 7, 6 before phase B, release them after it
#endif
#ifndef I8X_BLOAD
#define I8X_BLOAD 0  // 1: load a J tile only after the previous tile's MMAs (no TMA traffic under the MMAs)
#endif
constexpr int NCD = 4;    // column-data stages
constexpr int NEPI = 16;  // epilogue warps (4 per TMEM lane quarter)
constexpr int CPT = 16;   // columns per epilogue thread
constexpr int WARP_PROD = NEPI, WARP_MMA = NEPI + 1;
constexpr int NTHR = 32 * (NEPI + 2);
constexpr uint32_t TMEM_COLS = 512;
constexpr int KP_MAX = 96;
constexpr int SCR_LD = 33;   // transpose scratch row stride (doubles): conflict-free both ways
constexpr int CD_BYTES = TJ * 16;  // SQ_j (int64), v_j
constexpr int TAB = 64, TREP = 8;  // (T_j 2^-53, T_j / 4), T_j = 2^(-j/64), replicated 8x: conflict-free 16-B lookups

__device__ double2 g_xtab[TAB];
// profiling trace (debug bit 2): clock64 stamps of CTA 0, 16 per tile, first 64 tiles
constexpr int TRACE_TILES = 64;
__device__ long long g_xtrace[TRACE_TILES * 16];
#define X_TRACE(cond, tile, slot)                                                           \
    do {                                                                                    \
        if ((A.debug & 4) && blockIdx.x == 0 && (cond) && (tile) < TRACE_TILES)             \
            g_xtrace[(tile) * 16 + (slot)] = clock64();                                     \
    } while (0)

template <int KPT>
struct XCfg {
    static constexpr size_t A_BYTES = size_t(P) * TI * KPT;
    static constexpr size_t SLICE_B = size_t(TJ) * KPT;  // one J slice
    static constexpr size_t B_BYTES = P * SLICE_B;
    static constexpr size_t OFF_B = A_BYTES;
    static constexpr size_t OFF_CD = OFF_B + B_BYTES;
    static constexpr size_t OFF_SCR = OFF_CD + NCD * CD_BYTES;
    static constexpr size_t OFF_COLSCR = OFF_SCR + size_t(NEPI) * CPT * SCR_LD * 8;
    static constexpr size_t OFF_TAB = OFF_COLSCR + 2 * 4 * TJ * 8;
    static constexpr size_t OFF_PTAB = OFF_TAB + (I8X_QA ? TAB * TREP * 16 : 0);
    static constexpr size_t OFF_BARS = OFF_PTAB + (I8X_QA ? 0 : TAB * 16 * 8);
    static constexpr int NBARS = 2 + 2 * P + 2 * NCD + 2 * NGRP;
    static constexpr size_t SMEM = OFF_BARS + NBARS * 8 + 16;
};

struct XConsts {
    int sht;        // G - 21: u 2^G -> u 2^21
    int sh;         // 69 - G: u 2^G -> u 2^69
    int uhmax;      // high-word clamp (u <= ~700)
    int pad_;
};
// u- and E-independent constants (intexp.py:consts)
constexpr int K32H = 1549082005;                        // round(64/ln2 2^24)
constexpr uint32_t C69LO = 3907501270u, C69HI = 1488522235u;  // round(ln2/64 2^69)
// phase B polynomial (I8X_QA = 0): 2^(-53 n) / n!
constexpr double PB1 = 0x1p-53, PB2 = 0x1p-107, PB3 = 0x1.5555555555555p-162, PB4 = 0x1.5555555555555p-217,
                 PB5 = 0x1.1111111111111p-272;
constexpr int C3 = 1431655765, C4 = 1431655765, C5 = 286331153, C6 = 47721859;  // 2^35/24, /24, /120, /720

struct XArgs {
    const uint8_t* __restrict__ S;
    const long long* __restrict__ sq;  // SQ_i
    const double* __restrict__ v;
    double* __restrict__ part;
    const int2* __restrict__ tiles;
    int64_t n_pad;
    int st;
    int debug;  // profiling only (results invalid): bit 0 skips the MMAs, bit 1 phase A, bit 4 phase B
    XConsts c;
};

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, %0;\n" ::"n"(NEPI * 32) : "memory"); }

__device__ __forceinline__ int64_t mad_wide_s32(int a, int b, int64_t c) {
    int64_t d;
    asm("mad.wide.s32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}
__device__ __forceinline__ uint64_t mad_wide_u32(uint32_t a, uint32_t b, uint64_t c) {
    uint64_t d;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(d) : "r"(a), "r"(b), "l"(c));
    return d;
}
__device__ __forceinline__ int mad_hi_s32(int a, int b, int c) {
    int d;
    asm("mad.hi.s32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c));
    return d;
}

// Phase A (integer pipes only, under the next tile's MMAs): from nu = -u = P_ij - SQ_i - SQ_j
// (int64, units 2^-G) the reduction  exp(-u) = 2^(-k/64) exp(s),  k = round(u 64/ln2),
// s = k ln2/64 - u exactly (mod 2^64, units 2^-69, |s| <= ln2/128), and Q = (exp(s) - 1) 2^53
// from s, s^2/2 (two-limb square) and s^3 D(s) (32-bit Horner), packed as k << 47 | (Q + 2^46).
// (paper_1611_03220_b200/intexp.py:exp_neg, step for step.)  nu > 0 (d2 < 0 by the slice
// truncation, |nu| tiny) gives k = 0, s = -u and e = 1 + tiny.
__device__ __forceinline__ uint64_t xq_pack(int64_t nu, const XConsts& c) {
    const uint32_t nl = uint32_t(uint64_t(nu));
    const int nh = max(int(uint32_t(uint64_t(nu) >> 32)), -c.uhmax);        // u <= ~700: e stays normal
    const int nt = int(__funnelshift_rc(nl, uint32_t(nh), c.sht));           // -u 2^21
    const uint32_t k = uint32_t(__mulhi(nt, -K32H) + 4096) >> 13;           // round(u 64/ln2)
    const uint64_t nus = ((uint64_t(uint32_t(nh)) << 32) | nl) << c.sh;
    uint64_t sv = mad_wide_u32(k, C69LO, nus);
    sv += uint64_t(k * C69HI) << 32;
    const int64_t s = int64_t(sv);
    const int sh32 = int(uint32_t(sv >> 32));
    const uint32_t sl = uint32_t(sv);
    int64_t A = mad_wide_s32(sh32, sh32, 3ll << 20);                    // s^2 2^74 (+ rounding bias, intexp.py ABIAS)
    A = mad_wide_s32(__mulhi(sh32, int(sl >> 1)), 4, A);                // + the cross term
    const int a2 = int(__funnelshift_r(uint32_t(uint64_t(A)), uint32_t(uint64_t(A) >> 32), 28));  // s^2 2^46
    const int s38 = int(__funnelshift_r(sl, uint32_t(sh32), 31));       // s 2^38
    const int s3 = __mulhi(a2, s38);                                    // s^3 2^52
    const int sq = sh32 >> 5;                                           // s 2^32
    int t = __mulhi(C6, sq) + C5;
    t = __mulhi(t, sq) + C4;
    t = __mulhi(t, sq) + C3;                                            // (D(s) - 1/8) 2^35
    const int tail = __mulhi(s3, t) + s3 + 3;                           // s^3 D(s) 2^55
    A = mad_wide_s32(tail, 1 << 20, A);                                 // (s^2/2 + s^3 D) 2^75
    const uint64_t Qb = uint64_t((s >> 16) + (A >> 22)) + (1ull << 46); // Q + 2^46 in [0, 2^47)
    return (uint64_t(k) << 47) | Qb;
}

// Phase A variant (I8X_QA = 0): only k and s (rounded to 2^-53), packed k << 47 | (round(s 2^53) + 2^46);
// the polynomial then runs in FP64 in phase B.
__device__ __forceinline__ uint64_t xarg_pack(int64_t nu, const XConsts& c) {
    const uint32_t nl = uint32_t(uint64_t(nu));
    const int nh = max(int(uint32_t(uint64_t(nu) >> 32)), -c.uhmax);
    const int nt = int(__funnelshift_rc(nl, uint32_t(nh), c.sht));
    const uint32_t k = uint32_t(__mulhi(nt, -K32H) + 4096) >> 13;
    const uint64_t nus = ((uint64_t(uint32_t(nh)) << 32) | nl) << c.sh;
    uint64_t sv = mad_wide_u32(k, C69LO, nus + (1ull << 15) + (1ull << 62));  // + rounding, + 2^46 << 16
    sv += uint64_t(k * C69HI) << 32;
    return (uint64_t(k) << 47) | (sv >> 16);
}

__device__ __forceinline__ void arg_phase(const long long (&P_)[CPT], uint64_t (&E_)[CPT], const XConsts& c,
                                          const long long* __restrict__ cd_sq, long long sq_i, int colOff) {
#pragma unroll
    for (int k = 0; k < CPT; ++k)
        E_[k] = I8X_QA ? xq_pack(P_[k] - sq_i - cd_sq[colOff + k], c) : xarg_pack(P_[k] - sq_i - cd_sq[colOff + k], c);
}

// Phase B (FP64, while the tensor core is idle: INT8 MMAs throttle the FP64 pipe ~20x in situ,
// profiles/README.md): e = 2^-m T_j (1 + Q 2^-53) = fma(T_j 2^(-53-m), X, T_j 2^(-2-m)) with
// X = 1.5 2^52 + Q (exact, from the packed bits; T_j / 4 is exact, so e is rounded once), then the
// row sums (registers) and the column sums (per-warp transpose scratch; the 4 lane quarters
// combine in fixed order).
template <bool MASK>
__device__ __forceinline__ void exp_acc_phase(const uint64_t (&E_)[CPT], const double2* __restrict__ tab,
                                              const double* __restrict__ ptab,
                                              const double* __restrict__ cd_v, double* __restrict__ scr,
                                              double* __restrict__ colscr_q, double v_i, double& rowacc, int lane,
                                              int colOff, int mask_row) {
    double racc[4] = {0.0, 0.0, 0.0, 0.0};
    // I8X_BBW columns at a time, each step applied across the batch: independent FP64 chains side
    // by side for the scheduler (one column's chain is ~9 dependent FP64 operations)
#pragma unroll
    for (int k0 = 0; k0 < CPT; k0 += I8X_BBW) {
        double e[I8X_BBW], sd[I8X_BBW], q[I8X_BBW];
        uint32_t kk[I8X_BBW];
        if constexpr (I8X_QA) {
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) {
                const uint32_t hi = uint32_t(E_[k0 + b] >> 32), lo = uint32_t(E_[k0 + b]);
                kk[b] = hi >> 15;
                // bits of 1.5 2^52 + Q: the exponent of 2^52, mantissa 2^51 - 2^46 + (Q + 2^46)
                const double X = __hiloint2double(int((hi & 0x7FFFu) + (0x43300000u + 0x7C000u)), int(lo));
                const double2 tj = tab[(kk[b] & 63u) * TREP + (lane & (TREP - 1))];
                const double e1 = fma(tj.x, X, tj.y);  // T_j (1 + Q 2^-53) in (0.49, 1.01): 2^-m stays normal
                e[b] = __hiloint2double(__double2hiint(e1) - int((kk[b] >> 6) << 20), __double2loint(e1));
            }
        } else {
            // s 2^53 exactly (the bits of 2^52 + 2^46 + round(s 2^53), minus that constant), then
            // exp(s) - 1 by its degree-5 Taylor polynomial in s 2^53 (coefficients 2^-53n / n!)
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) {
                const uint32_t hi = uint32_t(E_[k0 + b] >> 32), lo = uint32_t(E_[k0 + b]);
                kk[b] = hi >> 15;
                sd[b] = __hiloint2double(int((hi & 0x7FFFu) | 0x43300000u), int(lo)) - 4573968371548160.0;
            }
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) q[b] = fma(sd[b], PB5, PB4);
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) q[b] = fma(q[b], sd[b], PB3);
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) q[b] = fma(q[b], sd[b], PB2);
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) q[b] = fma(q[b], sd[b], PB1);
#pragma unroll
            for (int b = 0; b < I8X_BBW; ++b) {
                q[b] = q[b] * sd[b];
                const double tj = ptab[(kk[b] & 63u) * 16 + (lane & 15)];
                const double ts = __hiloint2double(__double2hiint(tj) - int((kk[b] >> 6) << 20), __double2loint(tj));
                e[b] = fma(ts, q[b], ts);  // 2^-m T_j (1 + q)
            }
        }
#pragma unroll
        for (int b = 0; b < I8X_BBW; ++b) {
            const int k = k0 + b;
            if constexpr (MASK) e[b] = (colOff + k > mask_row) ? e[b] : 0.0;
            racc[k & 3] = fma(e[b], cd_v[colOff + k], racc[k & 3]);
            scr[k * SCR_LD + lane] = e[b] * v_i;  // column k, row `lane`
        }
    }
    rowacc += (racc[0] + racc[1]) + (racc[2] + racc[3]);
    __syncwarp();
    const double* src = scr + (lane % CPT) * SCR_LD + (lane / CPT) * 16;
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int r = 0; r < 16; r += 4) {
        a0 += src[r];
        a1 += src[r + 1];
        a2 += src[r + 2];
        a3 += src[r + 3];
    }
    double acc = (a0 + a1) + (a2 + a3);
    acc += __shfl_xor_sync(0xffffffffu, acc, CPT);
    if (lane < CPT) colscr_q[colOff + lane] = acc;
    __syncwarp();
}

template <int KPT>
__global__ void __launch_bounds__(NTHR, 1) gauss_matvec_i8x_kernel(const XArgs A) {
    using C = XCfg<KPT>;
    constexpr int kp = KPT;
    extern __shared__ __align__(1024) uint8_t smem[];
    uint8_t* sA = smem;
    uint8_t* sB = smem + C::OFF_B;
    uint8_t* sCD = smem + C::OFF_CD;
    double* scr_all = reinterpret_cast<double*>(smem + C::OFF_SCR);
    double* colscr = reinterpret_cast<double*>(smem + C::OFF_COLSCR);  // [2][4 quarters][64]
    double* rowbuf = scr_all;  // [NEPI/4 parts][128], only at pass ends (scratch idle)
    double2* tab = reinterpret_cast<double2*>(smem + C::OFF_TAB);
    double* ptab = reinterpret_cast<double*>(smem + C::OFF_PTAB);  // T_j replicated 16x (I8X_QA = 0)
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BARS);
    uint64_t* a_full = bars;
    uint64_t* a_empty = bars + 1;
    uint64_t* bs_full = bars + 2;      // per J slice
    uint64_t* bs_empty = bs_full + P;
    uint64_t* cd_full = bs_empty + P;
    uint64_t* cd_empty = cd_full + NCD;
    uint64_t* g_full = cd_empty + NCD;
    uint64_t* g_empty = g_full + NGRP;
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(g_empty + NGRP);

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
        for (int q = 0; q < P; ++q) {
            tc::mbar_init(bs_full + q, 1);
            tc::mbar_init(bs_empty + q, 1);
        }
        for (int s = 0; s < NCD; ++s) {
            tc::mbar_init(cd_full + s, 1);
            tc::mbar_init(cd_empty + s, NEPI);
        }
        for (int g = 0; g < NGRP; ++g) {
            tc::mbar_init(g_full + g, 1);
            tc::mbar_init(g_empty + g, NEPI);
        }
        tc::mbar_fence_init();
    }
    if (I8X_QA)
        for (int i = tid; i < TAB * TREP; i += NTHR) tab[i] = g_xtab[i / TREP];
    else
        for (int i = tid; i < TAB * 16; i += NTHR) ptab[i] = g_xtab[i / 16].y * 4.0;
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
                    const int64_t c0 = colBase + int64_t(jt) * TJ;
                    // slice q of this tile: after the previous tile's group q (its last reader)
                    for (int q = P - 1; q >= 0; --q) {
                        if (bq > 0) tc::mbar_wait_sleep(bs_empty + (I8X_BLOAD ? 0 : q), uint32_t((bq - 1) & 1));
                        tc::mbar_arrive_expect_tx(bs_full + q, uint32_t(C::SLICE_B));
                        tc::bulk_g2s(sB + q * C::SLICE_B, A.S + int64_t(q) * A.n_pad * kp + c0 * kp,
                                     uint32_t(C::SLICE_B), bs_full + q);
                    }
                    const int cs = bq % NCD;
                    if (bq >= NCD) tc::mbar_wait_sleep(cd_empty + cs, uint32_t(((bq / NCD) - 1) & 1));
                    tc::mbar_arrive_expect_tx(cd_full + cs, uint32_t(CD_BYTES));
                    uint8_t* cd = sCD + cs * CD_BYTES;
                    tc::bulk_g2s(cd, A.sq + c0, TJ * 8, cd_full + cs);
                    tc::bulk_g2s(cd + TJ * 8, A.v + c0, TJ * 8, cd_full + cs);
                }
            }
        }
    } else if (warp == WARP_MMA) {
        // ------------------------------------------------------------ MMA issuer
        const uint32_t idesc = tc::idesc_i8(TI, TJ);
        const uint32_t aBase = tc::smem_u32(sA);
        const uint64_t dA0 = tc::smem_desc(aBase, 128, sbo);
        const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sB), 128, sbo);
        int bq = 0;
        for (int it = 0; it < nTI; ++it) {
            tc::mbar_wait_sleep(a_full, uint32_t(it & 1));
            tc::fence_after();
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++bq) {
                const uint32_t ph = uint32_t(bq & 1);
#pragma unroll
                for (int c = NGRP - 1; c >= 0; --c) {
                    if (c == NGRP - 1) X_TRACE(lane == 0, bq, 8);
                    if (bq > 0) {
                        tc::mbar_wait_sleep(g_empty + c, uint32_t((bq - 1) & 1));
                        tc::fence_after();
                    }
                    if (c == 7 || c == 4 || c == 0) X_TRACE(lane == 0, bq, c == 7 ? 9 : (c == 4 ? 10 : 11));
                    if (c == NGRP - 1) {
                        // the first group reads every J slice (p ascending: slice 7 first, slice 0 —
                        // freed last by the previous tile — last): wait for each before its MMAs
#pragma unroll
                        for (int p = 0; p <= c; ++p) {
                            tc::mbar_wait_sleep(bs_full + (c - p), ph);
                            tc::fence_after();
                            if (tc::elect_one() && !(A.debug & 1))
#pragma unroll
                                for (int ks = 0; ks < ksteps; ++ks)
                                    tc::mma_i8(tmem_base + uint32_t(c * TJ), dA0 + uint64_t((p * TI * kp + ks * 256) >> 4),
                                               dB0 + uint64_t(((c - p) * TJ * kp + ks * 256) >> 4), idesc,
                                               (p == 0 && ks == 0) ? 0u : 1u);
                            __syncwarp();
                        }
                    } else if (tc::elect_one() && !(A.debug & 1)) {
#pragma unroll
                        for (int p = 0; p <= c; ++p)
#pragma unroll
                            for (int ks = 0; ks < ksteps; ++ks)
                                tc::mma_i8(tmem_base + uint32_t(c * TJ), dA0 + uint64_t((p * TI * kp + ks * 256) >> 4),
                                           dB0 + uint64_t(((c - p) * TJ * kp + ks * 256) >> 4), idesc,
                                           (p == 0 && ks == 0) ? 0u : 1u);
                    }
                    __syncwarp();
                    if (tc::elect_one()) {
                        tc::mma_commit(g_full + c);
                        tc::mma_commit(bs_empty + c);  // group c is the last reader of J slice c
                    }
                    __syncwarp();
                }
            }
            if (tc::elect_one()) tc::mma_commit(a_empty);
            __syncwarp();
        }
    } else {
        // ------------------------------------------------------------ epilogue
        const int ew = warp;                // 0..NEPI-1
        const int quarter = warp & 3;       // TMEM lane quarter this warp may access
        const int half = ew >> 2;           // which CPT of the 64 columns
        const int etid = ew * 32 + lane;
        const int row = quarter * 32 + lane;
        const uint32_t taddr = tmem_base + (uint32_t(quarter * 32) << 16) + uint32_t(half * CPT);
        double* scr = scr_all + ew * CPT * SCR_LD;
        // tiles of this CTA (the MMA warp's order), to know whether a next tile's MMAs are coming
        int ntiles_cta = 0;
        for (int it2 = 0; it2 < nTI; ++it2) ntiles_cta += nTJ - (diag ? it2 * (TI / TJ) : 0);
        int tq = 0;
        for (int it = 0; it < nTI; ++it) {
            const int64_t gi = rowBase + int64_t(it) * TI + row;
            const long long sq_i = A.sq[gi];
            const double v_i = A.v[gi];
            double rowacc = 0.0;
            int32_t b3[CPT];  // groups 7, 6 of the tile, loaded early (I8X_PRE6) while the previous one finishes
            bool have6 = false;
            for (int jt = diag ? it * (TI / TJ) : 0; jt < nTJ; ++jt, ++tq) {
                const uint32_t ph = uint32_t(tq & 1);
                // ---- drain the 8 groups in MMA completion order (7 -> 0) two at a time, combining
                // b_k = 128 G_2k + G_2k+1 into P = floor(W / 2^8) = b0 2^34 + b1 2^20 + b2 2^6 + (b3 >> 8)
                long long Pv[CPT];
                auto stage = [&](int ca, auto&& fn) {
                    uint32_t gl[CPT], gh[CPT];
                    tc::mbar_wait_sleep(g_full + ca + 1, ph);
                    tc::fence_after();
                    tc::tmem_ld16(taddr + uint32_t((ca + 1) * TJ), gl);
                    tc::mbar_wait_sleep(g_full + ca, ph);
                    tc::fence_after();
                    tc::tmem_ld16(taddr + uint32_t(ca * TJ), gh);
                    tc::tmem_wait_ld();
#pragma unroll
                    for (int k = 0; k < CPT; ++k) fn(k, int32_t(gh[k]) * 128 + int32_t(gl[k]));
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        tc::mbar_arrive(g_empty + ca + 1);
                        tc::mbar_arrive(g_empty + ca);
                    }
                };
                X_TRACE(etid == 0, tq, 0);
                if (!have6) stage(6, [&](int k, int32_t b) { b3[k] = b; });
                X_TRACE(etid == 0, tq, 1);
                stage(4, [&](int k, int32_t b) { Pv[k] = (long long)b * 64 + (long long)(b3[k] >> 8); });
                stage(2, [&](int k, int32_t b) { Pv[k] += (long long)b * (1 << 20); });
                stage(0, [&](int k, int32_t b) {
                    Pv[k] = (long long)((unsigned long long)Pv[k] + ((unsigned long long)(uint32_t(b * 4)) << 32));
                });

                X_TRACE(etid == 0, tq, 2);
                // ---- phase A (integer pipes, under the next tile's MMAs): e bits of 16 pairs
                const int cs = tq % NCD;
                tc::mbar_wait(cd_full + cs, uint32_t((tq / NCD) & 1));
                const uint8_t* cd = sCD + cs * CD_BYTES;
                const long long* cd_sq = reinterpret_cast<const long long*>(cd);
                const double* cd_v = reinterpret_cast<const double*>(cd + TJ * 8);
                double* colscr_q = colscr + ((tq & 1) * 4 + quarter) * TJ;
                const int colOff = half * CPT;
                const bool masked = diag && jt < (it + 1) * (TI / TJ);
                // the column owner's running sum (global), loaded now so its latency hides under phase A
                double* cdst = A.part + int64_t(sa) * A.n_pad + colBase + int64_t(jt) * TJ + etid;
                const double cprev = (etid < TJ && it > 0) ? *cdst : 0.0;
                uint64_t Eb[CPT];
                if (A.debug & 2) {
#pragma unroll
                    for (int k = 0; k < CPT; ++k) Eb[k] = uint64_t(Pv[k]) & 0x3FFFFFFFFFFFFFFFull;
                } else {
                    arg_phase(Pv, Eb, A.c, cd_sq, sq_i, colOff);
                }
                X_TRACE(etid == 0, tq, 3);
                // ---- phase B (FP64) once the next tile's MMAs are done, so the FP64 pipe runs
                // unthrottled; at a pass end the next I tile is still loading (tensor core idle)
                have6 = false;
                if (tq + 1 < ntiles_cta && jt + 1 < nTJ) {
                    tc::mbar_wait(g_full + 0, uint32_t((tq + 1) & 1));
                    if (I8X_PRE6) {
                        // the next tile's groups 7 and 6 into registers now; released after phase B, so
                        // the tensor core restarts without waiting for these TMEM loads
                        uint32_t gl[CPT], gh[CPT];
                        tc::fence_after();
                        tc::tmem_ld16(taddr + uint32_t(7 * TJ), gl);
                        tc::tmem_ld16(taddr + uint32_t(6 * TJ), gh);
                        tc::tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < CPT; ++k) b3[k] = int32_t(gh[k]) * 128 + int32_t(gl[k]);
                        have6 = true;
                    }
                }
                X_TRACE(etid == 0, tq, 4);
                if (A.debug & 16) {  // profiling: no phase B (results invalid)
                    uint64_t z = 0;
#pragma unroll
                    for (int k = 0; k < CPT; ++k) z ^= Eb[k];
                    rowacc += double(z & 1);
                } else if (masked)
                    exp_acc_phase<true>(Eb, tab, ptab, cd_v, scr, colscr_q, v_i, rowacc, lane, colOff,
                                        row - (jt - it * (TI / TJ)) * TJ);
                else
                    exp_acc_phase<false>(Eb, tab, ptab, cd_v, scr, colscr_q, v_i, rowacc, lane, colOff, 0);
                X_TRACE(etid == 0, tq, 5);
                if (have6) {
                    tc::fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        tc::mbar_arrive(g_empty + 7);
                        tc::mbar_arrive(g_empty + 6);
                    }
                }
                __syncwarp();
                if (lane == 0) tc::mbar_arrive(cd_empty + cs);
                epi_bar();
                X_TRACE(etid == 0, tq, 6);
                if (etid < TJ) {
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
__global__ void absmax_kernel(const double* __restrict__ X, int64_t total, unsigned long long* __restrict__ out) {
    double m = 0.0;
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < total; i += int64_t(gridDim.x) * blockDim.x)
        m = fmax(m, fabs(X[i]));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) == 0) atomicMax(out, static_cast<unsigned long long>(__double_as_longlong(m)));
}

// the 8 digits of u = fl(c x) 2^-E, rounded to nearest (exact in fp64): |a_0| <= 127, |a_p| <= 64
// after it, so the products the pair kernel drops (p + q >= 8) are ~4x smaller than with
// truncated 7-bit digits and the representation error is zero-mean (|u - u~| <= 2^-57)
__device__ __forceinline__ void digits(double x, double c, double c_lo, int E, int (&a)[P]) {
    // z = x sqrt(2 scale) with sqrt(2 scale) = c + c_lo (double-double): one rounding per element,
    // no systematic bias from rounding the constant itself
    double w = scalbn(fma(x, c, x * c_lo), 7 - E);
#pragma unroll
    for (int p = 0; p < P; ++p) {
        const double t = rint(w);
        a[p] = int(t);
        w = (w - t) * 128.0;
    }
}

__global__ void slice_x_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, int kp, double c,
                               double c_lo, int E, uint8_t* __restrict__ S) {
    const int64_t total = n_pad * kp;
    for (int64_t idx = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; idx < total;
         idx += int64_t(gridDim.x) * blockDim.x) {
        const int64_t row = idx / kp;
        const int k = int(idx % kp);
        const double x = (row < n && k < d) ? X[row * d + k] : 0.0;
        int a[P];
        digits(x, c, c_lo, E, a);
        const int64_t off = (row >> 3) * int64_t(kp) * 8 + (k >> 4) * 128 + (row & 7) * 16 + (k & 15);
#pragma unroll
        for (int p = 0; p < P; ++p) S[int64_t(p) * n_pad * kp + off] = uint8_t(int8_t(a[p]));
    }
}

// SQ_i = floor(|z~_i|^2 / 2 2^G) of the truncated digits z~ (one warp per row, exact integer sums).
// All products, c = p + q up to 14: the pair kernel keeps c <= 7, whose dropped terms are
// zero-mean for i != j, but on the diagonal the p = q squares would bias |z~|^2 low (~2^-49 |z|^2).
__global__ void sq_x_kernel(const double* __restrict__ X, int64_t n, int64_t d, int64_t n_pad, double c,
                            double c_lo, int E, long long* __restrict__ sq) {
    constexpr int NC = 2 * P - 1;
    const int lane = threadIdx.x & 31;
    const int64_t warps = int64_t(gridDim.x) * (blockDim.x >> 5);
    for (int64_t i = blockIdx.x * int64_t(blockDim.x >> 5) + (threadIdx.x >> 5); i < n_pad; i += warps) {
        long long g[NC];
#pragma unroll
        for (int cc = 0; cc < NC; ++cc) g[cc] = 0;
        if (i < n)
            for (int64_t k = lane; k < d; k += 32) {
                int a[P];
                digits(X[i * d + k], c, c_lo, E, a);
#pragma unroll
                for (int p = 0; p < P; ++p)
#pragma unroll
                    for (int q = 0; q < P; ++q) g[p + q] += (long long)(a[p] * a[q]);
            }
#pragma unroll
        for (int cc = 0; cc < NC; ++cc)
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) g[cc] += __shfl_xor_sync(0xffffffffu, g[cc], o);
        if (lane == 0) {
            // |z~|^2 2^G / 2 = sum_c 2^(40 - 7c) G_c = (sum_c 2^(98 - 7c) G_c) / 2^58
            __int128 w = 0;
#pragma unroll
            for (int cc = 0; cc < NC; ++cc) w += (__int128)g[cc] << (98 - 7 * cc);
            sq[i] = (long long)(w >> 58);
        }
    }
}

template <int KPT>
void launch_kp(const XArgs& a, int64_t num_tiles, cudaStream_t stream) {
    constexpr size_t smem = XCfg<KPT>::SMEM;
    static_assert(smem <= 227 * 1024, "K1-I8X shared memory");
    KRR_CUDA(cudaFuncSetAttribute(gauss_matvec_i8x_kernel<KPT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    gauss_matvec_i8x_kernel<KPT><<<unsigned(num_tiles), NTHR, smem, stream>>>(a);
}

void ensure_xtable(cudaStream_t stream) {
    static std::mutex mu;
    static bool done[64] = {};
    int dev = 0;
    KRR_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mu);
    if (dev < 64 && done[dev]) return;
    double2 t[TAB];
    for (int j = 0; j < TAB; ++j) {
        const double tj = double(exp2l(-(long double)j / 64.0L));  // 2^(-j/64), correctly rounded
        t[j] = make_double2(std::ldexp(tj, -53), std::ldexp(tj, -2));
    }
    KRR_CUDA(cudaMemcpyToSymbolAsync(g_xtab, t, sizeof(t), 0, cudaMemcpyHostToDevice, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    if (dev < 64) done[dev] = true;
}

XConsts make_xconsts(int E) {
    const int G = 55 - 2 * E;
    XConsts c{};
    c.sht = G - 21;
    c.sh = 69 - G;
    c.uhmax = int(std::floor(700.0L * std::ldexp(1.0L, G - 32)));
    c.pad_ = 0;
    return c;
}

}  // namespace

void i8x_read_trace(long long* out, int count) {
    count = std::min(count, TRACE_TILES * 16);
    KRR_CUDA(cudaMemcpyFromSymbol(out, g_xtrace, sizeof(long long) * size_t(count)));
}

bool i8x_supported(int64_t d, int st) { return i8_kp(d) <= KP_MAX && st % TI == 0 && st >= TI; }

int i8x_prepare_launch(const double* X, int64_t n, int64_t d, int64_t n_pad, double scale, uint8_t* S, long long* sq,
                       cudaStream_t stream) {
    ensure_xtable(stream);  // (synchronises once) so graph-captured launches never need to
    // max |x| (the bits of non-negative doubles order like the values) in a per-call scratch word,
    // so contexts preparing concurrently on one device do not share it
    unsigned long long* dmax = nullptr;
    KRR_CUDA(cudaMallocAsync(reinterpret_cast<void**>(&dmax), sizeof(unsigned long long), stream));
    KRR_CUDA(cudaMemsetAsync(dmax, 0, sizeof(unsigned long long), stream));
    const int64_t total = n * d;
    if (total > 0) {
        absmax_kernel<<<unsigned(std::min<int64_t>((total + 255) / 256, 148 * 8)), 256, 0, stream>>>(X, total, dmax);
        KRR_LAUNCH_CHECK();
    }
    unsigned long long bits = 0;
    KRR_CUDA(cudaMemcpyAsync(&bits, dmax, sizeof(bits), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaFreeAsync(dmax, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    double xmax = 0.0;
    std::memcpy(&xmax, &bits, sizeof(xmax));
    const double c = std::sqrt(2.0 * scale);
    const double c_lo = std::fma(-c, c, 2.0 * scale) / (2.0 * c);  // sqrt(2 scale) = c + c_lo
    const double zmax = std::fma(xmax, c, xmax * c_lo);  // = max_ik |z_ik|: the rounding is monotonic
    if (!std::isfinite(zmax)) return 0;
    int E = std::max(1, zmax > 0.0 ? std::ilogb(zmax) + 1 : 1);
    // the rounded leading digit stays <= 127 (with a margin for the per-element fma rounding)
    while (zmax * (1.0 + 0x1p-40) >= std::ldexp(127.5 / 128.0, E)) ++E;
    if (E > 8) return 0;  // |z| >= 128: out of K1-I8X's fixed-point range (K1-I8 / DMMA serve it)
    const int kp = i8_kp(d);
    const int64_t st = n_pad * kp;
    slice_x_kernel<<<unsigned(std::min<int64_t>((st + 255) / 256, 148 * 32)), 256, 0, stream>>>(X, n, d, n_pad, kp, c,
                                                                                               c_lo, E, S);
    KRR_LAUNCH_CHECK();
    sq_x_kernel<<<unsigned(std::min<int64_t>((n_pad + 7) / 8, 148 * 16)), 256, 0, stream>>>(X, n, d, n_pad, c, c_lo, E, sq);
    KRR_LAUNCH_CHECK();
    return E;
}

void gauss_matvec_i8x_launch(const GaussMatvecPlan& p, const uint8_t* S, const long long* sq, int E, const double* v,
                             double* part, int kp, cudaStream_t stream, int debug) {
    if (p.num_tiles == 0) return;
    ensure_xtable(stream);
    XArgs a;
    a.S = S;
    a.sq = sq;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.n_pad = p.n_pad;
    a.st = p.st;
    a.debug = debug;
    a.c = make_xconsts(E);

    if (kp == 32) launch_kp<32>(a, p.num_tiles, stream);
    else if (kp == 64) launch_kp<64>(a, p.num_tiles, stream);
    else if (kp == 96) launch_kp<96>(a, p.num_tiles, stream);
    else fail(KRR_ERR_INVALID_ARGUMENT, "K1-I8X: kp must be 32, 64 or 96");
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
