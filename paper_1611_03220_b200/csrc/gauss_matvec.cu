// K1 — fused, symmetric, on-the-fly Gaussian kernel mat-vec (K never stored).
//
// Replaces gram_matrix (reference kernels.cpp:72-88) + the dense apply_a GEMV
// (solver.cpp:75-77).  Per unordered pair {i, j} (i < j) it computes
//     d2  = |x_i|^2 + |x_j|^2 - 2 x_i.x_j      (ONE FP64 tensor-core contraction:
//           L_i . R_j with L_i = [x_i, |x_i|^2, 1], R_j = [-2 x_j, 1, |x_j|^2]),
//     e   = exp(-max(0, d2) / (2 sigma^2))    (register epilogue, gauss_exp.cuh),
//     out_i += e v_j  and  out_j += e v_i     (both halves of the symmetric matrix
//                                               from one evaluation => K_ij == K_ji
//                                               bitwise, as in kernels.cpp:85-86).
// The diagonal K_ii = 1 (kernels.cpp:81) and +lambda v_i are added by the finish
// kernel.
//
// Work decomposition (deterministic, no atomics):
//   rows are padded to n_pad (multiple of the super-tile edge ST, itself a multiple
//   of 128); super-tile (a, b), a <= b, covers rows [a ST, (a+1) ST) x cols
//   [b ST, (b+1) ST).  One CTA per super-tile.  Inside, 128 x 128 tiles are visited
//   column-tile-major (J outer, I inner); diagonal super-tiles visit only I <= J and
//   the I == J tile only strictly above its diagonal.
//   Row sums of a super-tile accumulate in shared memory (ST doubles) and are
//   written once to part[b][rows of a]; column sums of each J tile are reduced in
//   registers over the whole I sweep and written once to part[a][rows of b].  Every
//   slot part[x][rows of y] therefore has exactly one writer (for x == y the two
//   halves are combined in shared memory first), and the finish kernel sums the NS
//   slots of a row in a fixed order.
//
// Mainloop: 256 threads = 8 warps as 2 (M) x 4 (N), warp tile 64 x 32 =
// 8 x 4 DMMA.8x8x4 accumulators (64 doubles per thread).  Operands stream through a
// cp.async pipeline in k-chunks of 16 doubles (smem row stride 20 doubles =>
// conflict-free fragment loads); the pipeline runs across tile boundaries.
//
// Three pipeline shapes (same arithmetic, bitwise-identical results):
//   streaming  both L_I and R_J chunks stream (3 stages) — small super-tiles;
//   resident   R_J stays in shared memory for the whole I sweep, L_I streams;
//   grouped    (default for super-tiles >= 1024 rows) resident R_J and two decoupled,
//              phase-offset warp groups, each streaming its own half of L_I behind
//              its own named barrier.  Measured on B200: DMMA and DFMA share ONE FP64
//              datapath (split-warp microbenchmark: 37.0 TFLOP/s combined = DMMA
//              alone), so the only way to fill the latency-bound exp epilogue's idle
//              pipe cycles is another warp's DMMAs on the same SM sub-partition.
#include <type_traits>

#include "common.cuh"
#include "gauss_exp.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int BM = 128;           // tile edge (rows and cols)
constexpr int KC = 16;            // k-chunk (doubles)
constexpr int KS = 20;            // smem row stride (doubles), 20 = 4 mod 16
constexpr int MAX_SMEM = 227 * 1024;
constexpr int WGN = 4;            // warps along the tile's columns (warp tile 32 columns)

// Warp layout: MS m8-subtiles per warp (warp tile 8*MS x 32), WGM = 16/MS warps along
// the rows.  MS = 8: 8 warps, 64 accumulator doubles per thread (255 registers, 2 warps
// per SM sub-partition).  MS = 4: 16 warps, 32 accumulator doubles (<= 128 registers,
// 4 warps per sub-partition for latency hiding).
template <int MS>
struct Warps {
    static constexpr int WGM = 16 / MS;
    static constexpr int NT = 32 * WGM * WGN;
};

// Two pipeline shapes:
//  streaming (RES = false): each stage holds a k-chunk of both L_I and R_J (3 stages);
//  resident  (RES = true):  R_J (128 x dp) stays in shared memory for the whole I sweep
//                           and only L_I chunks stream (4 stages) — half the copy work.
template <bool RES>
struct Shape {
    static constexpr int NSTAGE = RES ? 4 : 3;
    static constexpr int STAGE_DOUBLES = (RES ? 1 : 2) * BM * KS;
};

struct MatvecArgs {
    const double* __restrict__ L;
    const double* __restrict__ R;
    const double* __restrict__ v;
    double* __restrict__ part;
    const int2* __restrict__ tiles;
    const double* __restrict__ exp_tab;
    int64_t n_pad;
    int dp;
    int st;
    int ksr;  // resident R_J row stride (doubles), = 4 or 12 mod 16
    ExpConsts ec;
};

// Epilogue of one warp tile: e = exp(-max(0, d2) scale) for the warp's MS x 4 DMMA
// accumulator blocks, then row partials rowp[ms] (over the warp's 32 columns, this
// thread's 8 of them) and column partials colacc (accumulated across the I sweep).
// On a diagonal tile only the strictly upper pairs (j > i) count.
template <int EXPMODE, int MS>
__device__ __forceinline__ void tile_epilogue(double (&acc)[MS][4][2], const double (&vi)[MS],
                                              const double (&vj)[4][2], double (&colacc)[4][2],
                                              double (&rowp)[MS], bool dtile, int il0, int jl0, int g,
                                              int t4, const ExpConsts& ec, const double* tab) {
#pragma unroll
    for (int ms = 0; ms < MS; ++ms) {
        rowp[ms] = 0.0;
        const int il = il0 + ms * 8 + g;
#pragma unroll
        for (int ns = 0; ns < 4; ++ns)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double e = gauss_exp<EXPMODE>(acc[ms][ns][h], ec, tab);
                if (dtile) {
                    const int jl = jl0 + ns * 8 + 2 * t4 + h;
                    e = (jl > il) ? e : 0.0;
                }
                rowp[ms] = fma(e, vj[ns][h], rowp[ms]);
                colacc[ns][h] = fma(e, vi[ms], colacc[ns][h]);
            }
    }
}

__device__ __forceinline__ void named_bar_sync(int id, int count) {
    asm volatile("bar.sync %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}
__device__ __forceinline__ void named_bar_arrive(int id, int count) {
    asm volatile("bar.arrive %0, %1;\n" ::"r"(id), "r"(count) : "memory");
}

template <int EXPMODE, bool RES, int MS>
__global__ void __launch_bounds__(Warps<MS>::NT, 1) gauss_matvec_kernel(const MatvecArgs A) {
    constexpr int WGM = Warps<MS>::WGM;
    constexpr int NTHREADS = Warps<MS>::NT;
    constexpr int WM = 8 * MS;
    constexpr int NSTAGE = Shape<RES>::NSTAGE;
    constexpr int STAGE_DOUBLES = Shape<RES>::STAGE_DOUBLES;
    extern __shared__ __align__(16) double smem[];
    double* rres = smem;                                    // RES: BM * ksr
    double* stages = smem + (RES ? BM * A.ksr : 0);          // NSTAGE * STAGE_DOUBLES
    double* rowacc = stages + NSTAGE * STAGE_DOUBLES;       // st
    double* scr_row = rowacc + A.st;                        // 4 x 128
    double* scr_col = scr_row + WGN * BM;                   // WGM x 128
    double* tab = scr_col + WGM * BM;                       // 64
    double* vjs = tab + 64;                                 // 128: v of the current J tile

    const int tid = threadIdx.x;
    const int lane = tid & 31, warp = tid >> 5;
    const int wm = warp % WGM, wn = warp / WGM;
    const int g = lane >> 2, t4 = lane & 3;

    const int2 tile = A.tiles[blockIdx.x];
    const int sa = tile.x, sb = tile.y;
    const bool diag = (sa == sb);
    const int nT = A.st / BM;
    const int64_t rowBase = int64_t(sa) * A.st;
    const int64_t colBase = int64_t(sb) * A.st;
    const int nk = (A.dp + KC - 1) / KC;
    const int ntiles = diag ? nT * (nT + 1) / 2 : nT * nT;
    const int total = ntiles * nk;

    for (int i = tid; i < A.st; i += NTHREADS) rowacc[i] = 0.0;
    if (EXPMODE == 1 && tid < 64) tab[tid] = A.exp_tab[tid];

    // ---- producer cursor over (jt, it, kc)
    int p_it = 0, p_jt = 0, p_kc = 0;
    auto issue = [&](int slot) {
        double* sL = stages + slot * STAGE_DOUBLES;
        double* sR = sL + BM * KS;
        const int k0 = p_kc * KC;
        const int pieces = min(KC, A.dp - k0) >> 1;  // 16-byte pieces per row
        const double* gL = A.L + (rowBase + int64_t(p_it) * BM) * A.dp + k0;
        const double* gR = A.R + (colBase + int64_t(p_jt) * BM) * A.dp + k0;
#pragma unroll
        for (int q = 0; q < ((RES ? 1 : 2) * BM * (KC / 2)) / NTHREADS; ++q) {
            const int idx = tid + q * NTHREADS;
            const int op = RES ? 0 : idx / (BM * (KC / 2));
            const int rem = idx % (BM * (KC / 2));
            const int row = rem / (KC / 2), pc = rem % (KC / 2);
            if (pc < pieces) {
                const double* gp = (op ? gR : gL) + int64_t(row) * A.dp + pc * 2;
                double* sp = (op ? sR : sL) + row * KS + pc * 2;
                cp_async16(sp, gp);
            }
        }
    };
    auto advance = [&]() {
        if (++p_kc == nk) {
            p_kc = 0;
            ++p_it;
            if (p_it > (diag ? p_jt : nT - 1)) {
                p_it = 0;
                ++p_jt;
            }
        }
    };

    int ps = 0;  // next stage index to issue
#pragma unroll
    for (int s = 0; s < NSTAGE - 1; ++s) {
        if (ps < total) {
            issue(ps % NSTAGE);
            advance();
        }
        cp_async_commit();
        ++ps;
    }
    __syncthreads();  // rowacc / tab initialised

    int cs = 0;  // consumer stage index
    for (int jt = 0; jt < nT; ++jt) {
        const int64_t J0 = colBase + int64_t(jt) * BM;
        if constexpr (RES) {
            // R_J for the whole I sweep: drain the pipeline, load, publish.
            __syncthreads();
            const int pieces = A.dp >> 1;
            const double* gR = A.R + J0 * A.dp;
            for (int idx = tid; idx < BM * pieces; idx += NTHREADS) {
                const int row = idx / pieces, pc = idx % pieces;
                cp_async16(rres + row * A.ksr + pc * 2, gR + int64_t(row) * A.dp + pc * 2);
            }
            cp_async_commit();
            cp_async_wait<0>();
            __syncthreads();
        }
        if (!RES) __syncthreads();  // previous J's epilogue is done with vjs
        if (tid < BM) vjs[tid] = A.v[J0 + tid];
        // published by the first mainloop barrier of this J
        double colacc[4][2];
#pragma unroll
        for (int ns = 0; ns < 4; ++ns) colacc[ns][0] = colacc[ns][1] = 0.0;

        const int itEnd = diag ? jt : nT - 1;
        for (int it = 0; it <= itEnd; ++it) {
            const int64_t I0 = rowBase + int64_t(it) * BM;
            double acc[MS][4][2];
#pragma unroll
            for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                for (int ns = 0; ns < 4; ++ns) acc[ms][ns][0] = acc[ms][ns][1] = 0.0;

            for (int kc = 0; kc < nk; ++kc, ++cs) {
                cp_async_wait<NSTAGE - 2>();
                __syncthreads();
                if (ps < total) {
                    issue(ps % NSTAGE);
                    advance();
                }
                cp_async_commit();
                ++ps;

                const double* sL = stages + (cs % NSTAGE) * STAGE_DOUBLES;
                const int nks = (min(KC, A.dp - kc * KC)) >> 2;
                const double* aBase = sL + (wm * WM + g) * KS + t4;
                const int bstride = RES ? A.ksr : KS;
                const double* bBase = RES ? rres + (wn * 32 + g) * A.ksr + t4 + kc * KC
                                          : sL + BM * KS + (wn * 32 + g) * KS + t4;
#pragma unroll
                for (int ks = 0; ks < KC / 4; ++ks) {
                    if (ks < nks) {
                        double af[MS], bf[4];
#pragma unroll
                        for (int ms = 0; ms < MS; ++ms) af[ms] = aBase[ms * 8 * KS + ks * 4];
#pragma unroll
                        for (int ns = 0; ns < 4; ++ns) bf[ns] = bBase[ns * 8 * bstride + ks * 4];
#pragma unroll
                        for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                            for (int ns = 0; ns < 4; ++ns)
                                dmma884(acc[ms][ns][0], acc[ms][ns][1], af[ms], bf[ns]);
                    }
                }
            }

            // ---- epilogue: exp, row sums, column sums
            const bool dtile = diag && (it == jt);
            double vi[MS];
#pragma unroll
            for (int ms = 0; ms < MS; ++ms) vi[ms] = A.v[I0 + wm * WM + ms * 8 + g];
            double vj[4][2];
#pragma unroll
            for (int ns = 0; ns < 4; ++ns) {
                const double2 p2 = *reinterpret_cast<const double2*>(vjs + wn * 32 + ns * 8 + 2 * t4);
                vj[ns][0] = p2.x;
                vj[ns][1] = p2.y;
            }
            double rowp[MS];
            tile_epilogue<EXPMODE, MS>(acc, vi, vj, colacc, rowp, dtile, wm * WM, wn * 32, g, t4, A.ec, tab);
#pragma unroll
            for (int ms = 0; ms < MS; ++ms) {
                double r = rowp[ms];
                r += __shfl_xor_sync(0xffffffffu, r, 1);
                r += __shfl_xor_sync(0xffffffffu, r, 2);
                if (t4 == 0) scr_row[wn * BM + wm * WM + ms * 8 + g] = r;
            }
            __syncthreads();
            if (tid < BM) {
                rowacc[it * BM + tid] += ((scr_row[tid] + scr_row[BM + tid]) + scr_row[2 * BM + tid]) +
                                         scr_row[3 * BM + tid];
            }
            // scr_row is rewritten only after the next tile's mainloop barriers.
        }

        // ---- column sums of this J tile: reduce over g, then over the two M warps
#pragma unroll
        for (int ns = 0; ns < 4; ++ns)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double c = colacc[ns][h];
                c += __shfl_xor_sync(0xffffffffu, c, 4);
                c += __shfl_xor_sync(0xffffffffu, c, 8);
                c += __shfl_xor_sync(0xffffffffu, c, 16);
                if (g == 0) scr_col[wm * BM + wn * 32 + ns * 8 + 2 * t4 + h] = c;
            }
        __syncthreads();
        if (tid < BM) {
            double c = scr_col[tid];
#pragma unroll
            for (int w = 1; w < WGM; ++w) c += scr_col[w * BM + tid];
            if (diag) {
                rowacc[jt * BM + tid] += c;
            } else {
                A.part[int64_t(sa) * A.n_pad + J0 + tid] = c;
            }
        }
        // scr_col is rewritten only after the next J's mainloop barriers.
    }
    __syncthreads();
    double* dst = A.part + int64_t(sb) * A.n_pad + rowBase;
    for (int i = tid; i < A.st; i += NTHREADS) dst[i] = rowacc[i];
}

// ---------------------------------------------------------------------------------
// v3: two decoupled warp groups.  Group gr (= warp / 4) owns rows [64 gr, 64 gr + 64)
// of every 128-row I tile, warp wn (= warp % 4) columns [32 wn, 32 wn + 32) of the
// J tile, so warps w and w + 4 share an SM sub-partition.  Each group streams its own
// half of L through its own 4-stage cp.async pipeline and synchronises with a named
// barrier of 128 threads; R_J is resident and shared (CTA-wide barrier only at J
// boundaries).  Group 1 starts every J sweep half a mainloop behind group 0, so the
// latency-bound exp epilogue of one group overlaps the DMMA mainloop of the other —
// DMMA and DFMA share one FP64 datapath, and this fills its idle epilogue cycles.
// Arithmetic (per element and per reduction) is identical to the 8-warp kernel.
template <int EXPMODE>
__global__ void __launch_bounds__(256, 1) gauss_matvec_grouped_kernel(const MatvecArgs A) {
    constexpr int MS = 8, WM = 64, GT = 128, NSTG = 4;
    constexpr int GSTAGE = WM * KS;
    extern __shared__ __align__(16) double smem[];
    double* rres = smem;                                  // BM * ksr
    double* gst = rres + BM * A.ksr;                      // 2 groups x NSTG x GSTAGE
    double* rowacc = gst + 2 * NSTG * GSTAGE;             // st
    double* scr_row = rowacc + A.st;                      // 2 groups x 4 x WM
    double* scr_col = scr_row + 2 * 4 * WM;               // 2 x BM
    double* tab = scr_col + 2 * BM;                       // 64
    double* vjs = tab + 64;                               // BM

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gr = warp >> 2, wn = warp & 3;
    const int gtid = tid & (GT - 1);
    const int g = lane >> 2, t4 = lane & 3;
    const int bar_id = 1 + gr;

    const int2 tile = A.tiles[blockIdx.x];
    const int sa = tile.x, sb = tile.y;
    const bool diag = (sa == sb);
    const int nT = A.st / BM;
    const int64_t rowBase = int64_t(sa) * A.st;
    const int64_t colBase = int64_t(sb) * A.st;
    const int nk = (A.dp + KC - 1) / KC;
    const int ntiles = diag ? nT * (nT + 1) / 2 : nT * nT;
    const int total = ntiles * nk;
    const int sig_kc = (nk - 1) / 2;  // group 0 releases group 1 after this chunk

    for (int i = tid; i < A.st; i += 256) rowacc[i] = 0.0;
    if (EXPMODE == 1 && tid < 64) tab[tid] = A.exp_tab[tid];

    double* mystages = gst + gr * NSTG * GSTAGE;
    int p_it = 0, p_jt = 0, p_kc = 0;
    auto issue = [&](int slot) {
        double* sL = mystages + slot * GSTAGE;
        const int k0 = p_kc * KC;
        const int pieces = min(KC, A.dp - k0) >> 1;
        const double* gL = A.L + (rowBase + int64_t(p_it) * BM + gr * WM) * A.dp + k0;
#pragma unroll
        for (int q = 0; q < (WM * (KC / 2)) / GT; ++q) {
            const int idx = gtid + q * GT;
            const int row = idx / (KC / 2), pc = idx % (KC / 2);
            if (pc < pieces) cp_async16(sL + row * KS + pc * 2, gL + int64_t(row) * A.dp + pc * 2);
        }
    };
    auto advance = [&]() {
        if (++p_kc == nk) {
            p_kc = 0;
            ++p_it;
            if (p_it > (diag ? p_jt : nT - 1)) {
                p_it = 0;
                ++p_jt;
            }
        }
    };
    int ps = 0;
#pragma unroll
    for (int s2 = 0; s2 < NSTG - 1; ++s2) {
        if (ps < total) {
            issue(ps % NSTG);
            advance();
        }
        cp_async_commit();
        ++ps;
    }

    int cs = 0;
    for (int jt = 0; jt < nT; ++jt) {
        const int64_t J0 = colBase + int64_t(jt) * BM;
        __syncthreads();  // everyone is done with the previous R_J, vjs, scr_col
        {
            const int pieces = A.dp >> 1;
            const double* gR = A.R + J0 * A.dp;
            for (int idx = tid; idx < BM * pieces; idx += 256) {
                const int row = idx / pieces, pc = idx % pieces;
                cp_async16(rres + row * A.ksr + pc * 2, gR + int64_t(row) * A.dp + pc * 2);
            }
            cp_async_commit();
            cp_async_wait<0>();
        }
        if (tid < BM) vjs[tid] = A.v[J0 + tid];
        __syncthreads();

        double colacc[4][2];
#pragma unroll
        for (int ns = 0; ns < 4; ++ns) colacc[ns][0] = colacc[ns][1] = 0.0;
        if (gr == 1) named_bar_sync(3, 256);  // phase offset: wait for group 0's signal

        const int itEnd = diag ? jt : nT - 1;
        for (int it = 0; it <= itEnd; ++it) {
            const int64_t I0 = rowBase + int64_t(it) * BM;
            double acc[MS][4][2];
#pragma unroll
            for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                for (int ns = 0; ns < 4; ++ns) acc[ms][ns][0] = acc[ms][ns][1] = 0.0;

            for (int kc = 0; kc < nk; ++kc, ++cs) {
                cp_async_wait<NSTG - 2>();
                named_bar_sync(bar_id, GT);
                if (ps < total) {
                    issue(ps % NSTG);
                    advance();
                }
                cp_async_commit();
                ++ps;

                const double* sL = mystages + (cs % NSTG) * GSTAGE;
                const int nks = (min(KC, A.dp - kc * KC)) >> 2;
                const double* aBase = sL + g * KS + t4;
                const double* bBase = rres + (wn * 32 + g) * A.ksr + t4 + kc * KC;
#pragma unroll
                for (int ks = 0; ks < KC / 4; ++ks) {
                    if (ks < nks) {
                        double af[MS], bf[4];
#pragma unroll
                        for (int ms = 0; ms < MS; ++ms) af[ms] = aBase[ms * 8 * KS + ks * 4];
#pragma unroll
                        for (int ns = 0; ns < 4; ++ns) bf[ns] = bBase[ns * 8 * A.ksr + ks * 4];
#pragma unroll
                        for (int ms = 0; ms < MS; ++ms)
#pragma unroll
                            for (int ns = 0; ns < 4; ++ns)
                                dmma884(acc[ms][ns][0], acc[ms][ns][1], af[ms], bf[ns]);
                    }
                }
                if (gr == 0 && it == 0 && kc == sig_kc) named_bar_arrive(3, 256);
            }

            const bool dtile = diag && (it == jt);
            double vi[MS];
#pragma unroll
            for (int ms = 0; ms < MS; ++ms) vi[ms] = A.v[I0 + gr * WM + ms * 8 + g];
            double vj[4][2];
#pragma unroll
            for (int ns = 0; ns < 4; ++ns) {
                const double2 p2 = *reinterpret_cast<const double2*>(vjs + wn * 32 + ns * 8 + 2 * t4);
                vj[ns][0] = p2.x;
                vj[ns][1] = p2.y;
            }
            double rowp[MS];
            tile_epilogue<EXPMODE, MS>(acc, vi, vj, colacc, rowp, dtile, gr * WM, wn * 32, g, t4, A.ec, tab);
#pragma unroll
            for (int ms = 0; ms < MS; ++ms) {
                double r = rowp[ms];
                r += __shfl_xor_sync(0xffffffffu, r, 1);
                r += __shfl_xor_sync(0xffffffffu, r, 2);
                if (t4 == 0) scr_row[(gr * 4 + wn) * WM + ms * 8 + g] = r;
            }
            named_bar_sync(bar_id, GT);
            if (gtid < WM) {
                const double* sr = scr_row + gr * 4 * WM + gtid;
                rowacc[it * BM + gr * WM + gtid] += ((sr[0] + sr[WM]) + sr[2 * WM]) + sr[3 * WM];
            }
            // scr_row[gr] is rewritten only after the group's next chunk barrier.
        }

#pragma unroll
        for (int ns = 0; ns < 4; ++ns)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                double c = colacc[ns][h];
                c += __shfl_xor_sync(0xffffffffu, c, 4);
                c += __shfl_xor_sync(0xffffffffu, c, 8);
                c += __shfl_xor_sync(0xffffffffu, c, 16);
                if (g == 0) scr_col[gr * BM + wn * 32 + ns * 8 + 2 * t4 + h] = c;
            }
        __syncthreads();
        if (tid < BM) {
            const double c = scr_col[tid] + scr_col[BM + tid];
            if (diag) {
                rowacc[jt * BM + tid] += c;
            } else {
                A.part[int64_t(sa) * A.n_pad + J0 + tid] = c;
            }
        }
    }
    __syncthreads();
    double* dst = A.part + int64_t(sb) * A.n_pad + rowBase;
    for (int i = tid; i < A.st; i += 256) dst[i] = rowacc[i];
}

// out_i = sum_x part[x][i] (owned slots only) + (K_ii + lambda) v_i  (diag, rank 0);
// K_ii = 1 for the Gaussian kernel (kernels.cpp:81), kdiag[i] for the polynomial kernel.
__global__ void matvec_finish_kernel(const double* __restrict__ part, int ns_count, int64_t n_pad,
                                     int64_t n, int st, const uint8_t* __restrict__ owned,
                                     const double* __restrict__ v, double lambda, int add_diag,
                                     const double* __restrict__ kdiag, double* __restrict__ out) {
    for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n_pad;
         i += int64_t(gridDim.x) * blockDim.x) {
        if (i >= n) {
            out[i] = 0.0;
            continue;
        }
        const int y = int(i / st);
        double s = 0.0;
        for (int x = 0; x < ns_count; ++x)
            if (!owned || owned[int64_t(x) * ns_count + y]) s += part[int64_t(x) * n_pad + i];
        if (add_diag) {
            const double vi = v[i];
            s = (s + (kdiag ? kdiag[i] * vi : vi)) + lambda * vi;
        }
        out[i] = s;
    }
}

int resident_stride(int dp) {
    int k = dp;
    while (k % 16 != 4 && k % 16 != 12) k += 4;
    return k;
}

template <bool RES>
size_t smem_bytes(int st, int dp) {
    // scratch sized for the widest warp layout (WGM = 4)
    return sizeof(double) * (size_t(RES ? BM * resident_stride(dp) : 0) +
                             size_t(Shape<RES>::NSTAGE) * Shape<RES>::STAGE_DOUBLES + st + WGN * BM +
                             4 * BM + 64 + BM);
}

template <int EXPMODE, bool RES, int MS>
void launch_variant(const MatvecArgs& a, int64_t ntiles, cudaStream_t stream) {
    const size_t smem = smem_bytes<RES>(a.st, a.dp);
    KRR_CUDA(cudaFuncSetAttribute(gauss_matvec_kernel<EXPMODE, RES, MS>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    gauss_matvec_kernel<EXPMODE, RES, MS><<<unsigned(ntiles), Warps<MS>::NT, smem, stream>>>(a);
}

template <int EXPMODE, int MS>
void launch_ms(const MatvecArgs& a, int64_t ntiles, bool res, cudaStream_t stream) {
    if (res)
        launch_variant<EXPMODE, true, MS>(a, ntiles, stream);
    else
        launch_variant<EXPMODE, false, MS>(a, ntiles, stream);
}

size_t grouped_smem_bytes(int st, int dp) {
    return sizeof(double) * (size_t(BM) * resident_stride(dp) + size_t(2) * 4 * 64 * KS + st +
                             2 * 4 * 64 + 2 * BM + 64 + BM);
}

template <int EXPMODE>
void launch_grouped(const MatvecArgs& a, int64_t ntiles, cudaStream_t stream) {
    const size_t smem = grouped_smem_bytes(a.st, a.dp);
    KRR_CUDA(cudaFuncSetAttribute(gauss_matvec_grouped_kernel<EXPMODE>,
                                  cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    gauss_matvec_grouped_kernel<EXPMODE><<<unsigned(ntiles), 256, smem, stream>>>(a);
}

}  // namespace

size_t gauss_matvec_smem_bytes(int st) { return smem_bytes<false>(st, 0); }

bool gauss_matvec_resident_ok(int st, int dp) { return smem_bytes<true>(st, dp) <= size_t(MAX_SMEM); }

void gauss_matvec_launch(const GaussMatvecPlan& p, const double* v, double* part, int exp_mode,
                         cudaStream_t stream) {
    if (p.num_tiles == 0) return;
    MatvecArgs a;
    a.L = p.L;
    a.R = p.R;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.exp_tab = p.exp_tab;
    a.n_pad = p.n_pad;
    a.dp = p.dp;
    a.st = p.st;
    a.ksr = resident_stride(p.dp);
    a.ec = p.ec;
    // The resident shape pays one pipeline drain per column tile: only worth it for
    // long I sweeps (super-tiles of >= 1024 rows).
    const bool res = p.resident && p.st >= 1024 && gauss_matvec_resident_ok(p.st, p.dp);
    const bool grouped = res && p.grouped && !p.warps16 && grouped_smem_bytes(p.st, p.dp) <= size_t(MAX_SMEM);
    auto dispatch = [&](auto mode) {
        constexpr int M = decltype(mode)::value;
        if (grouped)
            launch_grouped<M>(a, p.num_tiles, stream);
        else if (p.warps16)
            launch_ms<M, 4>(a, p.num_tiles, res, stream);
        else
            launch_ms<M, 8>(a, p.num_tiles, res, stream);
    };
    if (exp_mode == 2)
        dispatch(std::integral_constant<int, 2>{});
    else if (exp_mode == kPolyModeBase + 1)
        dispatch(std::integral_constant<int, kPolyModeBase + 1>{});
    else if (exp_mode == kPolyModeBase + 2)
        dispatch(std::integral_constant<int, kPolyModeBase + 2>{});
    else if (exp_mode == kPolyModeBase + 3)
        dispatch(std::integral_constant<int, kPolyModeBase + 3>{});
    else if (exp_mode == kPolyModeBase + 4)
        dispatch(std::integral_constant<int, kPolyModeBase + 4>{});
    else if (exp_mode == 0)
        dispatch(std::integral_constant<int, 0>{});
    else
        dispatch(std::integral_constant<int, 1>{});
    KRR_LAUNCH_CHECK();
}

void matvec_finish_launch(const GaussMatvecPlan& p, const double* part, const double* v,
                          double lambda, int add_diag, double* out, cudaStream_t stream) {
    const int64_t blocks = std::min<int64_t>((p.n_pad + 255) / 256, 148 * 8);
    matvec_finish_kernel<<<unsigned(blocks), 256, 0, stream>>>(part, p.ns, p.n_pad, p.n, p.st,
                                                                p.owned, v, lambda, add_diag, p.kdiag, out);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
