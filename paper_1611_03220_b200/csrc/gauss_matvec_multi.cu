// K1T — fused symmetric Gaussian mat-mat  OUT = (K + lambda I) V  for T right-hand sides
// (BASELINE config 5: t = 16 one-vs-all RLSC targets), K never stored.
//
// Same symmetric super-tile schedule, operands and exp epilogue as K1
// (gauss_matvec.cu), so every K_ij is the same bit pattern as in the single-column
// kernel.  After the exp, each 8 x 32 block of E (one m8 row block of a warp's tile)
// is re-laid-out with quad shuffles into DMMA A-fragments and contracted on the FP64
// tensor path against the T-wide operand tiles kept in shared memory:
//     rows:     O_I (8 x T)  = E_blk (8 x 32)    . V_J[32 cols x T]      (16 DMMA for T = 16)
//     columns:  O_J (32 x T) += E_blk^T (32 x 8) . V_I[8 rows x T]       (16 DMMA)
// i.e. 2T FP64 MACs per unordered pair on the DMMA pipe instead of 2T DFMAs.
//
// Reductions stay deterministic and atomic-free: per-tile row partials of the 4 column
// warps are summed in a fixed order through shared memory and accumulated (first write,
// then read-modify-write) into the CTA's private slot part[b][rows of a][T]; column
// partials accumulate in registers over the I sweep and land in part[a][rows of b][T].
// The finish kernel sums the NS slots of each row in fixed order.
//
// Layout: V, OUT and part are row-major with T interleaved columns (element (i, c) at
// i*T + c); rows >= n are zero.
#include <type_traits>

#include "common.cuh"
#include "gauss_exp.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int BM = 128;
constexpr int KC = 16;
constexpr int KS = 20;
constexpr int NSTAGE = 3;
constexpr int NT = 256;
constexpr int STAGE_DOUBLES = 2 * BM * KS;

struct MultiArgs {
    const double* __restrict__ L;
    const double* __restrict__ R;
    const double* __restrict__ v;   // n_pad x T
    double* __restrict__ part;      // NS x n_pad x T
    const int2* __restrict__ tiles;
    const double* __restrict__ exp_tab;
    int64_t n_pad;
    int dp;
    int st;
    ExpConsts ec;
};

__device__ __forceinline__ double shfl_d(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }

template <int T, int MODE>
__global__ void __launch_bounds__(NT, 1) gauss_matmat_kernel(const MultiArgs A) {
    constexpr int NTT = T / 8;  // n8 tiles of the RHS dimension
    // Row-major (row, T) tiles in shared memory with the column index XOR-swizzled by the row
    // parity when T = 16 (rows are 128 B = all 32 banks): the fragment reads of four
    // consecutive rows and the 8-row double2 stores then take the minimum number of
    // wavefronts (2 and 4) instead of 4 and 8 (ncu: 23 % of the shared-memory wavefronts
    // were bank conflicts at d = 440, t = 16).
    auto sw = [](int row, int col) { return row * T + (T == 16 ? (col ^ ((row & 1) << 3)) : col); };
    extern __shared__ __align__(16) double smem[];
    double* stages = smem;                                  // NSTAGE * STAGE_DOUBLES
    double* vjs = stages + NSTAGE * STAGE_DOUBLES;          // BM x T
    double* vis = vjs + BM * T;                             // BM x T
    double* scr = vis + BM * T;                             // 4 x BM x T
    double* tab = scr + 4 * BM * T;                         // 64

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp & 1, wn = warp >> 1;
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
    if (tid < 64) tab[tid] = A.exp_tab[tid];

    int p_it = 0, p_jt = 0, p_kc = 0;
    auto issue = [&](int slot) {
        double* sL = stages + slot * STAGE_DOUBLES;
        double* sR = sL + BM * KS;
        const int k0 = p_kc * KC;
        const int pieces = min(KC, A.dp - k0) >> 1;
        const double* gL = A.L + (rowBase + int64_t(p_it) * BM) * A.dp + k0;
        const double* gR = A.R + (colBase + int64_t(p_jt) * BM) * A.dp + k0;
#pragma unroll
        for (int q = 0; q < (2 * BM * (KC / 2)) / NT; ++q) {
            const int idx = tid + q * NT;
            const int op = idx / (BM * (KC / 2));
            const int rem = idx % (BM * (KC / 2));
            const int row = rem / (KC / 2), pc = rem % (KC / 2);
            if (pc < pieces) {
                const double* gp = (op ? gR : gL) + int64_t(row) * A.dp + pc * 2;
                cp_async16((op ? sR : sL) + row * KS + pc * 2, gp);
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
    int ps = 0;
#pragma unroll
    for (int s2 = 0; s2 < NSTAGE - 1; ++s2) {
        if (ps < total) {
            issue(ps % NSTAGE);
            advance();
        }
        cp_async_commit();
        ++ps;
    }

    int cs = 0;
    for (int jt = 0; jt < nT; ++jt) {
        const int64_t J0 = colBase + int64_t(jt) * BM;
        __syncthreads();  // previous J's users of vjs / scr are done
        for (int k = tid; k < BM * T; k += NT) vjs[sw(k / T, k % T)] = A.v[J0 * T + k];
        double colT[4][NTT][2];
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < NTT; ++nt) colT[mt][nt][0] = colT[mt][nt][1] = 0.0;

        const int itEnd = diag ? jt : nT - 1;
        for (int it = 0; it <= itEnd; ++it) {
            const int64_t I0 = rowBase + int64_t(it) * BM;
            double acc[8][4][2];
#pragma unroll
            for (int ms = 0; ms < 8; ++ms)
#pragma unroll
                for (int ns = 0; ns < 4; ++ns) acc[ms][ns][0] = acc[ms][ns][1] = 0.0;

            for (int kc = 0; kc < nk; ++kc, ++cs) {
                cp_async_wait<NSTAGE - 2>();
                __syncthreads();
                if (kc == 0)  // V_I for this tile (vis is free: last read before this barrier)
                    for (int k = tid; k < BM * T; k += NT) vis[sw(k / T, k % T)] = A.v[I0 * T + k];
                if (ps < total) {
                    issue(ps % NSTAGE);
                    advance();
                }
                cp_async_commit();
                ++ps;
                const double* sL = stages + (cs % NSTAGE) * STAGE_DOUBLES;
                const double* sR = sL + BM * KS;
                const int nks = (min(KC, A.dp - kc * KC)) >> 2;
                const double* aBase = sL + (wm * 64 + g) * KS + t4;
                const double* bBase = sR + (wn * 32 + g) * KS + t4;
#pragma unroll
                for (int ks = 0; ks < KC / 4; ++ks) {
                    if (ks < nks) {
                        double af[8], bf[4];
#pragma unroll
                        for (int ms = 0; ms < 8; ++ms) af[ms] = aBase[ms * 8 * KS + ks * 4];
#pragma unroll
                        for (int ns = 0; ns < 4; ++ns) bf[ns] = bBase[ns * 8 * KS + ks * 4];
#pragma unroll
                        for (int ms = 0; ms < 8; ++ms)
#pragma unroll
                            for (int ns = 0; ns < 4; ++ns)
                                dmma884(acc[ms][ns][0], acc[ms][ns][1], af[ms], bf[ns]);
                    }
                }
            }
            __syncthreads();  // vis written at kc == 0 is visible (also covers nk == 1)

            // ---- epilogue, one m8 row block at a time
            const bool dtile = diag && (it == jt);
#pragma unroll
            for (int ms = 0; ms < 8; ++ms) {
                const int il = wm * 64 + ms * 8 + g;
                double e[4][2];
#pragma unroll
                for (int ns = 0; ns < 4; ++ns)
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        double x = gauss_exp<MODE>(acc[ms][ns][h], A.ec, tab);
                        if (dtile) x = (wn * 32 + ns * 8 + 2 * t4 + h > il) ? x : 0.0;
                        e[ns][h] = x;
                    }
                // rows: O(8 x T) = E_blk(8 x 32) . V_J(32 x T)
                double oi[NTT][2];
#pragma unroll
                for (int nt = 0; nt < NTT; ++nt) oi[nt][0] = oi[nt][1] = 0.0;
#pragma unroll
                for (int kk = 0; kk < 8; ++kk) {
                    const int ns = kk >> 1, half = kk & 1;
                    const int src = g * 4 + half * 2 + (t4 >> 1);
                    const double v0 = shfl_d(e[ns][0], src), v1 = shfl_d(e[ns][1], src);
                    const double a = (t4 & 1) ? v1 : v0;  // E[g][ns*8 + half*4 + t4]
                    const int vr = wn * 32 + kk * 4 + t4;
#pragma unroll
                    for (int nt = 0; nt < NTT; ++nt) dmma884(oi[nt][0], oi[nt][1], a, vjs[sw(vr, g + nt * 8)]);
                }
#pragma unroll
                for (int nt = 0; nt < NTT; ++nt) {
                    double2 o2;
                    o2.x = oi[nt][0];
                    o2.y = oi[nt][1];
                    *reinterpret_cast<double2*>(scr + wn * BM * T + sw(wm * 64 + ms * 8 + g, nt * 8 + 2 * t4)) = o2;
                }
                // columns: O_J(32 x T) += E_blk^T(32 x 8) . V_I(8 x T)
#pragma unroll
                for (int mt = 0; mt < 4; ++mt)
#pragma unroll
                    for (int kk = 0; kk < 2; ++kk) {
                        const int src = (kk * 4 + t4) * 4 + (g >> 1);
                        const double v0 = shfl_d(e[mt][0], src), v1 = shfl_d(e[mt][1], src);
                        const double a = (g & 1) ? v1 : v0;  // E[kk*4 + t4][mt*8 + g]
                        const int vr = wm * 64 + ms * 8 + kk * 4 + t4;
#pragma unroll
                        for (int nt = 0; nt < NTT; ++nt)
                            dmma884(colT[mt][nt][0], colT[mt][nt][1], a, vis[sw(vr, g + nt * 8)]);
                    }
            }
            __syncthreads();
            // row partials: fixed-order sum over the 4 column warps, then into the CTA's slot
            {
                double* dst = A.part + (int64_t(sb) * A.n_pad + I0) * T;
                const bool first = diag ? (jt == it) : (jt == 0);
                for (int k = tid; k < BM * T; k += NT) {
                    const int q = sw(k / T, k % T);
                    const double s = ((scr[q] + scr[BM * T + q]) + scr[2 * BM * T + q]) + scr[3 * BM * T + q];
                    dst[k] = first ? s : dst[k] + s;
                }
            }
        }

        // column partials of J: reduce the two row warps in fixed order
        __syncthreads();
#pragma unroll
        for (int mt = 0; mt < 4; ++mt)
#pragma unroll
            for (int nt = 0; nt < NTT; ++nt) {
                double2 o2;
                o2.x = colT[mt][nt][0];
                o2.y = colT[mt][nt][1];
                *reinterpret_cast<double2*>(scr + wm * BM * T + sw(wn * 32 + mt * 8 + g, nt * 8 + 2 * t4)) = o2;
            }
        __syncthreads();
        {
            double* dst = A.part + (int64_t(sa) * A.n_pad + J0) * T;
            for (int k = tid; k < BM * T; k += NT) {
                const int q = sw(k / T, k % T);
                const double s = scr[q] + scr[BM * T + q];
                dst[k] = diag ? dst[k] + s : s;  // diag: the row partial of (jt, jt) is already there
            }
        }
    }
}

__global__ void matmat_finish_kernel(const double* __restrict__ part, int ns_count, int64_t n_pad, int64_t n,
                                     int st, int T, const uint8_t* __restrict__ owned,
                                     const double* __restrict__ v, double lambda, int add_diag,
                                     const double* __restrict__ kdiag, double* __restrict__ out) {
    const int64_t total = n_pad * T;
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < total;
         k += int64_t(gridDim.x) * blockDim.x) {
        const int64_t i = k / T;
        if (i >= n) {
            out[k] = 0.0;
            continue;
        }
        const int y = int(i / st);
        double s = 0.0;
        for (int x = 0; x < ns_count; ++x)
            if (!owned || owned[int64_t(x) * ns_count + y]) s += part[int64_t(x) * n_pad * T + k];
        if (add_diag) {
            const double vi = v[k];
            s = (s + (kdiag ? kdiag[i] * vi : vi)) + lambda * vi;
        }
        out[k] = s;
    }
}

template <int T>
size_t matmat_smem(int) {
    return sizeof(double) * (size_t(NSTAGE) * STAGE_DOUBLES + 2 * BM * T + 4 * BM * T + 64);
}

template <int T, int MODE>
void launch_matmat(const MultiArgs& a, int64_t ntiles, cudaStream_t stream) {
    const size_t smem = matmat_smem<T>(a.st);
    KRR_CUDA(cudaFuncSetAttribute(gauss_matmat_kernel<T, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  int(smem)));
    gauss_matmat_kernel<T, MODE><<<unsigned(ntiles), NT, smem, stream>>>(a);
}

}  // namespace

void gauss_matmat_launch(const GaussMatvecPlan& p, const double* v, int T, double* part, int mode,
                         cudaStream_t stream) {
    if (p.num_tiles == 0) return;
    MultiArgs a;
    a.L = p.L;
    a.R = p.R;
    a.v = v;
    a.part = part;
    a.tiles = p.tiles;
    a.exp_tab = p.exp_tab;
    a.n_pad = p.n_pad;
    a.dp = p.dp;
    a.st = p.st;
    a.ec = p.ec;
    auto by_mode = [&](auto tv) {
        constexpr int TT = decltype(tv)::value;
        switch (mode) {
            case 2: launch_matmat<TT, 2>(a, p.num_tiles, stream); break;
            case kPolyModeBase + 1: launch_matmat<TT, kPolyModeBase + 1>(a, p.num_tiles, stream); break;
            case kPolyModeBase + 2: launch_matmat<TT, kPolyModeBase + 2>(a, p.num_tiles, stream); break;
            case kPolyModeBase + 3: launch_matmat<TT, kPolyModeBase + 3>(a, p.num_tiles, stream); break;
            case kPolyModeBase + 4: launch_matmat<TT, kPolyModeBase + 4>(a, p.num_tiles, stream); break;
            default: launch_matmat<TT, 1>(a, p.num_tiles, stream);
        }
    };
    if (T == 8) {
        by_mode(std::integral_constant<int, 8>{});
    } else if (T == 16) {
        by_mode(std::integral_constant<int, 16>{});
    } else {
        fail(KRR_ERR_INVALID_ARGUMENT, "gauss_matmat: T must be 8 or 16");
    }
    KRR_LAUNCH_CHECK();
}

void matmat_finish_launch(const GaussMatvecPlan& p, const double* part, const double* v, int T,
                          double lambda, int add_diag, double* out, cudaStream_t stream) {
    const int64_t blocks = std::min<int64_t>((p.n_pad * T + 255) / 256, 148 * 8);
    matmat_finish_kernel<<<unsigned(blocks), 256, 0, stream>>>(part, p.ns, p.n_pad, p.n, p.st, T, p.owned, v,
                                                               lambda, add_diag, p.kdiag, out);
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
