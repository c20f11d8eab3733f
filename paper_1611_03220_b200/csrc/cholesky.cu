// K4 — Cholesky factor of the s x s Gram (numerics::cholesky, numerics.cpp:49-55: Eigen LLT, lower;
// a non-positive pivot -> NotPositiveDefinite), hand-written for the B200 FP64 tensor path.
//
// Blocked right-looking factorisation of the column-major lower triangle (element (i >= j) at
// G[j s + i], what K3-I8 writes and what K5 reads), panel width 64:
//   1. diag:   factor the 64 x 64 diagonal block in shared memory (one CTA; unblocked
//              right-looking; a pivot that is not > 0 or not finite sets the failure flag)
//   2. panel:  rows below it: L[i, J] = A[i, J] L_JJ^-T (one thread per row, forward substitution
//              against L_JJ in shared memory, the reference's division by the pivot)
//   3. update: the trailing lower triangle A[I, J'] -= L[I, J] L[J', J]^T, one CTA per 64 x 64
//              tile (I >= J'), K = 64 on DMMA m8n8k4 (8 warps x 8 accumulator tiles)
// Work s^3 / 6 FMAs, almost all in (3) (config 4: 9e10, config 5: 7e11); 3 launches per panel.
// The factor overwrites the lower triangle in place (the upper triangle is never touched).
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

constexpr int NB = 64;  // panel width

__global__ void __launch_bounds__(256) chol_diag_kernel(double* __restrict__ G, int64_t s, int64_t k0, int bw,
                                                        int* __restrict__ info) {
    __shared__ double D[NB][NB + 1];
    const int tid = threadIdx.x;
    for (int e = tid; e < NB * NB; e += 256) {
        const int c = e / NB, r = e % NB;  // consecutive threads: consecutive rows of one column
        D[r][c] = (r < bw && c < bw && r >= c) ? G[(k0 + c) * s + k0 + r] : 0.0;
    }
    __syncthreads();
    for (int c = 0; c < bw; ++c) {
        const double piv = D[c][c];
        const bool ok = piv > 0.0 && isfinite(piv);  // Eigen's LLT fails on a non-positive pivot
        if (!ok && tid == 0 && *info == 0) *info = int(k0 + c + 1);
        const double l = ok ? sqrt(piv) : 1.0;
        __syncthreads();
        if (tid == 0) D[c][c] = l;
        for (int r = c + 1 + tid; r < bw; r += 256) D[r][c] = D[r][c] / l;
        __syncthreads();
        const int m = bw - c - 1;  // trailing (r, q), c < q <= r < bw
        for (int e = tid; e < m * m; e += 256) {
            const int r = c + 1 + e / m, q = c + 1 + e % m;
            if (q <= r) D[r][q] = fma(-D[r][c], D[q][c], D[r][q]);
        }
        __syncthreads();
    }
    for (int e = tid; e < NB * NB; e += 256) {
        const int c = e / NB, r = e % NB;
        if (r < bw && c < bw && r >= c) G[(k0 + c) * s + k0 + r] = D[r][c];
    }
}

// rows i in [k1, s): x = a L_JJ^-T, i.e. x_c = (a_c - sum_{m<c} x_m L_cm) / L_cc
__global__ void __launch_bounds__(128) chol_panel_kernel(double* __restrict__ G, int64_t s, int64_t k0, int bw) {
    __shared__ double LJ[NB][NB + 1];
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
        const int c = e / NB, r = e % NB;
        LJ[r][c] = (r < bw && c < bw && r >= c) ? G[(k0 + c) * s + k0 + r] : (r == c ? 1.0 : 0.0);
    }
    __syncthreads();
    const int64_t i = k0 + bw + int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= s) return;
    double x[NB];
#pragma unroll
    for (int c = 0; c < NB; ++c) x[c] = c < bw ? G[(k0 + c) * s + i] : 0.0;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
        double a = x[c];
#pragma unroll
        for (int m = 0; m < c; ++m) a = fma(-x[m], LJ[c][m], a);
        x[c] = a / LJ[c][c];
    }
#pragma unroll
    for (int c = 0; c < NB; ++c)
        if (c < bw) G[(k0 + c) * s + i] = x[c];
}

// trailing update of the lower 64 x 64 tiles of rows/columns [k1, s): C -= P_I P_J^T, P = the
// panel's columns [k0, k1) (K = bw <= 64).  Tile t of the lower triangle: (ti >= tj).
constexpr int TLD = 64 + 4;  // smem row stride (doubles): DMMA fragment reads conflict-free
constexpr size_t UPD_SMEM = size_t(2) * NB * TLD * 8;
__global__ void __launch_bounds__(256) chol_update_kernel(double* __restrict__ G, int64_t s, int64_t k0, int bw) {
    extern __shared__ __align__(16) double upd_sm[];
    double (*PI)[TLD] = reinterpret_cast<double (*)[TLD]>(upd_sm);            // [m][i]
    double (*PJ)[TLD] = reinterpret_cast<double (*)[TLD]>(upd_sm + NB * TLD);  // [m][j]
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
    const int64_t t = blockIdx.x;
    int64_t ti = int64_t((sqrt(8.0 * double(t) + 1.0) - 1.0) * 0.5);
    while (ti * (ti + 1) / 2 > t) --ti;
    while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
    const int64_t tj = t - ti * (ti + 1) / 2;
    const int64_t k1 = k0 + bw;
    const int64_t I0 = k1 + ti * 64, J0 = k1 + tj * 64;
    for (int e = tid; e < NB * 64; e += 256) {
        const int m = e / 64, r = e % 64;
        PI[m][r] = (m < bw && I0 + r < s) ? G[(k0 + m) * s + I0 + r] : 0.0;
        PJ[m][r] = (m < bw && J0 + r < s) ? G[(k0 + m) * s + J0 + r] : 0.0;
    }
    __syncthreads();
    const int wr = warp >> 2, wc = warp & 3;  // warp tile: rows 32 wr .., columns 16 wc ..
    double acc[4][2][2];
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
    for (int kk = 0; kk < NB; kk += 4) {
        double av[4], bv[2];
#pragma unroll
        for (int a = 0; a < 4; ++a) av[a] = PI[kk + t4][wr * 32 + a * 8 + g];  // A[g][t4] = P[i][m]
#pragma unroll
        for (int b = 0; b < 2; ++b) bv[b] = PJ[kk + t4][wc * 16 + b * 8 + g];  // B[t4][g] = P[j][m]
#pragma unroll
        for (int a = 0; a < 4; ++a)
#pragma unroll
            for (int b = 0; b < 2; ++b) dmma884(acc[a][b][0], acc[a][b][1], av[a], bv[b]);
    }
#pragma unroll
    for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < 2; ++b)
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int64_t i = I0 + wr * 32 + a * 8 + g;
                const int64_t j = J0 + wc * 16 + b * 8 + 2 * t4 + e;
                if (i < s && j < s && i >= j) {
                    double* dst = G + j * s + i;
                    *dst = *dst - acc[a][b][e];
                }
            }
}

}  // namespace

// In-place Cholesky of the column-major lower triangle of G (s x s).  *info (device int) is
// set to 1 + the first failing pivot index (0: success).
void cholesky_launch(double* G, int64_t s, int* info, cudaStream_t stream) {
    KRR_CUDA(cudaMemsetAsync(info, 0, sizeof(int), stream));
    KRR_CUDA(cudaFuncSetAttribute(chol_update_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(UPD_SMEM)));
    for (int64_t k0 = 0; k0 < s; k0 += NB) {
        const int bw = int(std::min<int64_t>(NB, s - k0));
        chol_diag_kernel<<<1, 256, 0, stream>>>(G, s, k0, bw, info);
        KRR_LAUNCH_CHECK();
        const int64_t rest = s - k0 - bw;
        if (rest <= 0) break;
        chol_panel_kernel<<<unsigned((rest + 127) / 128), 128, 0, stream>>>(G, s, k0, bw);
        KRR_LAUNCH_CHECK();
        const int64_t nt = (rest + 63) / 64;
        chol_update_kernel<<<unsigned(nt * (nt + 1) / 2), 256, UPD_SMEM, stream>>>(G, s, k0, bw);
        KRR_LAUNCH_CHECK();
    }
}

}  // namespace krr
