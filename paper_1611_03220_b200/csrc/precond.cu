// K3-K6 support kernels: Gram diagonal ops, and the two
// HBM-bound GEMV passes of the Woodbury apply.
//
// Reference: RffMap::apply (sketches.cpp:37-41), build_preconditioner
// (precond.cpp:20-40), Preconditioner::apply (precond.cpp:10-13):
//     z = (r - U^T (U r)) / lambda_p,   U = L^-1 Z^T  (s x n).
// On the device U is stored as B = U^T (n x s row-major) — exactly the buffer the
// in-place TRSM over the row-major Z produces — so both passes stream B once:
//   pass 1 (gemvT):  W = B^T r   (column sums over row chunks, deterministic partials)
//   pass 2 (zrow):   z_i = (r_i - B[i].W) / lambda_p, with the r.z partial fused.
#include "common.cuh"
#include "kernels.cuh"

namespace krr {

namespace {

__global__ void diag_add_kernel(double* G, int64_t s, double add) {
    for (int64_t k = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; k < s;
         k += int64_t(gridDim.x) * blockDim.x)
        G[k * (s + 1)] += add;
}

__global__ void trace_kernel(const double* __restrict__ G, int64_t s, double* out) {
    __shared__ double scr[32];
    double acc = 0.0;
    for (int64_t k = threadIdx.x; k < s; k += blockDim.x) acc += G[k * (s + 1)];
    acc = block_sum(acc, scr);
    if (threadIdx.x == 0) *out = acc;
}

__global__ void diag_check_kernel(const double* __restrict__ G, int64_t s, double* out) {
    __shared__ double smin[256];
    __shared__ int sbad[256];
    double m = 1.0e308;
    int bad = 0;
    for (int64_t k = threadIdx.x; k < s; k += blockDim.x) {
        const double v = G[k * (s + 1)];
        if (!isfinite(v)) bad = 1;
        m = fmin(m, fabs(v));
    }
    smin[threadIdx.x] = m;
    sbad[threadIdx.x] = bad;
    __syncthreads();
    for (int o = blockDim.x / 2; o > 0; o >>= 1) {
        if (threadIdx.x < o) {
            smin[threadIdx.x] = fmin(smin[threadIdx.x], smin[threadIdx.x + o]);
            sbad[threadIdx.x] |= sbad[threadIdx.x + o];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        out[0] = smin[0];
        out[1] = sbad[0] ? 1.0 : 0.0;
    }
}

constexpr int GV_COLS_PER_THREAD = 4;
constexpr int GV_SLICE = 256 * GV_COLS_PER_THREAD;

__global__ void gemvT_partial_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                     const double* __restrict__ r, double* __restrict__ Wpart,
                                     int64_t rows_per_chunk) {
    const int64_t k0 = int64_t(blockIdx.x) * GV_SLICE + threadIdx.x;
    const int64_t i0 = int64_t(blockIdx.y) * rows_per_chunk;
    const int64_t i1 = min(n, i0 + rows_per_chunk);
    double acc[GV_COLS_PER_THREAD];
#pragma unroll
    for (int c = 0; c < GV_COLS_PER_THREAD; ++c) acc[c] = 0.0;
#pragma unroll 4
    for (int64_t i = i0; i < i1; ++i) {
        const double ri = r[i];
        const double* row = B + i * s;
#pragma unroll
        for (int c = 0; c < GV_COLS_PER_THREAD; ++c) {
            const int64_t k = k0 + c * 256;
            if (k < s) acc[c] = fma(row[k], ri, acc[c]);
        }
    }
#pragma unroll
    for (int c = 0; c < GV_COLS_PER_THREAD; ++c) {
        const int64_t k = k0 + c * 256;
        if (k < s) Wpart[int64_t(blockIdx.y) * s + k] = acc[c];
    }
}

// W[k] = sum_c Wpart[c][k]: one block per 32 columns, lane <-> column (coalesced rows);
// warp w sums a contiguous range of chunks in order (loads unrolled ahead of the adds), then
// the 8 warp sums are combined in order — a blocked forward sum over the rows of U^T:
// deterministic, close to the reference's sequential order, no long per-thread load chain.
__global__ void reduce_rows_kernel(const double* __restrict__ Wpart, int nchunks, int64_t s,
                                   double* __restrict__ W) {
    __shared__ double part[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t k = int64_t(blockIdx.x) * 32 + lane;
    const int per = (nchunks + 7) / 8;
    const int c0 = warp * per, c1 = min(nchunks, c0 + per);
    double acc = 0.0;
    if (k < s) {
#pragma unroll 8
        for (int c = c0; c < c1; ++c) acc += Wpart[int64_t(c) * s + k];
    }
    part[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && k < s) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += part[w][lane];
        W[k] = t;
    }
}

template <bool SMEM_W>
__global__ void precond_z_kernel(const double* __restrict__ B, int64_t n, int64_t s,
                                 const double* __restrict__ Wg, const double* __restrict__ r,
                                 double lambda_p, double* __restrict__ z,
                                 double* __restrict__ rz_part) {
    extern __shared__ double wsm[];
    __shared__ double scr[32];
    const double* W = Wg;
    if constexpr (SMEM_W) {
        for (int64_t k = threadIdx.x; k < s; k += blockDim.x) wsm[k] = Wg[k];
        __syncthreads();
        W = wsm;
    }
    const int lane = threadIdx.x & 31;
    const int wpb = blockDim.x >> 5;
    const int64_t stride = int64_t(gridDim.x) * wpb;
    double rz = 0.0;
    for (int64_t i = int64_t(blockIdx.x) * wpb + (threadIdx.x >> 5); i < n; i += stride) {
        const double* row = B + i * s;
        double a0 = 0.0, a1 = 0.0;
        int64_t k = lane;
        for (; k + 32 < s; k += 64) {
            a0 = fma(row[k], W[k], a0);
            a1 = fma(row[k + 32], W[k + 32], a1);
        }
        if (k < s) a0 = fma(row[k], W[k], a0);
        const double dot = warp_sum(a0 + a1);
        const double ri = r[i];
        const double zi = (ri - dot) / lambda_p;
        if (lane == 0) {
            z[i] = zi;
            rz = fma(ri, zi, rz);
        }
    }
    rz = block_sum(rz, scr);
    if (threadIdx.x == 0) rz_part[blockIdx.x] = rz;
}

}  // namespace


void diag_add_launch(double* G, int64_t s, double add, cudaStream_t stream) {
    diag_add_kernel<<<unsigned((s + 255) / 256), 256, 0, stream>>>(G, s, add);
    KRR_LAUNCH_CHECK();
}

void trace_launch(const double* G, int64_t s, double* out, cudaStream_t stream) {
    trace_kernel<<<1, 256, 0, stream>>>(G, s, out);
    KRR_LAUNCH_CHECK();
}

void diag_check_launch(const double* G, int64_t s, double* out, cudaStream_t stream) {
    diag_check_kernel<<<1, 256, 0, stream>>>(G, s, out);
    KRR_LAUNCH_CHECK();
}

int gemvT_chunks(int64_t n, int64_t s) {
    const int64_t slices = (s + GV_SLICE - 1) / GV_SLICE;
    int64_t chunks = std::max<int64_t>(1, (148 * 4) / slices);
    chunks = std::min<int64_t>(chunks, std::max<int64_t>(1, n / 16));
    return int(chunks);
}

void gemvT_partial_launch(const double* B, int64_t n, int64_t s, const double* r, double* Wpart,
                          int nchunks, cudaStream_t stream) {
    const int64_t rows_per = (n + nchunks - 1) / nchunks;
    dim3 grid(unsigned((s + GV_SLICE - 1) / GV_SLICE), unsigned(nchunks));
    gemvT_partial_kernel<<<grid, 256, 0, stream>>>(B, n, s, r, Wpart, rows_per);
    KRR_LAUNCH_CHECK();
}

void reduce_rows_launch(const double* Wpart, int nchunks, int64_t s, double* W,
                        cudaStream_t stream) {
    const unsigned blocks = unsigned(std::max<int64_t>(1, (s + 31) / 32));
    reduce_rows_kernel<<<blocks, 256, 0, stream>>>(Wpart, nchunks, s, W);
    KRR_LAUNCH_CHECK();
}

int zrow_blocks(int64_t n) {
    return int(std::max<int64_t>(1, std::min<int64_t>((n + 7) / 8, 148 * 4)));
}

void precond_z_launch(const double* B, int64_t n, int64_t s, const double* W, const double* r,
                      double lambda_p, double* z, double* rz_part, int nb, cudaStream_t stream) {
    const size_t wbytes = size_t(s) * sizeof(double);
    if (wbytes <= 160 * 1024) {
        KRR_CUDA(cudaFuncSetAttribute(precond_z_kernel<true>,
                                      cudaFuncAttributeMaxDynamicSharedMemorySize, int(wbytes)));
        precond_z_kernel<true><<<nb, 256, wbytes, stream>>>(B, n, s, W, r, lambda_p, z, rz_part);
    } else {
        precond_z_kernel<false><<<nb, 256, 0, stream>>>(B, n, s, W, r, lambda_p, z, rz_part);
    }
    KRR_LAUNCH_CHECK();
}

}  // namespace krr
