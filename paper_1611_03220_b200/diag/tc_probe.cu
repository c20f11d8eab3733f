// Diagnostic: one-CTA tcgen05 kind::i8 GEMM  C (128 x N, s32) = A (128 x K) . B (N x K)^T
// through the helpers in tc_i8.cuh — validates the descriptor / TMEM mechanics the
// INT8-slice mat-vec relies on (tests/test_gpu_tc.py).
#include <type_traits>

#include "common.cuh"
#include "diag.cuh"
#include "tc_i8.cuh"

namespace krr {
namespace {

// BF16 = true: A (128 x K/2), B (N x K/2) are bf16 bit patterns (K = bytes per row), the
// MMA is kind::f16 with an fp32 accumulator and C receives fp32 bit patterns.
template <int N, bool BF16 = false>
__global__ void __launch_bounds__(128) i8_probe_kernel(const int8_t* __restrict__ A, const int8_t* __restrict__ B,
                                                       int32_t* __restrict__ C, int K) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint8_t* sA = sm;
    uint8_t* sB = sm + 128 * K;
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    for (int idx = tid; idx < 128 * K; idx += 128) sA[tc::kmajor_offset(idx / K, idx % K, 128)] = uint8_t(A[idx]);
    for (int idx = tid; idx < N * K; idx += 128) sB[tc::kmajor_offset(idx / K, idx % K, N)] = uint8_t(B[idx]);
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0) {
        const uint32_t idesc = BF16 ? tc::idesc_bf16(128, N) : tc::idesc_i8(128, N);
        for (int ks = 0; ks < K / 32; ++ks) {
            const uint64_t da = tc::smem_desc(tc::smem_u32(sA) + ks * 2 * (128 * 16), 128 * 16, 128);
            const uint64_t db = tc::smem_desc(tc::smem_u32(sB) + ks * 2 * (N * 16), N * 16, 128);
            if constexpr (BF16) tc::mma_f16(tmem, da, db, idesc, ks > 0 ? 1u : 0u);
            else tc::mma_i8(tmem, da, db, idesc, ks > 0 ? 1u : 0u);
        }
        tc::mma_commit(&mbar);
    }
    tc::mbar_wait(&mbar, 0);
    tc::fence_after();
    for (int c0 = 0; c0 < N; c0 += 16) {
        uint32_t r[16];
        tc::tmem_ld16(tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0), r);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) C[(warp * 32 + lane) * N + c0 + j] = int32_t(r[j]);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// MMA throughput: one CTA per SM issues `reps` back-to-back tcgen05.mma (M = 128, N, K = 32)
// on zero operands (no swizzle, K-major) into TMEM; cycles per MMA -> out[blockIdx.x].
// mode 0: SS, descriptors rebuilt per MMA, one accumulator
//      1: SS, hoisted descriptors, one accumulator
//      2: SS, hoisted, 8 MMAs per iteration into rotating accumulators
//      3: TS (A in TMEM), descriptors rebuilt per MMA
//      4: TS, hoisted, rotating accumulators
//      5: SS, hoisted, rotating accumulators and distinct A/B smem tiles per MMA
template <int N, int MODE>
__global__ void __launch_bounds__(128) i8_mma_rate_kernel(int reps, int kbytes, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + N) * kbytes; i += 128) sm[i] = 0;
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    // accumulators: D at columns [0, 256) for TS (A at 256..), [0, 512) otherwise
    constexpr int NACC_SS = (512 / N) < 8 ? (512 / N) : 8;
    constexpr int NACC_TS = (256 / N) < 8 ? ((256 / N) < 1 ? 1 : (256 / N)) : 8;
    constexpr int KB = 96;  // hoisted modes: 96 bytes per row
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_i8(128, N);
        const uint32_t a = tc::smem_u32(sm), b = tc::smem_u32(sm + 128 * kbytes);
        const long long t0 = clock64();
        if constexpr (MODE == 1 || MODE == 2 || MODE == 5) {
            const uint64_t da = tc::smem_desc(a, 128, uint32_t(KB) * 8);
            const uint64_t db = tc::smem_desc(b, 128, uint32_t(KB) * 8);
            tc::mma_i8(tmem, da, db, idesc, 0u);
            for (int r = 0; r < reps / 8; ++r) {
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t d = MODE == 1 ? tmem : tmem + uint32_t((u % NACC_SS) * N);
                    const uint64_t off = MODE == 5 ? uint64_t((u % (KB / 32)) * 16) : 0;
                    tc::mma_i8(d, da + off, db + off, idesc, 1u);
                }
            }
        } else if constexpr (MODE == 4) {
            const uint64_t db = tc::smem_desc(b, 128, uint32_t(KB) * 8);
            for (int r = 0; r < reps / 8; ++r) {
#pragma unroll
                for (int u = 0; u < 8; ++u)
                    tc::mma_i8_ts(tmem + uint32_t((u % NACC_TS) * N), tmem + 256u + uint32_t(u * 8), db, idesc, 1u);
            }
        } else if constexpr (MODE == 3) {
            for (int r = 0; r < reps; ++r) {
                const int ks = r % (kbytes / 32);
                const uint64_t db = tc::smem_desc(b + ks * 256, 128, uint32_t(kbytes) * 8);
                tc::mma_i8_ts(tmem, tmem + 256u + uint32_t((r & 7) * 8), db, idesc, r > 0 ? 1u : 0u);
            }
        } else {
            for (int r = 0; r < reps; ++r) {
                const int ks = r % (kbytes / 32);
                const uint64_t da = tc::smem_desc(a + ks * 256, 128, uint32_t(kbytes) * 8);
                const uint64_t db = tc::smem_desc(b + ks * 256, 128, uint32_t(kbytes) * 8);
                tc::mma_i8(tmem, da, db, idesc, r > 0 ? 1u : 0u);
            }
        }
        tc::mma_commit(&mbar);
        tc::mbar_wait(&mbar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// In-situ order of the K1-I8 tile: M = 128, N = 64, kp = 96 (3 K steps), 8 A slices and
// 8 B slices resident, 36 products accumulated into 8 TMEM groups of 64 columns.
// ORDER 0: group-major (c = 7..0, p = 0..c) as the kernel issues them; ORDER 1: A-slice
// major (p outer, q inner: consecutive MMAs share the A operand).  Cycles per MMA.
template <int ORDER>
__global__ void __launch_bounds__(128) i8_tile_order_kernel(int tiles, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    constexpr int KP = 96, TI = 128, TJ = 64;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < 8 * (TI + TJ) * KP; i += 128) sm[i] = uint8_t(i * 7);
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (tid == 0) {
        const uint32_t idesc = tc::idesc_i8(TI, TJ);
        const uint64_t dA0 = tc::smem_desc(tc::smem_u32(sm), 128, KP * 8);
        const uint64_t dB0 = tc::smem_desc(tc::smem_u32(sm + 8 * TI * KP), 128, KP * 8);
        const long long t0 = clock64();
        for (int t = 0; t < tiles; ++t) {
            if constexpr (ORDER == 3) {
                // K1-I8's 7-slice order (balanced 8-bit digits): c = 6..0, p = 0..c, 3 K steps, 84 MMAs
#pragma unroll
                for (int c = 6; c >= 0; --c)
#pragma unroll
                    for (int p = 0; p <= c; ++p)
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks)
                            tc::mma_i8(tmem + uint32_t(c * TJ), dA0 + uint64_t((p * TI * KP + ks * 256) >> 4),
                                       dB0 + uint64_t(((c - p) * TJ * KP + ks * 256) >> 4), idesc,
                                       (p == 0 && ks == 0) ? 0u : 1u);
            } else if constexpr (ORDER == 2) {
                // K1T-I8's chunk order and layout: one 48 KB stage ([p][128 x 32 B] A, [p][64 x 32 B] B,
                // LBO 128 B, SBO 256 B), 14 K chunks of 36 MMAs into the same 8 accumulators
                const uint64_t a2 = tc::smem_desc(tc::smem_u32(sm), 128, 256);
                const uint64_t b2 = tc::smem_desc(tc::smem_u32(sm + 8 * TI * 32), 128, 256);
                for (int ks = 0; ks < 14; ++ks)
#pragma unroll
                    for (int c = 7; c >= 0; --c)
#pragma unroll
                        for (int p = 0; p <= c; ++p)
                            tc::mma_i8(tmem + uint32_t(c * TJ), a2 + uint64_t((p * TI * 32) >> 4),
                                       b2 + uint64_t(((c - p) * TJ * 32) >> 4), idesc, (ks == 0 && p == 0) ? 0u : 1u);
            } else if constexpr (ORDER == 0) {
#pragma unroll
                for (int c = 7; c >= 0; --c)
#pragma unroll
                    for (int p = 0; p <= c; ++p)
#pragma unroll
                        for (int ks = 0; ks < 3; ++ks)
                            tc::mma_i8(tmem + uint32_t(c * TJ), dA0 + uint64_t((p * TI * KP + ks * 256) >> 4),
                                       dB0 + uint64_t(((c - p) * TJ * KP + ks * 256) >> 4), idesc,
                                       (p == 0 && ks == 0) ? 0u : 1u);
            } else {
#pragma unroll
                for (int p = 0; p < 8; ++p)
#pragma unroll
                    for (int ks = 0; ks < 3; ++ks)
#pragma unroll
                        for (int q = 0; q + p < 8; ++q)
                            tc::mma_i8(tmem + uint32_t((p + q) * TJ), dA0 + uint64_t((p * TI * KP + ks * 256) >> 4),
                                       dB0 + uint64_t((q * TJ * KP + ks * 256) >> 4), idesc,
                                       (q == 0 ? (ks == 0) : (p == 0 && ks == 0)) ? 0u : 1u);
            }
        }
        tc::mma_commit(&mbar);
        tc::mbar_wait(&mbar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = (t1 - t0);
    }
    tc::fence_before();
    __syncthreads();
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// Does tensor-core INT8 work slow the FP64 pipe?  Warps 4-7 run 8 independent DADD (OP 0)
// or DFMA (OP 1) chains for `iters` iterations; with MMA != 0, thread 0 meanwhile issues
// back-to-back tcgen05.mma kind::i8 (M = 128, N = 64, K = 32, SS) until they finish.
// Returns cycles of the FP64 loop (max over SMs).
template <int OP, bool MMA>
__global__ void __launch_bounds__(1024) fp64_under_mma_kernel(int iters, long long* out, double* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    __shared__ volatile int stop;
    __shared__ long long tmax;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + 64) * 96; i += blockDim.x) sm[i] = 0;
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
        stop = 0;
        tmax = 0;
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (MMA && tid == 0) {
        const uint32_t idesc = tc::idesc_i8(128, 64);
        const uint64_t da = tc::smem_desc(tc::smem_u32(sm), 128, 96 * 8);
        const uint64_t db = tc::smem_desc(tc::smem_u32(sm + 128 * 96), 128, 96 * 8);
        int r = 0;
        const long long m0 = clock64();
        while (!stop && r < (1 << 22)) {
#pragma unroll
            for (int u = 0; u < 8; ++u) tc::mma_i8(tmem + uint32_t(u * 64), da, db, idesc, 1u);
            r += 8;
            if ((r & 63) == 0) {  // keep the queue bounded
                tc::mma_commit(&mbar);
                tc::mbar_wait(&mbar, uint32_t(((r >> 6) - 1) & 1));
            }
        }
        // MMA cycles per instruction while the other warps ran (completed batches only)
        if (r >= 64) out[gridDim.x + blockIdx.x] = (long long)(double(clock64() - m0) / double(r & ~63) * 1000.0);
    } else if (warp >= 4 && !(OP == 6 && warp == 4) && !(OP == 7 && warp != 4)) {
        // OP 0 DADD, 1 DFMA (FP64 pipe); 2 FFMA (FP32), 3 IMAD (integer): 8 chains per thread;
        // OP 6: FFMA on the three SM sub-partitions the MMA warp does not use (warps 5-7);
        // OP 7: FFMA on the MMA warp's sub-partition only (warp 4)
        // OP 4: idle workers (sleep for ~iters x 32 clk) — the MMA-alone baseline of this harness
        if constexpr (OP == 4) {
            const long long s0 = clock64();
            while (clock64() - s0 < (long long)iters * 32) __nanosleep(200);
            const long long s1 = clock64();
            atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(s1 - s0));
            __syncwarp();
            if (tid == 128) stop = 1;
            tc::fence_before();
            __syncthreads();
            if (tid == 0) out[blockIdx.x] = tmax;
            if (warp == 0) tc::tmem_dealloc(tmem, 512);
            return;
        }
        if constexpr (OP == 5) {  // shared-memory reads (LDS.128, conflict-free) beside the MMAs
            const uint4* src = reinterpret_cast<const uint4*>(sm);
            uint32_t x = 0;
            const long long s0 = clock64();
            for (int it = 0; it < iters; ++it) {
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const uint4 q = src[((it * 8 + i) * 32 + (tid & 31)) & 1023];
                    x ^= q.x ^ q.y ^ q.z ^ q.w;
                }
            }
            const long long s1 = clock64();
            if (x == 0x9876u) sink[0] = double(x);
            atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(s1 - s0));
            __syncwarp();
            if (tid == 128) stop = 1;
            tc::fence_before();
            __syncthreads();
            if (tid == 0) out[blockIdx.x] = tmax;
            if (warp == 0) tc::tmem_dealloc(tmem, 512);
            return;
        }
        using T = std::conditional_t<(OP <= 1), double,
                                     std::conditional_t<(OP == 2 || OP >= 6), float, uint32_t>>;
        T a[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = T(1.0 + 1e-3 * (i + tid));
        const T b = OP == 3 ? T(12345) : T(1e-9), c = OP == 3 ? T(2654435761u) : T(0.999999);
        const long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if constexpr (OP == 0) a[i] = a[i] + b;
                else if constexpr (OP == 3) a[i] = a[i] * c + b;
                else a[i] = fma(a[i], c, b);
            }
        }
        const long long t1 = clock64();
        double s = 0;
#pragma unroll
        for (int i = 0; i < 8; ++i) s += double(a[i]);
        if (s == 1234.5) sink[0] = s;
        atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(t1 - t0));
        __syncwarp();
        if (tid == (OP == 6 ? 160 : 128)) stop = 1;
    }
    tc::fence_before();
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = tmax;
    if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// 2-SM MMA rate: clusters of 2 CTAs; the leader issues `reps` tcgen05.mma.cta_group::2
// kind::i8 (M = 256: 128 rows from each CTA's smem, N columns split N/2 per CTA) into
// rotating accumulators; cycles per instruction -> out[blockIdx.x] (both CTAs).
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128)
    i8_mma_rate_pair_kernel(int reps, long long* out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    constexpr int KB = 96;
    const int tid = threadIdx.x, warp = tid >> 5;
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;\n" : "=r"(rank));
    for (int i = tid; i < (128 + N / 2) * KB; i += 128) sm[i] = uint8_t(i * 7 + rank);
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(tc::smem_u32(&tbase)),
                     "r"(512u)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;\n" ::: "memory");
    }
    tc::fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    tc::fence_after();
    const uint32_t tmem = tbase;
    constexpr int NACC = (512 / N) < 8 ? (512 / N) : 8;
    long long t0 = clock64();
    if (rank == 0 && tid == 0) {
        // M = 256 (two CTAs), idesc M field = M >> 4
        const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | (uint32_t(N >> 3) << 17) | (uint32_t(256 >> 4) << 24);
        const uint64_t da = tc::smem_desc(tc::smem_u32(sm), 128, KB * 8);
        const uint64_t db = tc::smem_desc(tc::smem_u32(sm + 128 * KB), 128, KB * 8);
        for (int r = 0; r < reps / 8; ++r) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t off = uint64_t((u % 3) * 16);
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem + uint32_t((u % NACC) * N)),
                    "l"(da + off), "l"(db + off), "r"(idesc), "r"(1u));
            }
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n" ::"r"(
                tc::smem_u32(&mbar)),
            "h"((unsigned short)3)
            : "memory");
    }
    if (tid == 0) {
        tc::mbar_wait(&mbar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
    }
    tc::fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;\n" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(512u) : "memory");
}

// TMEM read throughput: `warps` warps per CTA (one CTA per SM) each issue `reps`
// tcgen05.ld.32x32b.x16 (+ wait) from their lane quarter; cycles -> out[blockIdx.x].
__global__ void tmem_ld_rate_kernel(int reps, long long* out, unsigned* sink) {
    __shared__ uint32_t tbase;
    __shared__ long long tmax;
    const int tid = threadIdx.x, warp = tid >> 5;
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    if (tid == 0) tmax = 0;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase + (uint32_t((warp & 3) * 32) << 16);
    unsigned x = 0;
    const long long t0 = clock64();
    for (int r = 0; r < reps; ++r) {
        uint32_t v[16];
        tc::tmem_ld16(tmem + uint32_t(((r * 16) + (warp >> 2) * 128) & 511), v);
        tc::tmem_wait_ld();
#pragma unroll
        for (int j = 0; j < 16; ++j) x ^= v[j];
    }
    const long long t1 = clock64();
    atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(t1 - t0));
    if (x == 0x12345u) sink[0] = x;
    tc::fence_before();
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = tmax;
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

// TMEM loads (tcgen05.ld.32x32b.x16 + wait) by `warps` warps from columns [256, 512) while
// one more warp issues back-to-back kind::i8 MMAs (M = 128, N = 64, K = 96 B) into columns
// [0, 256): does the accumulator traffic of the MMAs slow the loads (and vice versa)?
// out[b] = load cycles, out[148 + b] = MMA cycles / instruction x 1000.
__global__ void tmem_ld_under_mma_kernel(int reps, int warps, long long* out, unsigned* sink) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ __align__(8) uint64_t mbar;
    __shared__ uint32_t tbase;
    __shared__ volatile int stop;
    __shared__ long long tmax;
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int i = tid; i < (128 + 64) * 96; i += blockDim.x) sm[i] = 0;
    tc::fence_proxy_async();
    if (tid == 0) {
        tc::mbar_init(&mbar, 1);
        tc::mbar_fence_init();
        stop = 0;
        tmax = 0;
    }
    if (warp == 0) tc::tmem_alloc(&tbase, 512);
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tmem = tbase;
    if (warp == warps) {
        if ((tid & 31) == 0) {
            const uint32_t idesc = tc::idesc_i8(128, 64);
            const uint64_t da = tc::smem_desc(tc::smem_u32(sm), 128, 96 * 8);
            const uint64_t db = tc::smem_desc(tc::smem_u32(sm + 128 * 96), 128, 96 * 8);
            int r = 0;
            const long long m0 = clock64();
            while (!stop && r < (1 << 22)) {
#pragma unroll
                for (int u = 0; u < 8; ++u) tc::mma_i8(tmem + uint32_t((u & 3) * 64), da, db, idesc, 1u);
                r += 8;
                if ((r & 63) == 0) {
                    tc::mma_commit(&mbar);
                    tc::mbar_wait(&mbar, uint32_t(((r >> 6) - 1) & 1));
                }
            }
            if (r >= 64) out[gridDim.x + blockIdx.x] = (long long)(double(clock64() - m0) / double(r & ~63) * 1000.0);
        }
    } else {
        const uint32_t taddr = tmem + (uint32_t((warp & 3) * 32) << 16) + 256u;
        unsigned x = 0;
        const long long t0 = clock64();
        for (int r = 0; r < reps; ++r) {
            uint32_t v[16];
            tc::tmem_ld16(taddr + uint32_t(((r * 16) + (warp >> 2) * 64) & 255), v);
            tc::tmem_wait_ld();
#pragma unroll
            for (int j = 0; j < 16; ++j) x ^= v[j];
        }
        const long long t1 = clock64();
        atomicMax(reinterpret_cast<unsigned long long*>(&tmax), (unsigned long long)(t1 - t0));
        if (x == 0x12345u) sink[0] = x;
        __syncwarp();
        if (warp == 0 && (tid & 31) == 0) stop = 1;
    }
    tc::fence_before();
    __syncthreads();
    if (tid == 0) out[blockIdx.x] = tmax;
    if (warp == 0) tc::tmem_dealloc(tbase, 512);
}

}  // namespace

double i8_mma_rate(int N, int reps, int kbytes, int mode, cudaStream_t stream) {
    long long* d = nullptr;
    KRR_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
    const size_t smem = size_t(128 + N) * kbytes;
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<148, 128, smem, stream>>>(reps, kbytes, d);
    };
    auto by_mode = [&](auto n) {
        constexpr int NN = decltype(n)::value;
        switch (mode) {
            case 0: run(i8_mma_rate_kernel<NN, 0>); break;
            case 1: run(i8_mma_rate_kernel<NN, 1>); break;
            case 2: run(i8_mma_rate_kernel<NN, 2>); break;
            case 3: run(i8_mma_rate_kernel<NN, 3>); break;
            case 4: run(i8_mma_rate_kernel<NN, 4>); break;
            default: run(i8_mma_rate_kernel<NN, 5>); break;
        }
    };
    if (N == 16) by_mode(std::integral_constant<int, 16>{});
    else if (N == 32) by_mode(std::integral_constant<int, 32>{});
    else if (N == 64) by_mode(std::integral_constant<int, 64>{});
    else if (N == 128) by_mode(std::integral_constant<int, 128>{});
    else by_mode(std::integral_constant<int, 256>{});
    KRR_LAUNCH_CHECK();
    long long h[148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    double mx = 0;
    for (long long v : h) mx = std::max(mx, double(v));
    return mx / reps;
}

double i8_tile_order_rate(int order, int tiles, cudaStream_t stream) {
    long long* d = nullptr;
    KRR_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
    const size_t smem = size_t(8) * (128 + 64) * 96;
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<148, 128, smem, stream>>>(tiles, d);
    };
    if (order == 0) run(i8_tile_order_kernel<0>);
    else if (order == 1) run(i8_tile_order_kernel<1>);
    else if (order == 2) run(i8_tile_order_kernel<2>);
    else run(i8_tile_order_kernel<3>);
    KRR_LAUNCH_CHECK();
    long long h[148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    double mx = 0;
    for (long long v : h) mx = std::max(mx, double(v));
    return mx / (double(tiles) * (order == 2 ? 14.0 * 36.0 : (order == 3 ? 84.0 : 108.0)));
}

double fp64_under_mma(int op, int mma, int iters, cudaStream_t stream, double* mma_cycles, int nwork) {
    long long* d = nullptr;
    double* sink = nullptr;
    KRR_CUDA(cudaMalloc(&d, 2 * 148 * sizeof(long long)));
    KRR_CUDA(cudaMemsetAsync(d, 0, 2 * 148 * sizeof(long long), stream));
    KRR_CUDA(cudaMalloc(&sink, sizeof(double)));
    const size_t smem = size_t(128 + 64) * 96;
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<148, 32 * (4 + nwork), smem, stream>>>(iters, d, sink);
    };
    switch (op * 2 + (mma ? 1 : 0)) {
        case 0: run(fp64_under_mma_kernel<0, false>); break;
        case 1: run(fp64_under_mma_kernel<0, true>); break;
        case 2: run(fp64_under_mma_kernel<1, false>); break;
        case 3: run(fp64_under_mma_kernel<1, true>); break;
        case 4: run(fp64_under_mma_kernel<2, false>); break;
        case 5: run(fp64_under_mma_kernel<2, true>); break;
        case 6: run(fp64_under_mma_kernel<3, false>); break;
        case 7: run(fp64_under_mma_kernel<3, true>); break;
        case 9: run(fp64_under_mma_kernel<4, true>); break;
        case 10: run(fp64_under_mma_kernel<5, false>); break;
        case 11: run(fp64_under_mma_kernel<5, true>); break;
        case 13: run(fp64_under_mma_kernel<6, true>); break;
        default: run(fp64_under_mma_kernel<7, true>); break;
    }
    KRR_LAUNCH_CHECK();
    long long h[2 * 148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    cudaFree(sink);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = std::max(mx, double(h[i]));
    if (mma_cycles) {
        double sum = 0;
        for (int i = 148; i < 2 * 148; ++i) sum += double(h[i]) / 1000.0;
        *mma_cycles = sum / 148.0;
    }
    // FP64 lane-ops per clock per SM: 4 warps x 32 lanes x 8 chains x iters / cycles (op 5: LDS
    // bytes per clock per SM: 4 warps x 32 lanes x 8 x 16 B x iters / cycles)
    return (op == 5 ? 16.0 : 1.0) * double(nwork) * 32 * 8 * double(iters) / mx;
}

double i8_mma_rate_pair(int N, int reps, cudaStream_t stream) {
    long long* d = nullptr;
    KRR_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
    const size_t smem = size_t(128 + N / 2) * 96;
    auto run = [&](auto kern) {
        KRR_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        kern<<<148, 128, smem, stream>>>(reps, d);
    };
    if (N == 64) run(i8_mma_rate_pair_kernel<64>);
    else if (N == 128) run(i8_mma_rate_pair_kernel<128>);
    else run(i8_mma_rate_pair_kernel<256>);
    KRR_LAUNCH_CHECK();
    long long h[148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    double mx = 0;
    for (long long v : h) mx = std::max(mx, double(v));
    return mx / reps;
}

double tmem_ld_rate(int warps, int reps, cudaStream_t stream) {
    long long* d = nullptr;
    unsigned* sink = nullptr;
    KRR_CUDA(cudaMalloc(&d, 148 * sizeof(long long)));
    KRR_CUDA(cudaMalloc(&sink, sizeof(unsigned)));
    tmem_ld_rate_kernel<<<148, 32 * warps, 0, stream>>>(reps, d, sink);
    KRR_LAUNCH_CHECK();
    long long h[148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    cudaFree(sink);
    double mx = 0;
    for (int i = 0; i < 148; ++i) mx = std::max(mx, double(h[i]));
    // bytes per clock per SM: warps x reps x (32 lanes x 16 columns x 4 B) / cycles
    return double(warps) * reps * 2048.0 / mx;
}

void bf16_probe_launch(const uint16_t* A, const uint16_t* B, float* C, int Kel, int N, cudaStream_t stream) {
    const int K = 2 * Kel;  // bytes per row
    const size_t smem = size_t(128 + N) * K;
    const auto* a = reinterpret_cast<const int8_t*>(A);
    const auto* b = reinterpret_cast<const int8_t*>(B);
    auto* c = reinterpret_cast<int32_t*>(C);
    if (N == 32) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<32, true><<<1, 128, smem, stream>>>(a, b, c, K);
    } else if (N == 64) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<64, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<64, true><<<1, 128, smem, stream>>>(a, b, c, K);
    } else {
        fail(KRR_ERR_INVALID_ARGUMENT, "bf16 probe: N must be 32 or 64");
    }
    KRR_LAUNCH_CHECK();
}

void i8_probe_launch(const int8_t* A, const int8_t* B, int32_t* C, int K, int N, cudaStream_t stream) {
    const size_t smem = size_t(128 + N) * K;
    if (N == 32) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<32><<<1, 128, smem, stream>>>(A, B, C, K);
    } else if (N == 64) {
        KRR_CUDA(cudaFuncSetAttribute(i8_probe_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        i8_probe_kernel<64><<<1, 128, smem, stream>>>(A, B, C, K);
    } else {
        fail(KRR_ERR_INVALID_ARGUMENT, "i8 probe: N must be 32 or 64");
    }
    KRR_LAUNCH_CHECK();
}

}  // namespace krr

namespace krr {
// TMEM load bandwidth (B/clk/SM) of `warps` warps beside back-to-back INT8 MMAs; *mma_cycles
// receives the MMA's cycles per instruction meanwhile.
double tmem_ld_under_mma(int warps, int reps, cudaStream_t stream, double* mma_cycles) {
    long long* d = nullptr;
    unsigned* sink = nullptr;
    KRR_CUDA(cudaMalloc(&d, 2 * 148 * sizeof(long long)));
    KRR_CUDA(cudaMemsetAsync(d, 0, 2 * 148 * sizeof(long long), stream));
    KRR_CUDA(cudaMalloc(&sink, sizeof(unsigned)));
    const size_t smem = size_t(128 + 64) * 96;
    KRR_CUDA(cudaFuncSetAttribute(tmem_ld_under_mma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    tmem_ld_under_mma_kernel<<<148, 32 * (warps + 1), smem, stream>>>(reps, warps, d, sink);
    KRR_LAUNCH_CHECK();
    long long h[2 * 148];
    KRR_CUDA(cudaMemcpyAsync(h, d, sizeof(h), cudaMemcpyDeviceToHost, stream));
    KRR_CUDA(cudaStreamSynchronize(stream));
    cudaFree(d);
    cudaFree(sink);
    double mx = 0, sum = 0;
    for (int i = 0; i < 148; ++i) mx = std::max(mx, double(h[i]));
    for (int i = 148; i < 2 * 148; ++i) sum += double(h[i]) / 1000.0;
    if (mma_cycles) *mma_cycles = sum / 148.0;
    return double(warps) * reps * 2048.0 / mx;
}
}  // namespace krr
