// Declarations of the diagnostics library's kernels (libkrr_diag.so only).
#pragma once
#include "kernels.cuh"

namespace krr {

// ---------------------------------------------------------------- diagnostics
// one-CTA tcgen05 kind::i8 GEMM probe: C (128 x N) = A (128 x K) B (N x K)^T, K % 32 == 0
void i8_probe_launch(const int8_t* A, const int8_t* B, int32_t* C, int K, int N, cudaStream_t stream);
// same with BF16 inputs (kind::f16, fp32 accumulate), K elements per row (K % 16 == 0)
void bf16_probe_launch(const uint16_t* A, const uint16_t* B, float* C, int K, int N, cudaStream_t stream);
// cycles per tcgen05.mma kind::i8 (M = 128, N, K = 32), one CTA per SM, back-to-back
double i8_mma_rate(int N, int reps, int kbytes, int mode, cudaStream_t stream);
double tmem_ld_rate(int warps, int reps, cudaStream_t stream);
double i8_tile_order_rate(int order, int tiles, cudaStream_t stream);
double fp64_under_mma(int op, int mma, int iters, cudaStream_t stream, double* mma_cycles = nullptr, int nwork = 4);
double tmem_ld_under_mma(int warps, int reps, cudaStream_t stream, double* mma_cycles);
double i8_mma_rate_pair(int N, int reps, cudaStream_t stream);
void debug_exp_launch(const double* d2, int64_t n, const ExpConsts& ec, const double* tab,
                      int mode, double* out, cudaStream_t stream);
// results: see krr_diag_microbench in include/krr_diag.h
void microbench_run(const ExpConsts& ec, const double* tab, double* results, cudaStream_t stream);

}  // namespace krr
