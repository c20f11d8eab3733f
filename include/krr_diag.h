/* libkrr_diag.so — measurement tooling behind profiles/ (NOT the drop-in library).
 *
 * Micro-benchmarks of the B200 pipes the kernels' rooflines use, the tcgen05 mechanics probes
 * the INT8 / BF16 tensor-core kernels were built on, and the clock traces of the K1-I8 / K1T-I8
 * kernels (recorded by libkrr_b200.so when its "i8_debug" option has bit 2 set).  Status codes
 * are include/krr_b200.h's; krr_diag_last_error() describes the last failure on this thread. */
#ifndef KRR_DIAG_H
#define KRR_DIAG_H

#include <stdint.h>

#include "krr_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

const char* krr_diag_last_error(void);
/* results[9]: FP64 DMMA (mma.sync m8n8k4) TFLOP/s, DFMA TFLOP/s, interleaved DMMA + DFMA TFLOP/s,
 * Gaussian exp epilogue Gevals/s (libdevice exp), (table exp), SM count, SM clock MHz,
 * half the warps DMMA / half DFMA TFLOP/s, legacy IMMA (mma.sync s8) TOPS. */
int krr_diag_microbench(int device, double* results);
/* the K1 table exp (mode 1) or libdevice exp (mode 0) of exp(-max(0, d2) * scale), elementwise */
int krr_diag_gauss_exp(int device, const double* d2, int64_t n, double scale, int mode, double* out);
/* one-CTA tcgen05 kind::i8 GEMM C (128 x N, s32) = A (128 x K) B (N x K)^T, K % 32 == 0, K <= 256 */
int krr_diag_i8_gemm(int device, const int8_t* A, const int8_t* B, int32_t* C, int K, int N);
/* the same with BF16 inputs (kind::f16, fp32 TMEM accumulator), K elements, K % 16 == 0 */
int krr_diag_bf16_gemm(int device, const uint16_t* A, const uint16_t* B, float* C, int K, int N);
/* tcgen05.mma kind::i8 issue-rate and pipe-contention probes (modes: tools/mma_rate.py) */
int krr_diag_i8_mma_rate(int device, int N, int reps, int kbytes, int mode, double* cycles_per_mma);
int krr_diag_tmem_ld_rate(int device, int warps, int reps, double* bytes_per_clk);
int krr_diag_tmem_ld_under_mma(int device, int warps, int reps, double* bytes_per_clk, double* mma_cycles);
/* clock64 stamps of CTA 0 from the last K1-I8 / K1T-I8 launch run with i8_debug bit 2 */
int krr_diag_i8_trace(long long* out, int count);
int krr_diag_i8x_trace(long long* out, int count);
int krr_diag_i8t_trace(long long* out, int count);

#ifdef __cplusplus
}
#endif
#endif
