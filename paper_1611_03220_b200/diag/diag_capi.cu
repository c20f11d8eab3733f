// C-ABI of the diagnostics library libkrr_diag.so (include/krr_diag.h): tensor-core and FP64
// micro-benchmarks, the tcgen05 mechanics probes and the K1-I8 / K1T-I8 clock traces behind
// profiles/.  Measurement tooling, not part of the drop-in library (libkrr_b200.so).
#include <algorithm>
#include <string>

#include "../../include/krr_diag.h"
#include "common.cuh"
#include "diag.cuh"

namespace krr {
namespace {

thread_local std::string g_diag_error;

// A stream on `device` for one diagnostic call.
struct DiagStream {
    cudaStream_t s = nullptr;
    explicit DiagStream(int device) {
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || device < 0 || device >= n) {
            cudaGetLastError();
            fail(KRR_ERR_CUDA, "CUDA device " + std::to_string(device) + " not available");
        }
        KRR_CUDA(cudaSetDevice(device));
        KRR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    }
    DiagStream(const DiagStream&) = delete;
    DiagStream& operator=(const DiagStream&) = delete;
    ~DiagStream() {
        if (s) {
            cudaStreamSynchronize(s);
            cudaStreamDestroy(s);
        }
    }
};

template <class T>
struct Buf {
    T* p = nullptr;
    explicit Buf(size_t n) { KRR_CUDA(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(T))); }
    Buf(const Buf&) = delete;
    Buf& operator=(const Buf&) = delete;
    ~Buf() {
        if (p) cudaFree(p);
    }
};

template <class F>
int guard(F&& f) {
    try {
        f();
        return KRR_OK;
    } catch (const Error& e) {
        g_diag_error = e.what();
        return e.status;
    } catch (const std::exception& e) {
        g_diag_error = e.what();
        return KRR_ERR_CUDA;
    }
}

}  // namespace
}  // namespace krr

using krr::fail;
using krr::guard;

extern "C" {

const char* krr_diag_last_error(void) { return krr::g_diag_error.c_str(); }

int krr_diag_microbench(int device, double* results) {
    return guard([&] {
        krr::DiagStream st(device);
        double tab[64];
        krr::make_exp_table(tab);
        krr::Buf<double> dt(64);
        KRR_CUDA(cudaMemcpy(dt.p, tab, sizeof(tab), cudaMemcpyHostToDevice));
        krr::microbench_run(krr::make_exp_consts(1.0 / 72.0), dt.p, results, st.s);
    });
}

int krr_diag_gauss_exp(int device, const double* d2, int64_t n, double scale, int mode, double* out) {
    return guard([&] {
        krr::DiagStream st(device);
        double tab[64];
        krr::make_exp_table(tab);
        krr::Buf<double> dt(64), din{size_t(n)}, dout{size_t(n)};
        KRR_CUDA(cudaMemcpyAsync(dt.p, tab, sizeof(tab), cudaMemcpyHostToDevice, st.s));
        KRR_CUDA(cudaMemcpyAsync(din.p, d2, sizeof(double) * size_t(n), cudaMemcpyHostToDevice, st.s));
        krr::debug_exp_launch(din.p, n, krr::make_exp_consts(scale), dt.p, mode, dout.p, st.s);
        KRR_CUDA(cudaMemcpyAsync(out, dout.p, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost, st.s));
        KRR_CUDA(cudaStreamSynchronize(st.s));
    });
}

int krr_diag_i8_gemm(int device, const int8_t* A, const int8_t* B, int32_t* C, int K, int N) {
    return guard([&] {
        if (K <= 0 || K % 32 != 0 || K > 256) fail(KRR_ERR_INVALID_ARGUMENT, "K must be a multiple of 32 <= 256");
        krr::DiagStream st(device);
        krr::Buf<int8_t> a(size_t(128 * K)), b(size_t(N * K));
        krr::Buf<int32_t> o(size_t(128 * N));
        KRR_CUDA(cudaMemcpyAsync(a.p, A, size_t(128 * K), cudaMemcpyHostToDevice, st.s));
        KRR_CUDA(cudaMemcpyAsync(b.p, B, size_t(N * K), cudaMemcpyHostToDevice, st.s));
        krr::i8_probe_launch(a.p, b.p, o.p, K, N, st.s);
        KRR_CUDA(cudaMemcpyAsync(C, o.p, sizeof(int32_t) * size_t(128 * N), cudaMemcpyDeviceToHost, st.s));
        KRR_CUDA(cudaStreamSynchronize(st.s));
    });
}

int krr_diag_bf16_gemm(int device, const uint16_t* A, const uint16_t* B, float* C, int K, int N) {
    return guard([&] {
        if (K <= 0 || K % 16 != 0 || K > 128) fail(KRR_ERR_INVALID_ARGUMENT, "K must be a multiple of 16 <= 128");
        krr::DiagStream st(device);
        krr::Buf<uint16_t> a(size_t(128 * K)), b(size_t(N * K));
        krr::Buf<float> o(size_t(128 * N));
        KRR_CUDA(cudaMemcpyAsync(a.p, A, sizeof(uint16_t) * size_t(128 * K), cudaMemcpyHostToDevice, st.s));
        KRR_CUDA(cudaMemcpyAsync(b.p, B, sizeof(uint16_t) * size_t(N * K), cudaMemcpyHostToDevice, st.s));
        krr::bf16_probe_launch(a.p, b.p, o.p, K, N, st.s);
        KRR_CUDA(cudaMemcpyAsync(C, o.p, sizeof(float) * size_t(128 * N), cudaMemcpyDeviceToHost, st.s));
        KRR_CUDA(cudaStreamSynchronize(st.s));
    });
}

int krr_diag_i8_mma_rate(int device, int N, int reps, int kbytes, int mode, double* cycles_per_mma) {
    return guard([&] {
        if (N != 16 && N != 32 && N != 64 && N != 128 && N != 256)
            fail(KRR_ERR_INVALID_ARGUMENT, "N must be 16/32/64/128/256");
        if (kbytes < 32 || kbytes % 32 != 0) fail(KRR_ERR_INVALID_ARGUMENT, "kbytes must be a multiple of 32");
        krr::DiagStream st(device);
        if (mode == 12) {  // 2-SM (cta_group::2) MMA, M = 256, N in {64, 128, 256}
            if (N != 64 && N != 128 && N != 256) fail(KRR_ERR_INVALID_ARGUMENT, "pair mode: N in {64, 128, 256}");
            *cycles_per_mma = krr::i8_mma_rate_pair(N, std::max(8, reps), st.s);
            return;
        }
        if (mode >= 8 && mode <= 11) {  // FP64 ops/clk/SM: 8 DADD, 9 DADD + MMA, 10 DFMA, 11 DFMA + MMA
            *cycles_per_mma = krr::fp64_under_mma((mode - 8) >> 1, (mode - 8) & 1, std::max(64, reps), st.s);
            return;
        }
        if (mode >= 13 && mode <= 16) {  // 13 FFMA, 14 FFMA + MMA, 15 IMAD, 16 IMAD + MMA (lane-ops/clk/SM)
            *cycles_per_mma = krr::fp64_under_mma(2 + ((mode - 13) >> 1), (mode - 13) & 1, std::max(64, reps), st.s);
            return;
        }
        if (mode >= 17 && mode <= 24 && mode != 23) {  // MMA cycles / instr beside 17 DADD, 18 DFMA, 19 FFMA,
            if (mode == 24) mode = 23;  // 20 IMAD, 21 idle, 22 LDS.128, 24 -> op 6 (FFMA off the MMA's SMSP)
            krr::fp64_under_mma(mode - 17, 1, std::max(64, reps), st.s, cycles_per_mma);
            return;
        }
        if (mode >= 26 && mode <= 29) {  // DFMA lane-ops/clk/SM with 16 (26, 27) or 8 (28, 29) worker warps
            const int nw = mode <= 27 ? 16 : 8;
            *cycles_per_mma = krr::fp64_under_mma(1, (mode - 26) & 1, std::max(64, reps), st.s, nullptr, nw);
            return;
        }
        if (mode == 25) {  // MMA cycles / instr beside FFMA on the MMA warp's own SMSP only (op 7)
            krr::fp64_under_mma(7, 1, std::max(64, reps), st.s, cycles_per_mma);
            return;
        }
        if (mode == 6 || mode == 7 || mode == 30 || mode == 31) {  // 31: K1-I8's 7-slice order (84 MMAs)  // in-situ K1-I8 tile order (N = 64, kp = 96), reps = tiles;
            // 30: K1T-I8's K-chunk order and stage layout (14 chunks x 36 MMAs, one resident stage)
            *cycles_per_mma = krr::i8_tile_order_rate(mode == 30 ? 2 : (mode == 31 ? 3 : mode - 6), std::max(1, reps), st.s);
            return;
        }
        if (reps < 8 || mode < 0 || mode > 5) fail(KRR_ERR_INVALID_ARGUMENT, "reps >= 8, mode in [0, 7]");
        if (size_t(128 + N) * size_t(kbytes) > 200 * 1024) fail(KRR_ERR_INVALID_ARGUMENT, "operands exceed smem");
        *cycles_per_mma = krr::i8_mma_rate(N, reps, kbytes, mode, st.s);
    });
}

int krr_diag_tmem_ld_rate(int device, int warps, int reps, double* bytes_per_clk) {
    return guard([&] {
        if (warps < 1 || warps > 32 || reps < 1) fail(KRR_ERR_INVALID_ARGUMENT, "warps in [1, 32], reps >= 1");
        krr::DiagStream st(device);
        *bytes_per_clk = krr::tmem_ld_rate(warps, reps, st.s);
    });
}

int krr_diag_tmem_ld_under_mma(int device, int warps, int reps, double* bytes_per_clk, double* mma_cycles) {
    return guard([&] {
        if (warps < 1 || warps > 16 || reps < 1) fail(KRR_ERR_INVALID_ARGUMENT, "warps in [1, 16], reps >= 1");
        krr::DiagStream st(device);
        *bytes_per_clk = krr::tmem_ld_under_mma(warps, reps, st.s, mma_cycles);
    });
}

int krr_diag_i8_trace(long long* out, int count) {
    return guard([&] { krr::i8_read_trace(out, count); });
}

int krr_diag_i8x_trace(long long* out, int count) {
    return guard([&] { krr::i8x_read_trace(out, count); });
}

int krr_diag_i8t_trace(long long* out, int count) {
    return guard([&] { krr::i8s_read_trace(out, count); });
}

}  // extern "C"
