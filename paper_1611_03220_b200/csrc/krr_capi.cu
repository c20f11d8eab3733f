// C-ABI implementation: device context, the device-resident PCG engine, the
// preconditioner build, and the NCCL plumbing.  See include/krr_b200.h for the
// reference interface each entry point replaces.
#include <cublas_v2.h>
#include <cusolverDn.h>
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <functional>
#include <memory>
#include <random>
#include <string>
#include <vector>

#include "common.cuh"
#include "host.hpp"
#include "kernels.cuh"

namespace krr {

namespace {

thread_local std::string g_last_error;

void cublas_check(cublasStatus_t st, const char* what) {
    if (st != CUBLAS_STATUS_SUCCESS)
        fail(KRR_ERR_CUDA, std::string(what) + ": cuBLAS status " + std::to_string(int(st)));
}
void cusolver_check(cusolverStatus_t st, const char* what) {
    if (st != CUSOLVER_STATUS_SUCCESS)
        fail(KRR_ERR_CUDA, std::string(what) + ": cuSOLVER status " + std::to_string(int(st)));
}
// NCCL is resolved lazily with dlopen("libnccl.so.2") and only when world > 1, so a
// single-GPU process never loads it and a process that already loaded an NCCL (e.g.
// torch's bundled one) shares that copy instead of mixing two versions.
struct NcclApi {
    ncclResult_t (*getUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*commInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*allReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    const char* (*getErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*commCount)(const ncclComm_t, int*) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.getUniqueId = reinterpret_cast<decltype(a.getUniqueId)>(dlsym(h, "ncclGetUniqueId"));
        a.commInitRank = reinterpret_cast<decltype(a.commInitRank)>(dlsym(h, "ncclCommInitRank"));
        a.allReduce = reinterpret_cast<decltype(a.allReduce)>(dlsym(h, "ncclAllReduce"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.getErrorString = reinterpret_cast<decltype(a.getErrorString)>(dlsym(h, "ncclGetErrorString"));
        a.commCount = reinterpret_cast<decltype(a.commCount)>(dlsym(h, "ncclCommCount"));
        return a;
    }();
    if (!api.getUniqueId || !api.commInitRank || !api.allReduce || !api.commDestroy)
        fail(KRR_ERR_NCCL, "libnccl.so.2 could not be loaded");
    return api;
}

void nccl_check(ncclResult_t st, const char* what) {
    if (st != ncclSuccess)
        fail(KRR_ERR_NCCL, std::string(what) + ": " +
                               (nccl().getErrorString ? nccl().getErrorString(st) : "nccl error"));
}

template <class T>
struct DevMem {
    T* p = nullptr;
    size_t count = 0;
    DevMem() = default;
    DevMem(const DevMem&) = delete;
    DevMem& operator=(const DevMem&) = delete;
    ~DevMem() { release(); }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        count = 0;
    }
    // returns true when the buffer was (re)allocated (its contents are then undefined)
    bool ensure(size_t n) {
        if (n <= count && p) return false;
        release();
        if (n == 0) return false;
        KRR_CUDA(cudaMalloc(&p, n * sizeof(T)));
        count = n;
        return true;
    }
    T* get() const { return p; }
};

// A set of CUDA events destroyed on scope exit (error paths included).
struct Events {
    std::vector<cudaEvent_t> e;
    explicit Events(size_t n) : e(n, nullptr) {
        try {
            for (auto& x : e) KRR_CUDA(cudaEventCreate(&x));
        } catch (...) {
            release();
            throw;
        }
    }
    Events(const Events&) = delete;
    Events& operator=(const Events&) = delete;
    ~Events() { release(); }
    void release() {
        for (auto& x : e)
            if (x) {
                cudaEventDestroy(x);
                x = nullptr;
            }
    }
    cudaEvent_t operator[](size_t i) const { return e[i]; }
};

struct PinnedScalars {
    double* p = nullptr;
    explicit PinnedScalars(size_t count = 16) { KRR_CUDA(cudaMallocHost(&p, count * sizeof(double))); }
    ~PinnedScalars() {
        if (p) cudaFreeHost(p);
    }
};

}  // namespace

struct Ctx {
    int device = 0, rank = 0, world = 1;
    cudaStream_t stream = nullptr;
    cublasHandle_t blas = nullptr;
    cusolverDnHandle_t sol = nullptr;
    ncclComm_t comm = nullptr;
    int exp_mode = 1;
    // Test-only single-GPU emulation of rank `emu_rank` of `emu_world` for the K1 / K1T
    // kernels (the B200_PROFILING rule: with fewer GPUs than ranks, emulate the ranks): the
    // schedule, owned slots and diagonal term of that rank, no collective — K v returns the
    // rank's partial sum.  Applied at krr_set_data; a single-rank context only.
    int emu_world = 1, emu_rank = 0;
    bool k1_resident = true;
    bool k1_warps16 = false;
    bool k1_grouped = true;

    // data
    bool has_data = false;
    int64_t n = 0, d = 0;
    double sigma = 1.0, scale = 0.5;
    // kernel family: 0 Gaussian, 1 polynomial (gamma x.z + offset)^degree
    int family = 0;
    double gamma = 1.0, offset = 0.0;
    int degree = 1;
    DevMem<double> kdiag;
    Schedule sched;
    GaussMatvecPlan plan;
    DevMem<double> X, L, R, part, exp_tab;
    DevMem<int2> tiles;
    DevMem<uint8_t> owned;
    // K1-I8 operands (int8 slices, row exponents, |x|^2)
    int k1_path = -1;  // -1 auto, 0 = FP64 DMMA, 1 = tcgen05 INT8 slices
    int i8_debug = 0; // profiling knob for K1-I8 (bit 0: skip MMAs, bit 1: skip exp phase)
    bool i8_ready = false;
    int kp8 = 0;
    DevMem<uint8_t> S8;
    DevMem<int> ex8, ejs8;
    DevMem<double> sq8;
    // K1-I8X operands (slices of z = sqrt(2 scale) x under one global exponent E, SQ_i = |z_i|^2/2
    // in fixed point); E = 0: not prepared or out of range (gauss_matvec_i8x.cu)
    int i8x_E = 0;
    DevMem<uint8_t> S8x;
    DevMem<long long> sq8x;
    // K1T-I8 operands (K-chunk-major slices for the multi-RHS kernel; prepared on first use)
    int k1t_path = -1;  // -1 auto, 0 = FP64 DMMA K1T, 1 = K1T-I8 (T = 16)
    int i8s_state = 0;  // 0 not prepared, 1 ready, -1 exponent range unsupported
    int kp8s = 0;
    DevMem<uint8_t> S8s;
    DevMem<int> ex8s, ejs8s;
    DevMem<double> sq8s;
    // K1-F32 operands (optional fp32 mode; prepared on first use)
    int precision = 64;  // 64: fp64 (oracle-matching); 32: fp32-accuracy K1
    bool f32_ready = false;
    DevMem<uint8_t> S32;
    DevMem<float> s32, v32;

    // PCG vectors (n_pad each) and reduction scratch
    DevMem<double> vin, vout, vx, vr, vz, vp, vap, vy, red, scal, mat_a, mat_b;
    std::unique_ptr<PinnedScalars> hscal;

    // preconditioner (row shard [z0, z1) of the n rows; world == 1 => all rows)
    bool has_sketch = false, has_pre = false;
    int64_t pn = 0, s = 0, z0 = 0, z1 = 0;
    double lambda_p = 1.0;
    double build_ms[3] = {0.0, 0.0, 0.0};  // last precond build: Z^T Z, Cholesky (+ retry), U = L^-1 Z^T
    // K3-I8 scratch (gram_i8.cu): one unit's slices, feature exponents, column maxima, flag, tile list
    DevMem<uint8_t> gscr;
    DevMem<int> gex, gbad;
    DevMem<unsigned long long> gmax;
    DevMem<int2> gtiles;
    DevMem<double> Z, G, Gcopy, W, Wpart, work, brff, wrff, wpad, chk;
    DevMem<int> info;

    int nb = 1;  // vector reduction blocks

    // batched multi-RHS state (n_pad x T interleaved blocks)
    bool batched = true;
    // single-RHS PCG with device operators runs as one CUDA graph: a conditional WHILE node whose
    // body is one iteration and a device-side stop decision (no host round trip per iteration)
    bool pcg_graph = true;
    bool poison_batched = false;  // test-only (krr_set_option "poison_batched")
    // test-only (krr_set_option "nccl_always"): run the collectives even on a one-rank
    // communicator (an identity all-reduce), so a single GPU exercises the multi-rank data path,
    // including NCCL kernels captured inside the graph-resident PCG loop
    bool nccl_always = false;
    DevMem<int> ctl;
    DevMem<double> dhist;
    DevMem<double> bx, br, bz, bp, bap, by, bin, bout, bpart, bred, bscal, bW;
    DevMem<int> bactive;
    std::unique_ptr<PinnedScalars> hscalT;
    int* hactive = nullptr;

    Ctx() = default;
    Ctx(const Ctx&) = delete;
    Ctx& operator=(const Ctx&) = delete;
    // Releases the handles on every path (also when a create call fails half way, e.g. in
    // ncclCommInitRank); the device buffers are freed by their own destructors afterwards.
    ~Ctx() {
        cudaSetDevice(device);
        if (stream) cudaStreamSynchronize(stream);
        if (comm) nccl().commDestroy(comm);
        if (sol) cusolverDnDestroy(sol);
        if (blas) cublasDestroy(blas);
        if (hactive) cudaFreeHost(hactive);
        if (stream) cudaStreamDestroy(stream);
    }

    void set_device() const { KRR_CUDA(cudaSetDevice(device)); }
    // the (world, rank) the K1 schedule is built for
    int k1_world() const { return world > 1 ? world : emu_world; }
    int k1_rank() const { return world > 1 ? rank : emu_rank; }
    void sync() const { KRR_CUDA(cudaStreamSynchronize(stream)); }
};

namespace {

// G (s x s, column-major lower triangle) = Z^T Z over `rows` rows of Z on K3-I8.
void gram_dev(Ctx& c, const double* Z, int64_t rows, int64_t s, double* G) {
    const int64_t sp = gram_i8_spad(s);
    c.gscr.ensure(gram_i8_scratch_bytes(rows, s));
    c.gex.ensure(size_t(sp));
    c.gmax.ensure(size_t(sp));
    c.gbad.ensure(1);
    c.gtiles.ensure(size_t((sp / 128) * (sp / 64)));
    gram_i8_launch(Z, rows, s, G, c.gscr.get(), c.gex.get(), c.gmax.get(), c.gbad.get(), c.gtiles.get(), c.stream);
}

void require_data(const Ctx& c) {
    if (!c.has_data) fail(KRR_ERR_STATE, "no data set on the context (call krr_set_data first)");
}

void allreduce_sum(Ctx& c, double* buf, int64_t count) {
    if (c.world <= 1 && !(c.nccl_always && c.comm)) return;
    nccl_check(nccl().allReduce(buf, buf, size_t(count), ncclDouble, ncclSum, c.comm, c.stream),
               "ncclAllReduce");
}

// K1 path selection: the INT8-slice tensor-core kernel where it is faster than the FP64
// DMMA kernel on B200 (measured: d >= ~48, profiles/README.md) and the data's exponent range
// allows it; the DMMA kernel otherwise.  Both are GPU kernels; neither is a fallback.
bool use_i8x(const Ctx& c);
bool use_i8(const Ctx& c) {
    if (!c.i8_ready || use_i8x(c)) return false;
    if (c.k1_path >= 0) return c.k1_path == 1;
    if (c.family != 0) {  // polynomial kernel (cheaper epilogue): profiles/r2_poly_k1_crossover_n65536.log
        const double dmma_ms = 2.22 + 0.1408 * double(c.d);
        const double i8_ms = c.kp8 <= 32 ? 6.91 : (c.kp8 <= 64 ? 7.36 : 7.75);
        return i8_ms < dmma_ms;  // K1-I8 for 37 <= d <= 96
    }
    // Cost model from the measured crossover (n = 65536, profiles/r2_k1_crossover_n65536_final.log, round 2's
    // final K1-I8: 28-product slices, TS-mode A operands, int64 tail, 4-column exp batches): the DMMA K1
    // grows linearly in its padded width dp = 4 ceil((d + 2) / 4), K1-I8 steps with the slice width
    // kp = 32 / 64 / 96.  K1-I8 for 27 <= d <= 96.
    const double dmma_ms = 3.72 + 0.1439 * double((c.d + 5) / 4 * 4);
    const double i8_ms = c.kp8 <= 32 ? 7.97 : (c.kp8 <= 64 ? 8.71 : 9.66);
    return i8_ms < dmma_ms;
}

// K1-I8X (integer exp argument under the next tile's MMAs, FP64 tail in a time-multiplexed
// phase; gauss_matvec_i8x.cu) on request (k1_path = 3) where the data's range allows it (1 <= E
// <= 8, Gaussian).  Measured at the speed of K1-I8 (profiles/README.md), so auto keeps K1-I8.
bool use_i8x(const Ctx& c) {
    return c.i8x_E > 0 && c.family == 0 && c.precision == 64 && c.k1_path == 3;
}

// K1-I8X operands: prepared when k1_path = 3 is requested (at krr_set_data, or by the option once
// data is set), outside any graph capture (the preparation reads E back to the host).
void i8x_ensure(Ctx& c) {
    c.i8x_E = 0;
    if (c.k1_path != 3 || c.family != 0 || !i8x_supported(c.d, int(c.sched.st))) return;
    const int64_t n_pad = c.plan.n_pad;
    c.S8x.ensure(size_t(8) * size_t(n_pad) * size_t(i8_kp(c.d)));
    c.sq8x.ensure(size_t(n_pad));
    c.i8x_E = i8x_prepare_launch(c.X.get(), c.n, c.d, n_pad, c.scale, c.S8x.get(), c.sq8x.get(), c.stream);
}

void f32_ensure(Ctx& c) {
    if (c.f32_ready) return;
    if (c.family != 0) fail(KRR_ERR_INVALID_ARGUMENT, "fp32 precision mode serves the Gaussian kernel only");
    if (!f32_supported(c.d, int(c.sched.st)))
        fail(KRR_ERR_INVALID_ARGUMENT, "fp32 precision mode supports d <= 128 (got d = " + std::to_string(c.d) + ")");
    const int kb = f32_kb(c.d);
    c.S32.ensure(size_t(3) * size_t(c.plan.n_pad) * size_t(kb));
    c.s32.ensure(size_t(c.plan.n_pad));
    c.v32.ensure(size_t(c.plan.n_pad));
    f32_prepare_launch(c.X.get(), c.n, c.d, c.plan.n_pad, c.L.get(), c.plan.dp, c.scale, c.S32.get(), c.s32.get(),
                       c.stream);
    c.f32_ready = true;
}

// out (n_pad) = (K + lambda I) v, v zero-padded to n_pad.  Replicated on all ranks.
void ensure_batched(Ctx& c, int T) {
    const size_t nt = size_t(c.plan.n_pad) * size_t(T);
    // K1T / K1T-I8 read the padded rows [n, n_pad) of their V operand and need them zero; the
    // Woodbury apply writes rows < n only, so every batched vector starts zeroed.
    for (auto* v : {&c.bx, &c.br, &c.bz, &c.bp, &c.bap, &c.by, &c.bin, &c.bout}) {
        if (v->ensure(nt)) KRR_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * v->count, c.stream));
        // test-only: all-ones bytes (NaN doubles) stand in for whatever a previous call left
        if (c.poison_batched) KRR_CUDA(cudaMemsetAsync(v->get(), 0xFF, sizeof(double) * v->count, c.stream));
    }
    c.bpart.ensure(size_t(c.sched.ns) * nt);
    c.bred.ensure(size_t(3) * 148 * 4 * 16);
    c.bscal.ensure(128);
    c.bactive.ensure(16);
    if (!c.hscalT) {
        c.hscalT = std::make_unique<PinnedScalars>(128);
        KRR_CUDA(cudaMallocHost(&c.hactive, 16 * sizeof(int)));
    }
}

// K1T path selection: the tcgen05 INT8-slice kernel (K1T-I8, T = 16, Gaussian) where it is
// faster than the FP64 DMMA K1T (measured crossover, profiles/), else K1T.  Neither is a
// fallback: both are GPU kernels parity-tested against the oracle.
bool use_i8T(Ctx& c, int T) {
    if (T != 16 || c.family != 0 || c.k1t_path == 0 || !i8s_supported(c.d, int(c.sched.st))) return false;
    if (c.k1t_path < 0 && c.d < kI8TMinD) return false;
    if (c.i8s_state == 0) {
        const int64_t n_pad = c.plan.n_pad;
        c.kp8s = i8s_kp(c.d);
        c.S8s.ensure(i8s_slice_bytes(n_pad, c.d));
        c.ex8s.ensure(size_t(n_pad));
        c.ejs8s.ensure(size_t(n_pad));
        c.sq8s.ensure(size_t(n_pad));
        c.i8s_state = i8s_prepare_launch(c.X.get(), c.n, c.d, n_pad, c.L.get(), c.plan.dp, c.plan.ec.kscale,
                                         c.S8s.get(), c.ex8s.get(), c.ejs8s.get(), c.sq8s.get(), c.stream)
                          ? 1
                          : -1;
    }
    return c.i8s_state == 1;
}

// Single right-hand sides with large d (where K1-I8 does not apply): one real column of a
// 16-column K1T-I8 pass beats the FP64 DMMA K1 from d ~ 160 (profiles/r1_k1_single_large_d.log:
// d = 192 27 vs 34 ms, d = 440 43 vs 75 ms at n = 65536).  Prepared outside graph capture.
bool use_i8T1(Ctx& c) {
    if (c.precision != 64 || c.family != 0 || c.k1_path == 0 || c.d < kI8T1MinD || use_i8(c) || use_i8x(c))
        return false;
    if (!use_i8T(c, 16)) return false;
    ensure_batched(c, 16);
    return true;
}

void matvec_dev(Ctx& c, const double* v, double* out, double lambda, cudaEvent_t k1a = nullptr,
                cudaEvent_t k1b = nullptr) {
    if (c.precision == 32) f32_ensure(c);
    if (k1a) KRR_CUDA(cudaEventRecord(k1a, c.stream));
    if (c.precision == 32)
        gauss_matvec_f32_launch(c.plan, c.S32.get(), c.s32.get(), v, c.v32.get(), c.part.get(), f32_kb(c.d), c.scale,
                                c.stream);
    else if (use_i8x(c))
        gauss_matvec_i8x_launch(c.plan, c.S8x.get(), c.sq8x.get(), c.i8x_E, v, c.part.get(), c.kp8, c.stream,
                                c.i8_debug);
    else if (use_i8(c))
        gauss_matvec_i8_launch(c.plan, c.S8.get(), c.ex8.get(), c.ejs8.get(), c.sq8.get(), v, c.part.get(), c.kp8,
                               c.stream, c.i8_debug, c.family == 1 ? c.degree : 0, c.gamma, c.offset);
    else if (use_i8T1(c)) {
        // v as column 0 of a zero-padded 16-column block through K1T-I8 (+ its finish, lambda,
        // all-reduce), column 0 back out
        pad_cols_launch(v, c.n, 1, 0, c.plan.n_pad, 16, c.bin.get(), c.stream);
        gauss_matmat_i8_launch(c.plan, c.S8s.get(), c.ex8s.get(), c.ejs8s.get(), c.sq8s.get(), c.bin.get(),
                               c.bpart.get(), c.kp8s, c.stream, c.i8_debug);
        if (k1b) KRR_CUDA(cudaEventRecord(k1b, c.stream));
        matmat_finish_launch(c.plan, c.bpart.get(), c.bin.get(), 16, lambda, c.k1_rank() == 0 ? 1 : 0, c.bout.get(),
                             c.stream);
        allreduce_sum(c, c.bout.get(), c.plan.n_pad * 16);
        unpad_cols_launch(c.bout.get(), c.n, 1, 0, 16, out, c.stream);
        return;
    } else
        gauss_matvec_launch(c.plan, v, c.part.get(), c.family == 1 ? poly_mode(c.degree) : c.exp_mode, c.stream);
    if (k1b) KRR_CUDA(cudaEventRecord(k1b, c.stream));
    matvec_finish_launch(c.plan, c.part.get(), v, lambda, c.k1_rank() == 0 ? 1 : 0, out, c.stream);
    allreduce_sum(c, out, c.plan.n_pad);
}

// KernelSpec::validate (kernels.cpp:36-44).
void validate_kernel(const krr_kernel_spec& k) {
    if (k.family == 0) {
        if (!(k.sigma > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: sigma must be positive");
    } else if (k.family == 1) {
        if (k.degree < 1) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: degree must be at least 1");
        if (k.offset < 0.0) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: offset must be non-negative");
        if (!(k.gamma > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: gamma must be positive");
    } else {
        fail(KRR_ERR_INVALID_ARGUMENT, "KernelSpec: unknown kernel family");
    }
}

krr_kernel_spec gaussian_spec(double sigma) {
    krr_kernel_spec k{};
    k.family = 0;
    k.sigma = sigma;
    return k;
}

void set_data(Ctx& c, const double* X, int64_t n, int64_t d, const krr_kernel_spec& ks) {
    if (n < 1 || d < 1) fail(KRR_ERR_INVALID_ARGUMENT, "krr_set_data: n and d must be positive");
    validate_kernel(ks);
    c.set_device();
    c.has_data = false;
    c.n = n;
    c.d = d;
    c.family = ks.family;
    c.sigma = ks.family == 0 ? ks.sigma : 1.0;
    c.scale = 1.0 / (2.0 * c.sigma * c.sigma);  // kernels.cpp:79
    c.gamma = ks.gamma;
    c.offset = ks.offset;
    c.degree = ks.degree;
    c.sched = make_schedule(n, c.k1_world(), c.k1_rank());
    const int dp = int(((d + 2) + 3) / 4 * 4);
    const int64_t n_pad = c.sched.n_pad;
    c.X.ensure(size_t(n * d));
    KRR_CUDA(cudaMemcpyAsync(c.X.get(), X, sizeof(double) * size_t(n * d), cudaMemcpyHostToDevice,
                             c.stream));
    c.L.ensure(size_t(n_pad * dp));
    c.R.ensure(size_t(n_pad * dp));
    if (c.family == 0) {
        build_operands_launch(c.X.get(), n, d, n_pad, dp, c.L.get(), c.R.get(), c.stream);
    } else {
        c.kdiag.ensure(size_t(n_pad));
        poly_operands_launch(c.X.get(), n, d, n_pad, dp, std::sqrt(c.gamma), std::sqrt(c.offset), c.degree,
                             c.L.get(), c.R.get(), c.kdiag.get(), c.stream);
    }
    const int64_t ntiles = int64_t(c.sched.tiles.size() / 2);
    c.tiles.ensure(size_t(std::max<int64_t>(1, ntiles)));
    if (ntiles)
        KRR_CUDA(cudaMemcpyAsync(c.tiles.get(), c.sched.tiles.data(), sizeof(int2) * size_t(ntiles),
                                 cudaMemcpyHostToDevice, c.stream));
    if (c.k1_world() > 1) {
        c.owned.ensure(c.sched.owned.size());
        KRR_CUDA(cudaMemcpyAsync(c.owned.get(), c.sched.owned.data(), c.sched.owned.size(),
                                 cudaMemcpyHostToDevice, c.stream));
    }
    double tab[64];
    make_exp_table(tab);
    c.exp_tab.ensure(64);
    KRR_CUDA(cudaMemcpyAsync(c.exp_tab.get(), tab, sizeof(tab), cudaMemcpyHostToDevice, c.stream));
    c.part.ensure(size_t(c.sched.ns * n_pad));
    for (auto* v : {&c.vin, &c.vout, &c.vx, &c.vr, &c.vz, &c.vp, &c.vap, &c.vy}) {
        v->ensure(size_t(n_pad));
        KRR_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * size_t(n_pad), c.stream));
    }
    c.nb = vec_blocks(n);
    c.red.ensure(size_t(4 * 1024));
    c.scal.ensure(16);
    KRR_CUDA(cudaMemsetAsync(c.scal.get(), 0, 16 * sizeof(double), c.stream));

    GaussMatvecPlan& p = c.plan;
    p.L = c.L.get();
    p.R = c.R.get();
    p.tiles = c.tiles.get();
    p.num_tiles = ntiles;
    p.owned = c.k1_world() > 1 ? c.owned.get() : nullptr;
    p.exp_tab = c.exp_tab.get();
    p.n = n;
    p.n_pad = n_pad;
    p.dp = dp;
    p.st = int(c.sched.st);
    p.ns = int(c.sched.ns);
    p.ec = c.family == 0 ? make_exp_consts(c.scale) : make_poly_consts(c.degree);
    p.kdiag = c.family == 1 ? c.kdiag.get() : nullptr;
    c.i8_ready = false;
    c.f32_ready = false;
    c.i8s_state = 0;
    c.i8x_E = 0;
    if (i8_supported(d, int(c.sched.st))) {
        c.kp8 = i8_kp(d);
        c.S8.ensure(size_t(8) * size_t(n_pad) * size_t(c.kp8));
        c.ex8.ensure(size_t(n_pad));
        c.ejs8.ensure(size_t(n_pad));
        c.sq8.ensure(size_t(n_pad));
        c.i8_ready = i8_prepare_launch(c.X.get(), n, d, n_pad, c.L.get(), dp,
                                       c.family == 0 ? p.ec.kscale : -1.0, c.S8.get(), c.ex8.get(), c.ejs8.get(),
                                       c.sq8.get(), c.stream, c.family == 1 ? c.gamma : 0.0);
    }
    p.resident = c.k1_resident;
    p.warps16 = c.k1_warps16;
    p.grouped = c.k1_grouped;
    i8x_ensure(c);
    c.sync();
    c.has_data = true;
}

// ---------------------------------------------------------------- preconditioner
void sketch_alloc(Ctx& c, int64_t n, int64_t s) {
    c.pn = n;
    c.s = s;
    shard_rows(n, c.world, c.rank, &c.z0, &c.z1);  // contiguous equal blocks
    c.Z.ensure(size_t(std::max<int64_t>(1, (c.z1 - c.z0) * s)));
    c.has_sketch = false;
    c.has_pre = false;
}

void rff_build(Ctx& c, const double* W, const double* b, int64_t s) {
    require_data(c);
    if (c.family != 0) fail(KRR_ERR_INVALID_ARGUMENT, "realize_chain: random Fourier features serve the Gaussian kernel");
    if (s < 1) fail(KRR_ERR_INVALID_ARGUMENT, "ChainSpec: s1 must be at least 1");
    c.set_device();
    sketch_alloc(c, c.n, s);
    c.wrff.ensure(size_t(s * c.d));
    c.brff.ensure(size_t(s));
    KRR_CUDA(cudaMemcpyAsync(c.wrff.get(), W, sizeof(double) * size_t(s * c.d),
                             cudaMemcpyHostToDevice, c.stream));
    KRR_CUDA(cudaMemcpyAsync(c.brff.get(), b, sizeof(double) * size_t(s), cudaMemcpyHostToDevice,
                             c.stream));
    const int64_t rows = c.z1 - c.z0;
    const int64_t s_pad = (s + 127) / 128 * 128;
    c.wpad.ensure(size_t(s_pad * c.plan.dp));
    rff_pad_w_launch(c.wrff.get(), s, c.d, s_pad, c.plan.dp, c.wpad.get(), c.stream);
    rff_features_launch(c.L.get() + c.z0 * c.plan.dp, c.wpad.get(), c.brff.get(), c.Z.get(), rows, s,
                        c.plan.dp, c.stream);
    c.sync();
    c.has_sketch = true;
}

void sketch_upload(Ctx& c, const double* Z, int64_t n, int64_t s) {
    if (n < 1 || s < 1) fail(KRR_ERR_INVALID_ARGUMENT, "krr_sketch_upload: empty sketch");
    c.set_device();
    sketch_alloc(c, n, s);
    const int64_t rows = c.z1 - c.z0;
    if (rows > 0)
        KRR_CUDA(cudaMemcpyAsync(c.Z.get(), Z + c.z0 * s, sizeof(double) * size_t(rows * s),
                                 cudaMemcpyHostToDevice, c.stream));
    c.sync();
    c.has_sketch = true;
}

// Returns true when the factorisation succeeded (finite, positive pivots): K4 (cholesky.cu).
bool try_potrf(Ctx& c, int64_t s) {
    // Non-finite input (e.g. Z'Z overflowed to inf) must fail like LLT on the reference's G.
    diag_check_launch(c.G.get(), s, c.chk.get(), c.stream);
    double h[2];
    KRR_CUDA(cudaMemcpyAsync(h, c.chk.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (h[1] != 0.0) return false;
    cholesky_launch(c.G.get(), s, c.info.get(), c.stream);
    int hinfo = 0;
    KRR_CUDA(cudaMemcpyAsync(&hinfo, c.info.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    diag_check_launch(c.G.get(), s, c.chk.get(), c.stream);
    KRR_CUDA(cudaMemcpyAsync(h, c.chk.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    return hinfo == 0 && h[1] == 0.0;
}

// build_preconditioner, precond.cpp:20-40.
void precond_build(Ctx& c, double lambda_p, int* jitter_used) {
    if (!(lambda_p > 0.0))
        fail(KRR_ERR_NON_POSITIVE_LAMBDA, "build_preconditioner: lambda_p must be positive");
    if (!c.has_sketch) fail(KRR_ERR_STATE, "no sketch on the context (krr_rff_build / krr_sketch_upload)");
    c.set_device();
    const int64_t s = c.s;
    const int64_t rows = c.z1 - c.z0;
    c.G.ensure(size_t(s * s));
    c.Gcopy.ensure(size_t(s * s));
    c.chk.ensure(4);
    c.info.ensure(1);
    Events ev(4);
    KRR_CUDA(cudaEventRecord(ev[0], c.stream));
    // G = Z^T Z (precond.cpp:23): K3-I8, column-major lower triangle (gram_i8.cu)
    gram_dev(c, c.Z.get(), rows, s, c.G.get());
    allreduce_sum(c, c.G.get(), s * s);
    diag_add_launch(c.G.get(), s, lambda_p, c.stream);  // precond.cpp:24
    KRR_CUDA(cudaEventRecord(ev[1], c.stream));
    KRR_CUDA(cudaMemcpyAsync(c.Gcopy.get(), c.G.get(), sizeof(double) * size_t(s * s),
                             cudaMemcpyDeviceToDevice, c.stream));
    if (jitter_used) *jitter_used = 0;
    if (!try_potrf(c, s)) {
        // precond.cpp:29-33: one retry with 1e-12 trace / s on the diagonal.
        KRR_CUDA(cudaMemcpyAsync(c.G.get(), c.Gcopy.get(), sizeof(double) * size_t(s * s),
                                 cudaMemcpyDeviceToDevice, c.stream));
        trace_launch(c.G.get(), s, c.chk.get() + 2, c.stream);
        double tr = 0.0;
        KRR_CUDA(cudaMemcpyAsync(&tr, c.chk.get() + 2, sizeof(double), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
        diag_add_launch(c.G.get(), s, 1e-12 * tr / double(s), c.stream);
        if (jitter_used) *jitter_used = 1;
        if (!try_potrf(c, s))
            fail(KRR_ERR_NOT_POSITIVE_DEFINITE, "cholesky: non-positive pivot encountered");
    }
    // numerics.cpp:62-63
    double h[2];
    diag_check_launch(c.G.get(), s, c.chk.get(), c.stream);
    KRR_CUDA(cudaMemcpyAsync(h, c.chk.get(), sizeof(h), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (h[0] < 1e-300) fail(KRR_ERR_SINGULAR_TRIANGULAR, "triangular_solve: diagonal entry below 1e-300");
    KRR_CUDA(cudaEventRecord(ev[2], c.stream));
    // U = L^-1 Z^T in place over the row-major Z (precond.cpp:38): K5 on DMMA (trsm.cu)
    trsm_lower_launch(c.Z.get(), rows, s, c.G.get(), c.stream);
    KRR_CUDA(cudaEventRecord(ev[3], c.stream));
    c.lambda_p = lambda_p;
    c.sync();
    for (int k = 0; k < 3; ++k) {
        float ms = 0.0f;
        KRR_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
        c.build_ms[k] = ms;
    }
    c.has_pre = true;
}

// z (full length pn, zero-padded beyond) = (r - U^T U r) / lambda_p
void precond_apply_dev(Ctx& c, const double* r, double* z) {
    if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
    const int64_t s = c.s;
    const int64_t rows = c.z1 - c.z0;
    const int nchunks = gemvT_chunks(std::max<int64_t>(1, rows), s);
    c.W.ensure(size_t(s));
    c.Wpart.ensure(size_t(nchunks) * size_t(s));
    if (rows > 0) {
        gemvT_partial_launch(c.Z.get(), rows, s, r + c.z0, c.Wpart.get(), nchunks, c.stream);
        reduce_rows_launch(c.Wpart.get(), nchunks, s, c.W.get(), c.stream);
    } else {
        KRR_CUDA(cudaMemsetAsync(c.W.get(), 0, sizeof(double) * size_t(s), c.stream));
    }
    allreduce_sum(c, c.W.get(), s);
    const int nbz = zrow_blocks(std::max<int64_t>(1, rows));
    c.red.ensure(size_t(4 * 1024));
    if (rows > 0)
        precond_z_launch(c.Z.get(), rows, s, c.W.get(), r + c.z0, c.lambda_p, z + c.z0,
                         c.red.get() + 3 * 1024, nbz, c.stream);
    if (c.world > 1) {
        // Every rank owns an equal block `per` of rows (the last one possibly short);
        // zero the non-owned rows and sum — an all-gather expressed as an all-reduce,
        // valid for any n.
        if (c.z0 > 0) KRR_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * size_t(c.z0), c.stream));
        if (c.z1 < c.pn)
            KRR_CUDA(cudaMemsetAsync(z + c.z1, 0, sizeof(double) * size_t(c.pn - c.z1), c.stream));
        allreduce_sum(c, z, c.pn);
    }
}

// ---------------------------------------------------------------- PCG core (solver.cpp:22-67)
using DevOp = std::function<void(const double* din, double* dout)>;
using HostObserver = std::function<void(int, const double* dx)>;

struct PcgOut {
    int iterations = 0;
    int converged = 0;
    double final_residual = 0.0;
};

// Vectors live in c.vx/vr/vz/vp/vap (length >= n, zero beyond n).  y is a device
// vector of length n (zero-padded to the buffer length).  The solution is left in c.vx.
// The graph-resident PCG loop: the same kernels in the same order as pcg_core's host loop
// (bitwise-identical iterates), captured once into the body of a conditional WHILE node; a
// one-thread control kernel makes solver.cpp:37-52's stop / breakdown decision on the device.
// No host observer (any world size).  Precondition: the caller ran the prologue (x = 0, r = y,
// z = M r, p = z, scal[2] = r'z) and norm_y > 0.
// Returns false — and leaves the vectors of the prologue untouched — only when a multi-rank context
// cannot build the graph (the captured NCCL collectives are the one part no single-GPU run can
// exercise): every rank fails the same way, reports it on stderr and takes the host-driven loop.
bool pcg_graph_loop(Ctx& c, int64_t n, const DevOp& A, const DevOp* M, double norm_y, double tau, int max_iter,
                    double* hist, PcgOut& out) {
    if (c.precision == 32) f32_ensure(c);  // one-off preparation synchronises: not inside the capture
    use_i8T1(c);                            // (same for the large-d single-column K1T-I8 route)
    const int nb = vec_blocks(n);
    double* red = c.red.get();
    double* pap_part = red;
    double* rr_part = red + 1024;
    double* rz_part = red + 2048;
    double* scal = c.scal.get();
    c.ctl.ensure(4);
    c.dhist.ensure(size_t(std::max(1, max_iter)));
    KRR_CUDA(cudaMemsetAsync(c.ctl.get(), 0, 4 * sizeof(int), c.stream));
    double* z = M ? c.vz.get() : c.vr.get();

    cudaGraph_t g = nullptr;
    cudaGraphExec_t exec = nullptr;
    struct Cleanup {
        cudaGraph_t& g;
        cudaGraphExec_t& e;
        ~Cleanup() {
            if (e) cudaGraphExecDestroy(e);
            if (g) cudaGraphDestroy(g);
        }
    } cleanup{g, exec};
    try {
    KRR_CUDA(cudaGraphCreate(&g, 0));
    cudaGraphConditionalHandle cond;
    KRR_CUDA(cudaGraphConditionalHandleCreate(&cond, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams np{};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = cond;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    KRR_CUDA(cudaGraphAddNode(&node, g, nullptr, 0, &np));
    cudaGraph_t body = np.conditional.phGraph_out[0];
    KRR_CUDA(cudaStreamBeginCaptureToGraph(c.stream, body, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    try {
        A(c.vp.get(), c.vap.get());
        dot_partial_launch(c.vp.get(), c.vap.get(), n, pap_part, nb, c.stream);
        pcg_update_xr_launch(pap_part, nb, scal + 2, c.vx.get(), c.vr.get(), c.vp.get(), c.vap.get(), n, rr_part,
                             scal, c.stream);
        sum_partials_launch(rr_part, nb, scal + 4, c.stream);
        pcg_control_launch(scal, c.ctl.get(), c.dhist.get(), scal + 6, norm_y, tau, max_iter, cond, c.stream);
        // (after a stop the rest of the body still runs once; it touches only z, p and r'z)
        if (M) (*M)(c.vr.get(), z);
        dot_partial_launch(c.vr.get(), z, n, rz_part, nb, c.stream);
        pcg_update_p_launch(rz_part, nb, scal + 2, scal + 3, c.vp.get(), z, n, c.stream);
        scalar_copy_launch(scal + 2, scal + 3, c.stream);
    } catch (...) {
        cudaGraph_t dummy = nullptr;
        cudaStreamEndCapture(c.stream, &dummy);
        throw;
    }
    KRR_CUDA(cudaStreamEndCapture(c.stream, &body));
    KRR_CUDA(cudaGraphInstantiate(&exec, g, 0));
    } catch (const Error& e) {
        if (c.world <= 1) throw;  // single-GPU contexts: the graph loop is tested, a failure is a bug
        cudaGetLastError();
        std::fprintf(stderr, "krr: rank %d: graph-resident PCG loop unavailable (%s); using the host-driven loop\n",
                     c.rank, e.what());
        c.pcg_graph = false;
        return false;
    }
    KRR_CUDA(cudaGraphLaunch(exec, c.stream));
    int hctl[4];
    double* hs = c.hscal->p;
    KRR_CUDA(cudaMemcpyAsync(hctl, c.ctl.get(), sizeof(hctl), cudaMemcpyDeviceToHost, c.stream));
    KRR_CUDA(cudaMemcpyAsync(hs + 6, scal + 6, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const int its = hctl[0];
    if (hist && its > 0) {
        KRR_CUDA(cudaMemcpyAsync(hist, c.dhist.get(), sizeof(double) * size_t(hctl[1] == 3 ? its - 1 : its),
                                 cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    }
    if (hctl[1] == 3) fail(KRR_ERR_BREAKDOWN, "pcg_solve: p'Ap <= 0, operator is not positive definite");
    out.iterations = its;
    out.final_residual = hs[6];
    out.converged = hctl[1] == 1 ? 1 : 0;
    return true;
}

// device_ops: A and M only enqueue device work on c.stream (no host callbacks, no host
// synchronisation) — the precondition for the graph-resident loop.
PcgOut pcg_core(Ctx& c, int64_t n, const DevOp& A, const DevOp* M, const double* y, double tau,
                int max_iter, double* hist, const HostObserver* obs, bool device_ops) {
    if (!(tau > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "pcg_solve: tau must be positive");
    if (max_iter < 1) fail(KRR_ERR_INVALID_ARGUMENT, "pcg_solve: max_iter must be at least 1");
    const int nb = vec_blocks(n);
    double* red = c.red.get();
    double* pap_part = red;
    double* rr_part = red + 1024;
    double* rz_part = red + 2048;
    double* scal = c.scal.get();  // [0] pap [1] alpha [2] rz(even) [3] rz(odd) [4] rr [5] yy
    double* hs = c.hscal->p;
    PcgOut out;
    KRR_CUDA(cudaMemsetAsync(c.vx.get(), 0, sizeof(double) * size_t(n), c.stream));
    dot_partial_launch(y, y, n, rr_part, nb, c.stream);
    sum_partials_launch(rr_part, nb, scal + 5, c.stream);
    KRR_CUDA(cudaMemcpyAsync(hs + 5, scal + 5, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    const double norm_y = std::sqrt(hs[5]);
    if (norm_y == 0.0) {  // solver.cpp:30-34
        out.converged = 1;
        return out;
    }
    copy_launch(c.vr.get(), y, n, c.stream);  // r = y
    double* z = c.vz.get();
    if (M) {
        (*M)(c.vr.get(), z);
    } else {
        z = c.vr.get();
    }
    copy_launch(c.vp.get(), z, n, c.stream);  // p = z
    dot_partial_launch(c.vr.get(), z, n, rz_part, nb, c.stream);
    sum_partials_launch(rz_part, nb, scal + 2, c.stream);
    // multi-rank too: the NCCL all-reduces are captured into the loop body (relaxed capture), and
    // every stop decision is made from all-reduced (rank-identical) vectors, so all ranks run the
    // same number of iterations without a host round trip
    if (device_ops && c.pcg_graph && !obs) {
        if (pcg_graph_loop(c, n, A, M, norm_y, tau, max_iter, hist, out)) return out;
    }
    int cur = 0;
    for (int it = 1; it <= max_iter; ++it) {
        A(c.vp.get(), c.vap.get());
        dot_partial_launch(c.vp.get(), c.vap.get(), n, pap_part, nb, c.stream);
        pcg_update_xr_launch(pap_part, nb, scal + 2 + cur, c.vx.get(), c.vr.get(), c.vp.get(),
                             c.vap.get(), n, rr_part, scal, c.stream);
        sum_partials_launch(rr_part, nb, scal + 4, c.stream);
        KRR_CUDA(cudaMemcpyAsync(hs, scal, 5 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        const double pap = hs[0];
        if (!(pap > 0.0))
            fail(KRR_ERR_BREAKDOWN, "pcg_solve: p'Ap <= 0, operator is not positive definite");
        const double rel = std::sqrt(hs[4]) / norm_y;
        out.iterations = it;
        out.final_residual = rel;
        if (hist) hist[it - 1] = rel;
        if (obs) (*obs)(it, c.vx.get());
        if (rel <= tau) {
            out.converged = 1;
            return out;
        }
        if (M) (*M)(c.vr.get(), z);
        dot_partial_launch(c.vr.get(), z, n, rz_part, nb, c.stream);
        pcg_update_p_launch(rz_part, nb, scal + 2 + cur, scal + 2 + (cur ^ 1), c.vp.get(), z, n,
                            c.stream);
        cur ^= 1;
    }
    out.converged = 0;
    return out;
}

// ---------------------------------------------------------------- batched multi-RHS (t > 1)
int batch_width(int64_t t) { return t <= 8 ? 8 : 16; }


// out (n_pad x T) = (K + lambda I) v (n_pad x T), replicated on all ranks.
void matvecT_dev(Ctx& c, const double* v, double* out, int T, double lambda) {
    if (use_i8T(c, T))
        gauss_matmat_i8_launch(c.plan, c.S8s.get(), c.ex8s.get(), c.ejs8s.get(), c.sq8s.get(), v, c.bpart.get(),
                               c.kp8s, c.stream, c.i8_debug);
    else
        gauss_matmat_launch(c.plan, v, T, c.bpart.get(), c.family == 1 ? poly_mode(c.degree) : 1, c.stream);
    matmat_finish_launch(c.plan, c.bpart.get(), v, T, lambda, c.k1_rank() == 0 ? 1 : 0, out, c.stream);
    allreduce_sum(c, out, c.plan.n_pad * T);
}

// z (pn x T) = (r - U^T U r) / lambda_p for T interleaved columns (precond.cpp:15-18): the two
// K6T passes over the row shard of B = U^T (precond_multi.cu), the s x T all-reduce between them.
void precondT_apply_dev(Ctx& c, const double* r, double* z, int T) {
    if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
    const int64_t s = c.s, rows = c.z1 - c.z0;
    if (!k6t_supported(s, c.Z.get())) {  // odd s: row starts not 16-byte aligned; column by column (K6)
        c.vin.ensure(size_t(c.pn));
        c.vout.ensure(size_t(c.pn));
        for (int j = 0; j < T; ++j) {
            gather_col_launch(r, c.pn, T, j, c.vin.get(), c.stream);
            precond_apply_dev(c, c.vin.get(), c.vout.get());
            scatter_col_launch(c.vout.get(), c.pn, T, j, z, c.stream);
        }
        return;
    }
    const int nsplit = k6t_splits(std::max<int64_t>(1, rows), s);
    c.bW.ensure(size_t(s * T));
    c.Wpart.ensure(size_t(nsplit) * size_t(s * T));
    precond_multi_launch(c.Z.get(), rows, s, r + c.z0 * T, c.lambda_p, z + c.z0 * T, c.Wpart.get(), nsplit,
                         c.bW.get(), T, 1, c.stream);
    allreduce_sum(c, c.bW.get(), s * T);
    precond_multi_launch(c.Z.get(), rows, s, r + c.z0 * T, c.lambda_p, z + c.z0 * T, c.Wpart.get(), nsplit,
                         c.bW.get(), T, 2, c.stream);
    if (c.world > 1) {
        if (c.z0 > 0) KRR_CUDA(cudaMemsetAsync(z, 0, sizeof(double) * size_t(c.z0 * T), c.stream));
        if (c.z1 < c.pn)
            KRR_CUDA(cudaMemsetAsync(z + c.z1 * T, 0, sizeof(double) * size_t((c.pn - c.z1) * T), c.stream));
        allreduce_sum(c, z, c.pn * T);
    }
}

// Batched PCG over T interleaved columns, t_real of which are real.  Every column runs
// exactly the reference's per-column recurrence (solver.cpp:22-67) with its own alpha,
// beta and stopping test; converged columns are frozen by a device mask.
void pcgT_core(Ctx& c, int T, int t_real, double lambda, bool use_pre, double tau, int max_iter,
               krr_rhs_stats* stats, double* hist, int64_t hist_stride) {
    if (!(tau > 0.0)) fail(KRR_ERR_INVALID_ARGUMENT, "pcg_solve: tau must be positive");
    if (max_iter < 1) fail(KRR_ERR_INVALID_ARGUMENT, "pcg_solve: max_iter must be at least 1");
    const int64_t n = c.n, nt = c.plan.n_pad * T;
    const int nb = vecT_blocks(n, T);
    double* pap_part = c.bred.get();
    double* rr_part = pap_part + size_t(nb) * T;
    double* rz_part = rr_part + size_t(nb) * T;
    double* sc = c.bscal.get();  // [0,16) pap  [16,32) rz even  [32,48) rz odd  [48,64) rr  [64,80) yy
    double* hs = c.hscalT->p;
    KRR_CUDA(cudaMemsetAsync(c.bx.get(), 0, sizeof(double) * size_t(nt), c.stream));
    dotT_partial_launch(c.by.get(), c.by.get(), n, T, rr_part, nb, c.stream);
    sumT_partials_launch(rr_part, nb, T, sc + 64, c.stream);
    KRR_CUDA(cudaMemcpyAsync(hs + 64, sc + 64, sizeof(double) * T, cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    std::vector<double> norm_y(static_cast<size_t>(T));
    int n_active = 0;
    for (int j = 0; j < T; ++j) {
        norm_y[size_t(j)] = std::sqrt(hs[64 + j]);
        const bool act = j < t_real && norm_y[size_t(j)] != 0.0;
        c.hactive[j] = act ? 1 : 0;
        n_active += act;
        if (j < t_real) stats[j] = krr_rhs_stats{0, act ? 0 : 1, 0.0};  // zero RHS: converged, 0 its
    }
    KRR_CUDA(cudaMemcpyAsync(c.bactive.get(), c.hactive, sizeof(int) * T, cudaMemcpyHostToDevice, c.stream));
    if (n_active == 0) return;
    copy_launch(c.br.get(), c.by.get(), nt, c.stream);
    // precondT_apply_dev writes rows < n only; bz's padded tail feeds bp (copied below), which
    // K1T reads, so it must be zero whatever an earlier call left there
    if (use_pre) KRR_CUDA(cudaMemsetAsync(c.bz.get(), 0, sizeof(double) * size_t(nt), c.stream));
    double* z = use_pre ? c.bz.get() : c.br.get();
    if (use_pre) precondT_apply_dev(c, c.br.get(), z, T);
    copy_launch(c.bp.get(), z, nt, c.stream);
    dotT_partial_launch(c.br.get(), z, n, T, rz_part, nb, c.stream);
    sumT_partials_launch(rz_part, nb, T, sc + 16, c.stream);
    int cur = 0;
    for (int it = 1; it <= max_iter && n_active > 0; ++it) {
        matvecT_dev(c, c.bp.get(), c.bap.get(), T, lambda);
        dotT_partial_launch(c.bp.get(), c.bap.get(), n, T, pap_part, nb, c.stream);
        pcgT_update_xr_launch(pap_part, nb, T, sc + 16 + 16 * cur, c.bactive.get(), c.bx.get(), c.br.get(),
                              c.bp.get(), c.bap.get(), n, rr_part, sc, c.stream);
        sumT_partials_launch(rr_part, nb, T, sc + 48, c.stream);
        KRR_CUDA(cudaMemcpyAsync(hs, sc, sizeof(double) * 64, cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        bool changed = false;
        for (int j = 0; j < t_real; ++j) {
            if (!c.hactive[j]) continue;
            if (!(hs[j] > 0.0))
                fail(KRR_ERR_BREAKDOWN, "pcg_solve: p'Ap <= 0, operator is not positive definite");
            const double rel = std::sqrt(hs[48 + j]) / norm_y[size_t(j)];
            stats[j].iterations = it;
            stats[j].final_residual = rel;
            if (hist) hist[j * hist_stride + it - 1] = rel;
            if (rel <= tau) {
                stats[j].converged = 1;
                c.hactive[j] = 0;
                --n_active;
                changed = true;
            }
        }
        if (n_active == 0) break;
        if (changed)
            KRR_CUDA(cudaMemcpyAsync(c.bactive.get(), c.hactive, sizeof(int) * T, cudaMemcpyHostToDevice,
                                     c.stream));
        if (use_pre) precondT_apply_dev(c, c.br.get(), z, T);
        dotT_partial_launch(c.br.get(), z, n, T, rz_part, nb, c.stream);
        pcgT_update_p_launch(rz_part, nb, T, sc + 16 + 16 * cur, sc + 16 + 16 * (cur ^ 1), c.bactive.get(),
                             c.bp.get(), z, n, c.stream);
        cur ^= 1;
    }
}

DevOp gaussian_op(Ctx& c, double lambda) {
    return [&c, lambda](const double* din, double* dout) { matvec_dev(c, din, dout, lambda); };
}

DevOp precond_op(Ctx& c) {
    return [&c](const double* din, double* dout) { precond_apply_dev(c, din, dout); };
}

// (K + lambda I) V for V n x t row-major on the device (K1T batches, or column by column).
void matmat_dev(Ctx& c, const double* V, int64_t t, double lambda, double* Out) {
    const int64_t n = c.n;
    if (t > 1 && c.batched && c.precision == 64) {
        const int T = batch_width(t);
        ensure_batched(c, T);
        for (int64_t c0 = 0; c0 < t; c0 += T) {
            pad_cols_launch(V, n, t, c0, c.plan.n_pad, T, c.bin.get(), c.stream);
            matvecT_dev(c, c.bin.get(), c.bout.get(), T, lambda);
            unpad_cols_launch(c.bout.get(), n, t, c0, T, Out, c.stream);
        }
    } else {
        for (int64_t j = 0; j < t; ++j) {
            gather_col_launch(V, n, t, j, c.vin.get(), c.stream);
            matvec_dev(c, c.vin.get(), c.vout.get(), lambda);
            scatter_col_launch(c.vout.get(), n, t, j, Out, c.stream);
        }
    }
}

// ---------------------------------------------------------------- f3: quality test / adaptive sizing
// symmetric_eigen (numerics.cpp:144-154): eigenvalues descending, eigenvectors as columns (in
// place of A, col-major s x s); cuSOLVER returns them ascending, the caller reads them reversed.
void syevd_dev(Ctx& c, double* A, int64_t s, double* evals) {
    int lwork = 0;
    cusolver_check(cusolverDnSetStream(c.sol, c.stream), "cusolverDnSetStream");
    cusolver_check(cusolverDnDsyevd_bufferSize(c.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(s), A,
                                               int(s), evals, &lwork),
                   "syevd_bufferSize");
    DevMem<double> work;
    DevMem<int> info;
    work.ensure(size_t(std::max(1, lwork)));
    info.ensure(1);
    cusolver_check(cusolverDnDsyevd(c.sol, CUSOLVER_EIG_MODE_VECTOR, CUBLAS_FILL_MODE_LOWER, int(s), A, int(s), evals,
                                    work.get(), lwork, info.get()),
                   "syevd");
    int h = 0;
    KRR_CUDA(cudaMemcpyAsync(&h, info.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (h != 0) fail(KRR_ERR_NO_CONVERGENCE, "symmetric_eigen: eigensolver did not converge");  // types.hpp:34
}

// quality_test (precond.cpp:60-100) of the context's raw sketch Z against its data's K.
krr_quality_report quality_test_dev(Ctx& c, double lambda) {
    if (!(lambda > 0.0)) fail(KRR_ERR_NON_POSITIVE_LAMBDA, "quality_test: lambda must be positive");
    if (!c.has_sketch || c.has_pre) fail(KRR_ERR_STATE, "quality_test needs the raw sketch (before the preconditioner)");
    if (c.world != 1) fail(KRR_ERR_STATE, "quality_test is single-rank");
    if (c.pn != c.n) fail(KRR_ERR_DIMENSION_MISMATCH, "quality_test: K and Z dimensions do not match");
    c.set_device();
    const int64_t n = c.n, s = c.s;
    krr_quality_report r{};
    r.lambda = lambda;
    r.sketch_size = s;
    r.spectrum_cut = 0.05 * lambda;
    r.cond1_threshold = 0.1 * lambda;
    r.ratio_low_threshold = 0.9;
    r.ratio_high_threshold = 1.1;
    r.cond2_ratio_low = 1.0;
    r.cond2_ratio_high = 1.0;
    const double one = 1.0, zero = 0.0, mone = -1.0;
    cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
    // retained_left_singular_basis (precond.cpp:42-58): eig(Z^T Z), B = Z V_k / sqrt(ev)
    DevMem<double> G, ev;
    G.ensure(size_t(s * s));
    ev.ensure(size_t(s));
    gram_dev(c, c.Z.get(), n, s, G.get());  // Z^T Z on K3-I8 (lower triangle, what syevd reads)
    syevd_dev(c, G.get(), s, ev.get());
    std::vector<double> evh(static_cast<size_t>(s));
    KRR_CUDA(cudaMemcpyAsync(evh.data(), ev.get(), sizeof(double) * size_t(s), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    std::reverse(evh.begin(), evh.end());  // descending
    const double max_ev = s > 0 ? std::max(0.0, evh[0]) : 0.0;
    const double zero_floor = 1e-20 * max_ev;
    int64_t k = 0;
    while (k < s && evh[size_t(k)] > r.spectrum_cut && evh[size_t(k)] > zero_floor) ++k;
    r.rank_of_p = k;
    DevMem<double> Vk, Bt, tk, v, w, w2;
    if (k > 0) {
        // V_k scaled: column i = eigenvector of the i-th largest eigenvalue / sqrt(ev_i)
        // (cuSOLVER's ascending column s-1-i); host-side scale list, device gather
        std::vector<double> sc(static_cast<size_t>(k));
        for (int64_t i = 0; i < k; ++i) sc[size_t(i)] = 1.0 / std::sqrt(evh[size_t(i)]);
        Vk.ensure(size_t(s * k));
        for (int64_t i = 0; i < k; ++i) {
            KRR_CUDA(cudaMemcpyAsync(Vk.get() + i * s, G.get() + (s - 1 - i) * s, sizeof(double) * size_t(s),
                                     cudaMemcpyDeviceToDevice, c.stream));
            cublas_check(cublasDscal(c.blas, int(s), &sc[size_t(i)], Vk.get() + i * s, 1), "cublasDscal");
        }
        // B (n x k row-major) = col-major B^T (k x n) = V_k^T (k x s) . Z^T (s x n)
        Bt.ensure(size_t(k * n));
        cublas_check(cublasDgemm(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, int(k), int(n), int(s), &one, Vk.get(), int(s),
                                 c.Z.get(), int(s), &zero, Bt.get(), int(k)),
                     "cublasDgemm(B)");
        tk.ensure(size_t(k));
    }
    // condition 1: power_iteration_spectral_norm (numerics.cpp:156-190) on (I-P) K (I-P),
    // start vector from mt19937_64(7) normal draws, tol 1e-4, 500 iterations
    const int64_t n_pad = c.plan.n_pad;
    v.ensure(size_t(n_pad));
    w.ensure(size_t(n_pad));
    w2.ensure(size_t(n_pad));
    KRR_CUDA(cudaMemsetAsync(v.get(), 0, sizeof(double) * size_t(n_pad), c.stream));
    KRR_CUDA(cudaMemsetAsync(w.get(), 0, sizeof(double) * size_t(n_pad), c.stream));
    KRR_CUDA(cudaMemsetAsync(w2.get(), 0, sizeof(double) * size_t(n_pad), c.stream));
    {
        std::vector<double> v0(static_cast<size_t>(n));
        power_iteration_start(7, n, v0.data());
        KRR_CUDA(cudaMemcpyAsync(v.get(), v0.data(), sizeof(double) * size_t(n), cudaMemcpyHostToDevice, c.stream));
    }
    auto deflate = [&](double* x) {  // x -= B (B^T x)
        if (k == 0) return;
        cublas_check(cublasDgemv(c.blas, CUBLAS_OP_N, int(k), int(n), &one, Bt.get(), int(k), x, 1, &zero, tk.get(), 1),
                     "gemv B^T x");
        cublas_check(cublasDgemv(c.blas, CUBLAS_OP_T, int(k), int(n), &mone, Bt.get(), int(k), tk.get(), 1, &one, x, 1),
                     "gemv x - B t");
    };
    double prev = 0.0;
    r.cond1_value = 0.0;
    for (int it = 1; it <= 500; ++it) {
        KRR_CUDA(cudaMemcpyAsync(w2.get(), v.get(), sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, c.stream));
        deflate(w2.get());
        matvec_dev(c, w2.get(), w.get(), 0.0);  // K (no diagonal shift)
        deflate(w.get());
        double rq = 0.0, nw = 0.0;
        cublas_check(cublasDdot(c.blas, int(n), v.get(), 1, w.get(), 1, &rq), "dot");
        cublas_check(cublasDnrm2(c.blas, int(n), w.get(), 1, &nw), "nrm2");
        r.cond1_value = rq;
        if (nw == 0.0) {
            r.cond1_value = 0.0;
            break;
        }
        if (it > 1 && std::abs(rq - prev) <= 1e-4 * std::abs(rq)) break;
        prev = rq;
        const double inv = 1.0 / nw;
        KRR_CUDA(cudaMemcpyAsync(v.get(), w.get(), sizeof(double) * size_t(n), cudaMemcpyDeviceToDevice, c.stream));
        cublas_check(cublasDscal(c.blas, int(n), &inv, v.get(), 1), "scal");
    }
    // condition 2 on range(P): eigenvalues of Sigma^-1 (B^T K B) Sigma^-1, symmetrised
    if (k > 0) {
        DevMem<double> B, KB, M;
        B.ensure(size_t(n * k));
        KB.ensure(size_t(n * k));
        // B row-major n x k is exactly Bt col-major: the same buffer
        matmat_dev(c, Bt.get(), k, 0.0, KB.get());
        M.ensure(size_t(k * k));
        // M (k x k) = B^T (K B): col-major Bt (k x n) . KBt (k x n)^T
        cublas_check(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_T, int(k), int(k), int(n), &one, Bt.get(), int(k),
                                 KB.get(), int(k), &zero, M.get(), int(k)),
                     "cublasDgemm(B^T K B)");
        std::vector<double> mh(static_cast<size_t>(k * k));
        KRR_CUDA(cudaMemcpyAsync(mh.data(), M.get(), sizeof(double) * size_t(k * k), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        std::vector<double> inv_sigma(static_cast<size_t>(k));
        for (int64_t i = 0; i < k; ++i) inv_sigma[size_t(i)] = 1.0 / std::sqrt(evh[size_t(i)]);
        std::vector<double> sym(static_cast<size_t>(k * k));
        for (int64_t i = 0; i < k; ++i)
            for (int64_t j = 0; j < k; ++j) {
                const double a = inv_sigma[size_t(i)] * mh[size_t(j * k + i)] * inv_sigma[size_t(j)];
                const double b = inv_sigma[size_t(j)] * mh[size_t(i * k + j)] * inv_sigma[size_t(i)];
                sym[size_t(j * k + i)] = (a + b) / 2.0;
            }
        KRR_CUDA(cudaMemcpyAsync(M.get(), sym.data(), sizeof(double) * size_t(k * k), cudaMemcpyHostToDevice, c.stream));
        DevMem<double> ev2;
        ev2.ensure(size_t(k));
        syevd_dev(c, M.get(), k, ev2.get());
        std::vector<double> e2(static_cast<size_t>(k));
        KRR_CUDA(cudaMemcpyAsync(e2.data(), ev2.get(), sizeof(double) * size_t(k), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        r.cond2_ratio_high = e2[size_t(k - 1)];
        r.cond2_ratio_low = e2[0];
    }
    r.passed = r.cond1_value <= r.cond1_threshold && r.cond2_ratio_low >= r.ratio_low_threshold &&
               r.cond2_ratio_high <= r.ratio_high_threshold;
    return r;
}

// solve_regularized (solver.cpp:69-94): per-column sequential PCG.
void solve_gaussian(Ctx& c, double lambda, const double* Y, int64_t t, double tau, int max_iter,
                    int use_precond, double* C, krr_rhs_stats* stats, double* hist,
                    int64_t* total_matvecs) {
    require_data(c);
    if (!(lambda > 0.0)) fail(KRR_ERR_NON_POSITIVE_LAMBDA, "train: lambda must be positive");
    if (t < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "solve_regularized: Y needs at least one column");
    if (use_precond) {
        if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
        if (c.pn != c.n)
            fail(KRR_ERR_DIMENSION_MISMATCH, "Preconditioner: dimension mismatch");
    }
    c.set_device();
    const int64_t n = c.n;
    c.mat_a.ensure(size_t(n * t));
    c.mat_b.ensure(size_t(n * t));
    KRR_CUDA(cudaMemcpyAsync(c.mat_a.get(), Y, sizeof(double) * size_t(n * t), cudaMemcpyHostToDevice,
                             c.stream));
    if (t > 1 && c.batched && c.precision == 64) {
        // Independent columns in batches of T = 8 or 16 sharing every K1T pass.
        const int T = batch_width(t);
        ensure_batched(c, T);
        int64_t total = 0;
        for (int64_t c0 = 0; c0 < t; c0 += T) {
            const int t_real = int(std::min<int64_t>(T, t - c0));
            pad_cols_launch(c.mat_a.get(), n, t, c0, c.plan.n_pad, T, c.by.get(), c.stream);
            pcgT_core(c, T, t_real, lambda, use_precond != 0, tau, max_iter, stats + c0,
                      hist ? hist + c0 * max_iter : nullptr, max_iter);
            unpad_cols_launch(c.bx.get(), n, t, c0, T, c.mat_b.get(), c.stream);
            for (int j = 0; j < t_real; ++j) total += stats[c0 + j].iterations;
        }
        KRR_CUDA(cudaMemcpyAsync(C, c.mat_b.get(), sizeof(double) * size_t(n * t), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
        if (total_matvecs) *total_matvecs = total;
        return;
    }
    const DevOp A = gaussian_op(c, lambda);
    const DevOp M = precond_op(c);
    int64_t total = 0;
    for (int64_t j = 0; j < t; ++j) {
        // K1 reads the padded tail of p: keep every PCG vector zero beyond n.
        for (auto* v : {&c.vx, &c.vr, &c.vz, &c.vp, &c.vap, &c.vy})
            KRR_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * v->count, c.stream));
        gather_col_launch(c.mat_a.get(), n, t, j, c.vy.get(), c.stream);
        const PcgOut o = pcg_core(c, n, A, use_precond ? &M : nullptr, c.vy.get(), tau, max_iter,
                                  hist ? hist + j * max_iter : nullptr, nullptr, true);
        scatter_col_launch(c.vx.get(), n, t, j, c.mat_b.get(), c.stream);
        stats[j].iterations = o.iterations;
        stats[j].converged = o.converged;
        stats[j].final_residual = o.final_residual;
        total += o.iterations;
    }
    KRR_CUDA(cudaMemcpyAsync(C, c.mat_b.get(), sizeof(double) * size_t(n * t), cudaMemcpyDeviceToHost,
                             c.stream));
    c.sync();
    if (total_matvecs) *total_matvecs = total;
}

void ctx_init_common(Ctx& c) {
    c.set_device();
    KRR_CUDA(cudaStreamCreateWithFlags(&c.stream, cudaStreamNonBlocking));
    cublas_check(cublasCreate(&c.blas), "cublasCreate");
    cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
    cublas_check(cublasSetMathMode(c.blas, CUBLAS_DEFAULT_MATH), "cublasSetMathMode");
    cusolver_check(cusolverDnCreate(&c.sol), "cusolverDnCreate");
    cusolver_check(cusolverDnSetStream(c.sol, c.stream), "cusolverDnSetStream");
    c.hscal = std::make_unique<PinnedScalars>();
    c.red.ensure(size_t(4 * 1024));
    c.scal.ensure(16);
}

template <class F>
int guard(F&& f) {
    try {
        f();
        return KRR_OK;
    } catch (const Error& e) {
        g_last_error = e.what();
        return e.status;
    } catch (const std::invalid_argument& e) {
        g_last_error = e.what();
        return KRR_ERR_INVALID_ARGUMENT;
    } catch (const std::bad_alloc& e) {
        g_last_error = std::string("host allocation failed: ") + e.what();
        return KRR_ERR_CUDA;
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return KRR_ERR_CUDA;
    }
}

Ctx* as_ctx(krr_ctx* p) {
    if (!p) fail(KRR_ERR_INVALID_ARGUMENT, "null context");
    return reinterpret_cast<Ctx*>(p);
}

}  // namespace
}  // namespace krr

using krr::Ctx;
using krr::fail;
using krr::guard;

extern "C" {

const char* krr_last_error(void) { return krr::g_last_error.c_str(); }
int krr_abi_version(void) { return KRR_B200_ABI_VERSION; }

int krr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

int krr_ctx_create(int device, krr_ctx** out) {
    return guard([&] {
        if (!out) fail(KRR_ERR_INVALID_ARGUMENT, "null output pointer");
        *out = nullptr;
        if (krr_device_count() <= device || device < 0)
            fail(KRR_ERR_CUDA, "CUDA device " + std::to_string(device) + " not available");
        auto c = std::make_unique<Ctx>();
        c->device = device;
        krr::ctx_init_common(*c);
        *out = reinterpret_cast<krr_ctx*>(c.release());
    });
}

int krr_nccl_unique_id(void* out_128_bytes) {
    return guard([&] {
        ncclUniqueId id;
        krr::nccl_check(krr::nccl().getUniqueId(&id), "ncclGetUniqueId");
        static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
        std::memcpy(out_128_bytes, &id, sizeof(id));
    });
}

int krr_ctx_create_dist(int device, int rank, int world, const void* nccl_id, krr_ctx** out) {
    return guard([&] {
        if (!out || !nccl_id) fail(KRR_ERR_INVALID_ARGUMENT, "null pointer");
        *out = nullptr;
        if (world < 1 || rank < 0 || rank >= world) fail(KRR_ERR_INVALID_ARGUMENT, "bad rank/world");
        if (krr_device_count() <= device || device < 0)
            fail(KRR_ERR_CUDA, "CUDA device " + std::to_string(device) + " not available");
        auto c = std::make_unique<Ctx>();
        c->device = device;
        c->rank = rank;
        c->world = world;
        krr::ctx_init_common(*c);
        // world == 1 with an id: a one-rank communicator (collectives are identities; the data
        // path skips them) — lets a single-GPU box exercise the NCCL plumbing
        ncclUniqueId id;
        std::memcpy(&id, nccl_id, sizeof(id));
        krr::nccl_check(krr::nccl().commInitRank(&c->comm, world, id, rank), "ncclCommInitRank");
        *out = reinterpret_cast<krr_ctx*>(c.release());
    });
}

int krr_ctx_destroy(krr_ctx* ctx) {
    return guard([&] {
        if (!ctx) return;
        delete krr::as_ctx(ctx);  // ~Ctx releases the handles, then the device buffers
    });
}

int krr_ctx_launch_count(krr_ctx* ctx, int64_t* out) {
    return guard([&] {
        (void)krr::as_ctx(ctx);
        *out = krr::g_launches.load();
    });
}

int krr_set_option(krr_ctx* ctx, const char* key, double value) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        const std::string k = key ? key : "";
        if (k == "k1_resident") {
            c.k1_resident = value != 0.0;
            c.plan.resident = c.k1_resident;
        } else if (k == "k1_warps") {
            if (value != 8.0 && value != 16.0) fail(KRR_ERR_INVALID_ARGUMENT, "k1_warps must be 8 or 16");
            c.k1_warps16 = value == 16.0;
            c.plan.warps16 = c.k1_warps16;
        } else if (k == "k1_grouped") {
            c.k1_grouped = value != 0.0;
            c.plan.grouped = c.k1_grouped;
        } else if (k == "i8_debug") {
            c.i8_debug = int(value);
        } else if (k == "k1_path") {
            if (value != 0.0 && value != 1.0 && value != 3.0 && value != -1.0)
                fail(KRR_ERR_INVALID_ARGUMENT, "k1_path must be -1 (auto), 0 (dmma), 1 (i8) or 3 (i8x)");
            c.k1_path = int(value);
            if (c.has_data && c.k1_path == 3 && c.i8x_E == 0) krr::i8x_ensure(c);
        } else if (k == "k1t_path") {
            if (value != 0.0 && value != 1.0 && value != -1.0)
                fail(KRR_ERR_INVALID_ARGUMENT, "k1t_path must be -1 (auto), 0 (dmma) or 1 (i8)");
            c.k1t_path = int(value);
        } else if (k == "batched_rhs") {
            c.batched = value != 0.0;
        } else if (k == "exp_mode") {
            c.exp_mode = value != 0.0 ? 1 : 0;
        } else if (k == "pcg_graph") {
            c.pcg_graph = value != 0.0;
        } else if (k == "poison_batched") {
            c.poison_batched = value != 0.0;
        } else if (k == "nccl_always") {
            if (!c.comm && value != 0.0) fail(KRR_ERR_STATE, "nccl_always needs a communicator (krr_ctx_create_dist)");
            c.nccl_always = value != 0.0;
        } else if (k == "emulate_world" || k == "emulate_rank") {
            if (c.world != 1) fail(KRR_ERR_STATE, "rank emulation is for single-rank contexts");
            const int iv = int(value);
            if (double(iv) != value || iv < 0 || (k == "emulate_world" && iv < 1))
                fail(KRR_ERR_INVALID_ARGUMENT, k + " must be a non-negative integer (world >= 1)");
            (k == "emulate_world" ? c.emu_world : c.emu_rank) = iv;
            c.has_data = false;  // the schedule is rebuilt by the next krr_set_data
        } else {
            fail(KRR_ERR_INVALID_ARGUMENT, "unknown option '" + k + "'");
        }
    });
}

int krr_set_precision(krr_ctx* ctx, int bits) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (bits != 64 && bits != 32) fail(KRR_ERR_INVALID_ARGUMENT, "precision must be 64 (fp64) or 32 (fp32 mode)");
        c.precision = bits;
    });
}

int krr_get_option(krr_ctx* ctx, const char* key, double* value) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        const std::string k = key ? key : "";
        if (k == "k1_path") {
            *value = c.k1_path;
        } else if (k == "precision") {
            *value = c.precision;
        } else if (k == "k1_path_effective") {  // the K1 kernel a mat-vec runs now
            krr::require_data(c);
            *value = krr::use_i8x(c) ? 3.0 : (krr::use_i8(c) ? 1.0 : (krr::use_i8T1(c) ? 2.0 : 0.0));
        } else if (k == "k1t_path") {
            *value = c.k1t_path;
        } else if (k == "k1t_path_effective") {  // the K1T kernel a 16-column batch runs now
            krr::require_data(c);
            *value = krr::use_i8T(c, 16) ? 1.0 : 0.0;
        } else if (k == "i8_supported") {
            krr::require_data(c);
            *value = c.i8_ready ? 1.0 : 0.0;
        } else if (k == "i8x_exponent") {  // K1-I8X's global exponent E of z (0: not available)
            krr::require_data(c);
            *value = c.i8x_E;
        } else if (k == "exp_mode") {
            *value = c.exp_mode;
        } else if (k == "batched_rhs") {
            *value = c.batched ? 1.0 : 0.0;
        } else if (k == "pcg_graph") {
            *value = c.pcg_graph ? 1.0 : 0.0;
        } else if (k == "build_gram_ms" || k == "build_cholesky_ms" || k == "build_trsm_ms") {
            // CUDA-event split of the last krr_precond_build (precond.cpp:23 / :26-34 / :38)
            *value = c.build_ms[k == "build_gram_ms" ? 0 : (k == "build_cholesky_ms" ? 1 : 2)];
        } else if (k == "nccl_nranks") {  // ncclCommCount of the context's communicator (1 without one)
            int nr = 1;
            if (c.comm && krr::nccl().commCount) krr::nccl_check(krr::nccl().commCount(c.comm, &nr), "ncclCommCount");
            *value = nr;
        } else if (k == "emulate_world") {
            *value = c.emu_world;
        } else if (k == "emulate_rank") {
            *value = c.emu_rank;
        } else {
            fail(KRR_ERR_INVALID_ARGUMENT, "unknown option '" + k + "'");
        }
    });
}

int krr_set_data(krr_ctx* ctx, const double* X, int64_t n, int64_t d, double sigma) {
    return guard([&] { krr::set_data(*krr::as_ctx(ctx), X, n, d, krr::gaussian_spec(sigma)); });
}

int krr_kernel_matvec_device(krr_ctx* ctx, double lambda, const double* dV, int64_t t,
                             double* dOut) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (t < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "matvec: V needs at least one column");
        c.set_device();
        const int64_t n = c.n;
        for (int64_t j = 0; j < t; ++j) {
            if (t == 1) {
                KRR_CUDA(cudaMemcpyAsync(c.vin.get(), dV, sizeof(double) * size_t(n),
                                         cudaMemcpyDeviceToDevice, c.stream));
            } else {
                krr::gather_col_launch(dV, n, t, j, c.vin.get(), c.stream);
            }
            krr::matvec_dev(c, c.vin.get(), c.vout.get(), lambda);
            if (t == 1) {
                KRR_CUDA(cudaMemcpyAsync(dOut, c.vout.get(), sizeof(double) * size_t(n),
                                         cudaMemcpyDeviceToDevice, c.stream));
            } else {
                krr::scatter_col_launch(c.vout.get(), n, t, j, dOut, c.stream);
            }
        }
        c.sync();
    });
}

int krr_kernel_matvec(krr_ctx* ctx, double lambda, const double* V, int64_t t, double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (t < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "matvec: V needs at least one column");
        c.set_device();
        const int64_t n = c.n;
        c.mat_a.ensure(size_t(n * t));
        c.mat_b.ensure(size_t(n * t));
        KRR_CUDA(cudaMemcpyAsync(c.mat_a.get(), V, sizeof(double) * size_t(n * t),
                                 cudaMemcpyHostToDevice, c.stream));
        krr::matmat_dev(c, c.mat_a.get(), t, lambda, c.mat_b.get());
        KRR_CUDA(cudaMemcpyAsync(out, c.mat_b.get(), sizeof(double) * size_t(n * t),
                                 cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int krr_predict_scores(krr_ctx* ctx, const double* Xq, int64_t m, const double* C, int64_t t,
                       double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (t < 1 || m < 0) fail(KRR_ERR_DIMENSION_MISMATCH, "predict: bad shapes");
        c.set_device();
        if (m == 0) return;
        krr::DevMem<double> q, cc, o;
        q.ensure(size_t(m * c.d));
        cc.ensure(size_t(c.n * t));
        o.ensure(size_t(m * t));
        KRR_CUDA(cudaMemcpyAsync(q.get(), Xq, sizeof(double) * size_t(m * c.d), cudaMemcpyHostToDevice,
                                 c.stream));
        KRR_CUDA(cudaMemcpyAsync(cc.get(), C, sizeof(double) * size_t(c.n * t), cudaMemcpyHostToDevice,
                                 c.stream));
        if (c.family == 1)
            krr::cross_poly_launch(q.get(), m, c.X.get(), c.n, c.d, cc.get(), t, std::sqrt(c.gamma),
                                   std::sqrt(c.offset), c.degree, o.get(), c.stream);
        else
            krr::cross_matvec_launch(q.get(), m, c.X.get(), c.n, c.d, cc.get(), t, c.scale, o.get(),
                                     c.stream);
        KRR_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * size_t(m * t), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
    });
}

// ---------------------------------------------------------------- f1: RF sketch-and-solve baseline
// train_random_features_baseline (solver.cpp:175-193) and baseline_predict_scores
// (solver.cpp:195-197): w = (Z^T Z + lambda I)^{-1} Z^T Y with Z the RFF features (K2), LLT
// with no jitter (numerics::cholesky throws NotPositiveDefinite), then the two triangular
// solves (potrs).  Single-rank.
namespace krr {
namespace {
void rf_features_dev(Ctx& c, const double* Xdev, int64_t m, const double* W, const double* b, int64_t s,
                     DevMem<double>& Z) {
    const int dp = c.plan.dp;
    const int64_t m_pad = (m + 127) / 128 * 128;
    DevMem<double> L, R, wdev, bdev, wpad;
    L.ensure(size_t(m_pad * dp));
    R.ensure(size_t(m_pad * dp));
    build_operands_launch(Xdev, m, c.d, m_pad, dp, L.get(), R.get(), c.stream);
    wdev.ensure(size_t(s * c.d));
    bdev.ensure(size_t(s));
    KRR_CUDA(cudaMemcpyAsync(wdev.get(), W, sizeof(double) * size_t(s * c.d), cudaMemcpyHostToDevice, c.stream));
    KRR_CUDA(cudaMemcpyAsync(bdev.get(), b, sizeof(double) * size_t(s), cudaMemcpyHostToDevice, c.stream));
    const int64_t s_pad = (s + 127) / 128 * 128;
    wpad.ensure(size_t(s_pad * dp));
    rff_pad_w_launch(wdev.get(), s, c.d, s_pad, dp, wpad.get(), c.stream);
    Z.ensure(size_t(m * s));
    rff_features_launch(L.get(), wpad.get(), bdev.get(), Z.get(), m, s, dp, c.stream);
    c.sync();  // temporaries are released on return
}
}  // namespace
}  // namespace krr

namespace krr {
namespace {
// w = (Z^T Z + lambda I)^{-1} Z^T Y for a device Z (n x s row-major): the solve half of
// train_random_features_baseline (solver.cpp:175-193).
void rf_baseline_solve(Ctx& c, DevMem<double>& Z, int64_t s, const double* Y, int64_t t, double lambda,
                       double* w_out) {
    {
        const int64_t n = c.n;
        krr::DevMem<double> G, Yd, Rm, work;
        krr::DevMem<int> info;
        // G = Z^T Z + lambda I (lower): Z row-major n x s == col-major Z^T (s x n)
        G.ensure(size_t(s * s));
        const double one = 1.0, zero = 0.0;
        krr::cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
        krr::cublas_check(cublasDsyrk(c.blas, CUBLAS_FILL_MODE_LOWER, CUBLAS_OP_N, int(s), int(n), &one, Z.get(),
                                      int(s), &zero, G.get(), int(s)),
                          "cublasDsyrk(Z^T Z)");
        krr::diag_add_launch(G.get(), s, lambda, c.stream);
        int lwork = 0;
        krr::cusolver_check(cusolverDnSetStream(c.sol, c.stream), "cusolverDnSetStream");
        krr::cusolver_check(
            cusolverDnDpotrf_bufferSize(c.sol, CUBLAS_FILL_MODE_LOWER, int(s), G.get(), int(s), &lwork),
            "potrf_bufferSize");
        work.ensure(size_t(std::max(1, lwork)));
        info.ensure(1);
        krr::cusolver_check(cusolverDnDpotrf(c.sol, CUBLAS_FILL_MODE_LOWER, int(s), G.get(), int(s), work.get(), lwork,
                                             info.get()),
                            "potrf");
        int hinfo = 0;
        KRR_CUDA(cudaMemcpyAsync(&hinfo, info.get(), sizeof(int), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        if (hinfo != 0) krr::fail(KRR_ERR_NOT_POSITIVE_DEFINITE, "cholesky: non-positive pivot encountered");
        // numerics.cpp:62-63 (triangular_solve's singular check) on the factor's diagonal
        std::vector<double> dg(static_cast<size_t>(s));
        KRR_CUDA(cudaMemcpy2DAsync(dg.data(), sizeof(double), G.get(), sizeof(double) * size_t(s + 1), sizeof(double),
                                   size_t(s), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
        for (double v : dg)
            if (!(std::fabs(v) >= 1e-300)) krr::fail(KRR_ERR_SINGULAR_TRIANGULAR, "triangular_solve: singular matrix");
        // rhs = Z^T Y (s x t, col-major): Y row-major n x t == col-major Y^T (t x n)
        Yd.ensure(size_t(n * t));
        KRR_CUDA(cudaMemcpyAsync(Yd.get(), Y, sizeof(double) * size_t(n * t), cudaMemcpyHostToDevice, c.stream));
        Rm.ensure(size_t(s * t));
        krr::cublas_check(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_T, int(s), int(t), int(n), &one, Z.get(), int(s),
                                      Yd.get(), int(t), &zero, Rm.get(), int(s)),
                          "cublasDgemm(Z^T Y)");
        krr::cusolver_check(cusolverDnDpotrs(c.sol, CUBLAS_FILL_MODE_LOWER, int(s), int(t), G.get(), int(s), Rm.get(),
                                             int(s), info.get()),
                            "potrs");
        std::vector<double> wcm(static_cast<size_t>(s * t));
        KRR_CUDA(cudaMemcpyAsync(wcm.data(), Rm.get(), sizeof(double) * size_t(s * t), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
        for (int64_t k = 0; k < s; ++k)
            for (int64_t j = 0; j < t; ++j) w_out[k * t + j] = wcm[size_t(j * s + k)];
    }
}
}  // namespace
}  // namespace krr

int krr_rf_baseline_train(krr_ctx* ctx, const double* W, const double* b, int64_t s, const double* Y, int64_t t,
                          double lambda, double* w_out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (!(lambda > 0.0)) krr::fail(KRR_ERR_NON_POSITIVE_LAMBDA, "baseline: lambda must be positive");
        if (s < 1) krr::fail(KRR_ERR_INVALID_ARGUMENT, "ChainSpec: s1 must be at least 1");
        if (t < 1) krr::fail(KRR_ERR_DIMENSION_MISMATCH, "baseline: Y needs at least one column");
        if (c.world != 1) krr::fail(KRR_ERR_STATE, "the random-features baseline is single-rank");
        if (c.family != 0) krr::fail(KRR_ERR_INVALID_ARGUMENT, "realize_chain: random Fourier features serve the Gaussian kernel");
        c.set_device();
        krr::DevMem<double> Z;
        krr::rf_features_dev(c, c.X.get(), c.n, W, b, s, Z);
        krr::rf_baseline_solve(c, Z, s, Y, t, lambda, w_out);
    });
}

int krr_rf_baseline_predict(krr_ctx* ctx, const double* Xq, int64_t m, const double* W, const double* b, int64_t s,
                            const double* w, int64_t t, double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (s < 1 || t < 1 || m < 0) krr::fail(KRR_ERR_DIMENSION_MISMATCH, "baseline predict: bad shapes");
        c.set_device();
        if (m == 0) return;
        krr::DevMem<double> q, Zq, wd, o;
        q.ensure(size_t(m * c.d));
        KRR_CUDA(cudaMemcpyAsync(q.get(), Xq, sizeof(double) * size_t(m * c.d), cudaMemcpyHostToDevice, c.stream));
        krr::rf_features_dev(c, q.get(), m, W, b, s, Zq);
        wd.ensure(size_t(s * t));
        KRR_CUDA(cudaMemcpyAsync(wd.get(), w, sizeof(double) * size_t(s * t), cudaMemcpyHostToDevice, c.stream));
        o.ensure(size_t(m * t));
        const double one = 1.0, zero = 0.0;
        krr::cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
        // out (m x t row-major) = Zq (m x s) w (s x t): col-major out^T = w^T Zq^T
        krr::cublas_check(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, int(t), int(m), int(s), &one, wd.get(), int(t),
                                      Zq.get(), int(s), &zero, o.get(), int(t)),
                          "cublasDgemm(Zq w)");
        KRR_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * size_t(m * t), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int krr_rff_realize(uint64_t master_seed, int64_t d, int64_t s, double sigma, double* W,
                    double* b) {
    return guard([&] { krr::rff_realize(master_seed, d, s, sigma, W, b); });
}

int krr_rff_build(krr_ctx* ctx, const double* W, const double* b, int64_t s) {
    return guard([&] { krr::rff_build(*krr::as_ctx(ctx), W, b, s); });
}

int krr_rff_download(krr_ctx* ctx, double* Zout) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (!c.has_sketch || c.has_pre) fail(KRR_ERR_STATE, "no raw sketch on the device");
        if (c.world != 1) fail(KRR_ERR_STATE, "krr_rff_download is single-rank only");
        c.set_device();
        KRR_CUDA(cudaMemcpyAsync(Zout, c.Z.get(), sizeof(double) * size_t(c.pn * c.s),
                                 cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int krr_sketch_upload(krr_ctx* ctx, const double* Z, int64_t n, int64_t s) {
    return guard([&] { krr::sketch_upload(*krr::as_ctx(ctx), Z, n, s); });
}

int krr_precond_build(krr_ctx* ctx, double lambda_p, int* jitter_used) {
    return guard([&] { krr::precond_build(*krr::as_ctx(ctx), lambda_p, jitter_used); });
}

int krr_precond_apply(krr_ctx* ctx, const double* Rm, int64_t t, double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
        if (t < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "Preconditioner: dimension mismatch");
        c.set_device();
        const int64_t n = c.pn;
        krr::DevMem<double> a, b, vi, vo;
        a.ensure(size_t(n * t));
        b.ensure(size_t(n * t));
        KRR_CUDA(cudaMemcpyAsync(a.get(), Rm, sizeof(double) * size_t(n * t), cudaMemcpyHostToDevice,
                                 c.stream));
        if (t > 1 && c.batched) {  // apply_columns: K6T over batches of T = 8 / 16 columns
            const int T = krr::batch_width(t);
            vi.ensure(size_t(n * T));
            vo.ensure(size_t(n * T));
            for (int64_t c0 = 0; c0 < t; c0 += T) {
                krr::pad_cols_launch(a.get(), n, t, c0, n, T, vi.get(), c.stream);
                krr::precondT_apply_dev(c, vi.get(), vo.get(), T);
                krr::unpad_cols_launch(vo.get(), n, t, c0, T, b.get(), c.stream);
            }
            KRR_CUDA(cudaMemcpyAsync(out, b.get(), sizeof(double) * size_t(n * t), cudaMemcpyDeviceToHost,
                                     c.stream));
            c.sync();
            return;
        }
        vi.ensure(size_t(n));
        vo.ensure(size_t(n));
        for (int64_t j = 0; j < t; ++j) {
            krr::gather_col_launch(a.get(), n, t, j, vi.get(), c.stream);
            krr::precond_apply_dev(c, vi.get(), vo.get());
            krr::scatter_col_launch(vo.get(), n, t, j, b.get(), c.stream);
        }
        KRR_CUDA(cudaMemcpyAsync(out, b.get(), sizeof(double) * size_t(n * t), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
    });
}

int krr_precond_download_u(krr_ctx* ctx, double* U) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
        if (c.world != 1) fail(KRR_ERR_STATE, "krr_precond_download_u is single-rank only");
        c.set_device();
        std::vector<double> b(static_cast<size_t>(c.pn * c.s));
        KRR_CUDA(cudaMemcpyAsync(b.data(), c.Z.get(), sizeof(double) * b.size(), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
        for (int64_t i = 0; i < c.pn; ++i)
            for (int64_t k = 0; k < c.s; ++k) U[k * c.pn + i] = b[size_t(i * c.s + k)];
    });
}

int krr_precond_read_u(krr_ctx* ctx, int64_t row0, int64_t nrows, const int64_t* cols, int64_t ncols,
                       double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
        if (row0 < 0 || nrows < 0 || row0 + nrows > c.s || ncols < 0)
            fail(KRR_ERR_DIMENSION_MISMATCH, "krr_precond_read_u: row block outside U's s rows");
        c.set_device();
        // U[k, i] lives at Z[(i - z0) * s + k] (U^T row-major over the rank's row shard)
        std::vector<double> row(static_cast<size_t>(nrows));
        for (int64_t j = 0; j < ncols; ++j) {
            const int64_t i = cols[j];
            if (i < 0 || i >= c.pn) fail(KRR_ERR_DIMENSION_MISMATCH, "krr_precond_read_u: column outside U's n");
            if (i < c.z0 || i >= c.z1) {  // another rank's shard
                for (int64_t k = 0; k < nrows; ++k) out[k * ncols + j] = 0.0;
                continue;
            }
            if (nrows > 0)
                KRR_CUDA(cudaMemcpyAsync(row.data(), c.Z.get() + (i - c.z0) * c.s + row0, sizeof(double) * size_t(nrows),
                                         cudaMemcpyDeviceToHost, c.stream));
            c.sync();
            for (int64_t k = 0; k < nrows; ++k) out[k * ncols + j] = row[size_t(k)];
        }
    });
}

int krr_precond_drop(krr_ctx* ctx) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        c.has_pre = false;
        c.has_sketch = false;
        c.Z.release();
        c.G.release();
        c.Gcopy.release();
    });
}

int krr_pcg_solve(krr_ctx* ctx, double lambda, const double* Y, int64_t t, double tau, int max_iter,
                  int use_precond, double* C, krr_rhs_stats* stats, double* residual_history,
                  int64_t* total_matvecs) {
    return guard([&] {
        krr::solve_gaussian(*krr::as_ctx(ctx), lambda, Y, t, tau, max_iter, use_precond, C, stats,
                            residual_history, total_matvecs);
    });
}

int krr_pcg_solve_operator(krr_ctx* ctx, int64_t n, krr_operator_cb apply_a, void* user_a,
                           krr_operator_cb apply_m, void* user_m, const double* y, double tau,
                           int max_iter, krr_observer_cb observer, void* user_obs, double* x,
                           krr_rhs_stats* stats, double* residual_history) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (n < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "pcg_solve: empty system");
        if (!apply_a) fail(KRR_ERR_INVALID_ARGUMENT, "pcg_solve: null operator");
        c.set_device();
        // Use private vectors sized n (independent of any data on the context).
        for (auto* v : {&c.vx, &c.vr, &c.vz, &c.vp, &c.vap, &c.vy})
            if (v->count < size_t(n)) {
                v->ensure(size_t(n));
                KRR_CUDA(cudaMemsetAsync(v->get(), 0, sizeof(double) * size_t(n), c.stream));
            }
        std::vector<double> hin(static_cast<size_t>(n)), hout(static_cast<size_t>(n));
        auto host_op = [&](krr_operator_cb cb, void* user) {
            return krr::DevOp([&, cb, user](const double* din, double* dout) {
                KRR_CUDA(cudaMemcpyAsync(hin.data(), din, sizeof(double) * size_t(n),
                                         cudaMemcpyDeviceToHost, c.stream));
                c.sync();
                if (cb(user, hin.data(), hout.data(), n) != 0)
                    fail(KRR_ERR_CALLBACK, "operator callback failed");
                KRR_CUDA(cudaMemcpyAsync(dout, hout.data(), sizeof(double) * size_t(n),
                                         cudaMemcpyHostToDevice, c.stream));
                c.sync();
            });
        };
        const krr::DevOp A = host_op(apply_a, user_a);
        const krr::DevOp M = apply_m ? host_op(apply_m, user_m) : krr::DevOp();
        std::vector<double> hx(static_cast<size_t>(n));
        const krr::HostObserver obs = [&](int it, const double* dx) {
            KRR_CUDA(cudaMemcpyAsync(hx.data(), dx, sizeof(double) * size_t(n), cudaMemcpyDeviceToHost,
                                     c.stream));
            c.sync();
            observer(user_obs, it, hx.data(), n);
        };
        KRR_CUDA(cudaMemcpyAsync(c.vy.get(), y, sizeof(double) * size_t(n), cudaMemcpyHostToDevice,
                                 c.stream));
        const krr::PcgOut o = krr::pcg_core(c, n, A, apply_m ? &M : nullptr, c.vy.get(), tau, max_iter,
                                            residual_history, observer ? &obs : nullptr, false);
        KRR_CUDA(cudaMemcpyAsync(x, c.vx.get(), sizeof(double) * size_t(n), cudaMemcpyDeviceToHost,
                                 c.stream));
        c.sync();
        stats->iterations = o.iterations;
        stats->converged = o.converged;
        stats->final_residual = o.final_residual;
    });
}

int krr_train(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const double* Y, int64_t t,
              double sigma, double lambda, double lambda_p, int64_t s, uint64_t master_seed, double tau,
              int max_iter, double* C, krr_rhs_stats* stats, double* residual_history,
              int64_t* total_matvecs, double* phase_ms) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (n < 1) fail(KRR_ERR_INVALID_ARGUMENT, "train: dataset is empty");          // solver.cpp:97
        if (!(lambda > 0.0)) fail(KRR_ERR_NON_POSITIVE_LAMBDA, "train: lambda must be positive");
        if (s < 1) fail(KRR_ERR_INVALID_ARGUMENT, "ChainSpec: s1 must be at least 1");
        const double lp = lambda_p > 0.0 ? lambda_p : lambda;                           // solver.cpp:102
        krr::set_data(c, X, n, d, krr::gaussian_spec(sigma));
        std::vector<double> W(static_cast<size_t>(s * d)), b(static_cast<size_t>(s));
        krr::rff_realize(master_seed, d, s, sigma, W.data(), b.data());
        krr::Events ev(4);
        KRR_CUDA(cudaEventRecord(ev[0], c.stream));
        krr::rff_build(c, W.data(), b.data(), s);
        KRR_CUDA(cudaEventRecord(ev[1], c.stream));
        krr::precond_build(c, lp, nullptr);
        KRR_CUDA(cudaEventRecord(ev[2], c.stream));
        krr::solve_gaussian(c, lambda, Y, t, tau, max_iter, 1, C, stats, residual_history,
                            total_matvecs);
        KRR_CUDA(cudaEventRecord(ev[3], c.stream));
        KRR_CUDA(cudaEventSynchronize(ev[3]));
        if (phase_ms) {
            float a = 0, b2 = 0, c3 = 0, tot = 0;
            KRR_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
            KRR_CUDA(cudaEventElapsedTime(&b2, ev[1], ev[2]));
            KRR_CUDA(cudaEventElapsedTime(&c3, ev[2], ev[3]));
            KRR_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[3]));
            phase_ms[0] = a;
            phase_ms[1] = b2;
            phase_ms[2] = c3;
            phase_ms[3] = tot;
        }
    });
}

int krr_schedule(int64_t n, int world, int rank, int64_t* super_rows, int64_t* num_super,
                 int32_t* tiles, int64_t max_tiles, int64_t* num_tiles) {
    return guard([&] {
        const krr::Schedule s = krr::make_schedule(n, world, rank);
        if (super_rows) *super_rows = s.st;
        if (num_super) *num_super = s.ns;
        const int64_t nt = int64_t(s.tiles.size() / 2);
        if (num_tiles) *num_tiles = nt;
        if (tiles) {
            if (max_tiles < nt) fail(KRR_ERR_DIMENSION_MISMATCH, "krr_schedule: tile buffer too small");
            std::memcpy(tiles, s.tiles.data(), sizeof(int32_t) * s.tiles.size());
        }
    });
}

int krr_shard_rows(int64_t n, int world, int rank, int64_t* row_begin, int64_t* row_end) {
    return guard([&] { krr::shard_rows(n, world, rank, row_begin, row_end); });
}

int krr_generate_config(int cfg, int64_t n, int64_t d, int64_t t, uint64_t seed, double* X,
                        double* Y) {
    return guard([&] { krr::generate_config(cfg, n, d, t, seed, X, Y); });
}

int krr_quality_test(krr_ctx* ctx, double lambda, krr_quality_report* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        *out = krr::quality_test_dev(c, lambda);
    });
}

int krr_model_save(const char* path, double sigma, double lambda, uint64_t seed, const double* label_map,
                   int64_t nlabels, const double* X, int64_t n, int64_t d, const double* C, int64_t t) {
    return guard([&] { krr::model_save(path, 0, sigma, 0.0, 0.0, 0, lambda, seed, label_map, nlabels, X, n, d, C, t); });
}

int krr_model_info(const char* path, int64_t* n, int64_t* d, int64_t* t, int64_t* nlabels, double* sigma,
                   double* lambda, uint64_t* seed) {
    return guard([&] {
        const krr::ModelMeta m = krr::model_info(path);
        *n = m.n;
        *d = m.d;
        *t = m.t;
        *nlabels = int64_t(m.label_map.size());
        *sigma = m.sigma;
        *lambda = m.lambda;
        *seed = m.seed;
    });
}

int krr_model_load(const char* path, double* label_map, double* X, double* C) {
    return guard([&] { krr::model_load(path, label_map, X, C); });
}

int krr_rlsc_encode(const int32_t* classes, int64_t n, int32_t num_classes, double* Y) {
    return guard([&] { krr::rlsc_encode(classes, n, num_classes, Y); });
}

int krr_bench_matvec(krr_ctx* ctx, double lambda, int steps, double* total_ms, double* k1_ms) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (steps < 1) fail(KRR_ERR_INVALID_ARGUMENT, "steps must be positive");
        c.set_device();
        {
            std::vector<double> v(size_t(c.plan.n_pad), 0.0);
            std::mt19937_64 gen(12345);
            std::normal_distribution<double> nd(0.0, 1.0);
            for (int64_t i = 0; i < c.n; ++i) v[size_t(i)] = nd(gen);
            KRR_CUDA(cudaMemcpyAsync(c.vin.get(), v.data(), sizeof(double) * v.size(),
                                     cudaMemcpyHostToDevice, c.stream));
            c.sync();
        }
        krr::Events ev(size_t(2 * steps + 2));
        KRR_CUDA(cudaEventRecord(ev[0], c.stream));
        for (int k = 0; k < steps; ++k)
            krr::matvec_dev(c, c.vin.get(), c.vout.get(), lambda, ev[size_t(2 + 2 * k)],
                            ev[size_t(3 + 2 * k)]);
        KRR_CUDA(cudaEventRecord(ev[1], c.stream));
        KRR_CUDA(cudaEventSynchronize(ev[1]));
        float tot = 0.f;
        KRR_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[1]));
        double k1 = 0.0;
        for (int k = 0; k < steps; ++k) {
            float ms = 0.f;
            KRR_CUDA(cudaEventElapsedTime(&ms, ev[size_t(2 + 2 * k)], ev[size_t(3 + 2 * k)]));
            k1 += ms;
        }
        *total_ms = tot;
        *k1_ms = k1 / steps;
    });
}

}  // extern "C"

// ============================================================================= SURVEY 8f4
// Kernel families and sketch chains: realize_chain (sketches.cpp:213-242) with the host's
// libstdc++ draws, SketchChain::apply_rows (sketches.cpp:194-211) on the device.
namespace krr {
namespace {

constexpr int kInvalid = KRR_ERR_INVALID_ARGUMENT;

struct ChainOwned {
    std::vector<double> w, b, ts_sign, srht_sign, proj;
    std::vector<uint32_t> ts_hash;
    std::vector<int64_t> srht_rows;
    krr_chain_tables t{};
};

void validate_chain(const krr_chain_spec& sp) {  // ChainSpec::validate (sketches.cpp:155-165)
    if (sp.first != 0 && sp.first != 1) fail(kInvalid, "ChainSpec: unknown first stage");
    if (sp.s1 < 1) fail(kInvalid, "ChainSpec: s1 must be at least 1");
    if (sp.s2 < 0 || sp.s3 < 0) fail(kInvalid, "ChainSpec: stage sizes must be non-negative");
    int64_t prev = sp.s1;
    if (sp.s2 > 0) {
        if (sp.s2 > prev) fail(kInvalid, "ChainSpec: stage sizes must be non-increasing");
        prev = sp.s2;
    }
    if (sp.s3 > 0 && sp.s3 > prev) fail(kInvalid, "ChainSpec: stage sizes must be non-increasing");
}

int64_t chain_out_dim(int64_t s1, int64_t s2, int64_t s3) { return s3 > 0 ? s3 : (s2 > 0 ? s2 : s1); }

krr_chain_spec chain_scaled_to(const krr_chain_spec& sp, int64_t target) {  // sketches.cpp:173-192
    validate_chain(sp);
    if (target < 1) fail(kInvalid, "ChainSpec: target size must be at least 1");
    const double factor = double(target) / double(chain_out_dim(sp.s1, sp.s2, sp.s3));
    auto scale = [&](int64_t v) { return std::max<int64_t>(target, int64_t(std::ceil(double(v) * factor))); };
    krr_chain_spec o = sp;
    o.s1 = scale(sp.s1);
    if (sp.s2 > 0) o.s2 = scale(sp.s2);
    if (sp.s3 > 0) o.s3 = scale(sp.s3);
    if (o.s3 > 0)
        o.s3 = target;
    else if (o.s2 > 0)
        o.s2 = target;
    else
        o.s1 = target;
    validate_chain(o);
    return o;
}

void check_family(const Ctx& c, int first) {  // sketches.cpp:217-220
    if (first == 0 && c.family != 0) fail(kInvalid, "realize_chain: random Fourier features serve the Gaussian kernel");
    if (first == 1 && c.family != 1) fail(kInvalid, "realize_chain: TensorSketch serves the polynomial kernel");
}

void realize_chain_host(const Ctx& c, const krr_chain_spec& sp, uint64_t master, ChainOwned& o) {
    validate_chain(sp);
    check_family(c, sp.first);
    krr_chain_tables& t = o.t;
    t = krr_chain_tables{};
    t.first = sp.first;
    t.s1 = sp.s1;
    t.s2 = sp.s2;
    t.s3 = sp.s3;
    if (sp.first == 0) {
        t.in_dim = c.d;
        o.w.resize(size_t(sp.s1 * c.d));
        o.b.resize(size_t(sp.s1));
        rff_realize(master, c.d, sp.s1, c.sigma, o.w.data(), o.b.data());  // stage_seed(master, 0) inside
        t.rff_w = o.w.data();
        t.rff_b = o.b.data();
    } else {
        t.in_dim = c.d + 1;  // augmented representation (sketches.cpp:229)
        t.degree = c.degree;
        o.ts_hash.resize(size_t(c.degree * t.in_dim));
        o.ts_sign.resize(size_t(c.degree * t.in_dim));
        tensorsketch_realize(stage_seed(master, 0), t.in_dim, sp.s1, c.degree, o.ts_hash.data(), o.ts_sign.data());
        t.ts_hash = o.ts_hash.data();
        t.ts_sign = o.ts_sign.data();
    }
    int64_t prev = sp.s1;
    if (sp.s2 > 0) {
        o.srht_sign.resize(size_t(next_pow2(prev)));
        o.srht_rows.resize(size_t(sp.s2));
        srht_realize(stage_seed(master, 1), prev, sp.s2, o.srht_sign.data(), o.srht_rows.data());
        t.srht_sign = o.srht_sign.data();
        t.srht_rows = o.srht_rows.data();
        prev = sp.s2;
    }
    if (sp.s3 > 0) {
        o.proj.resize(size_t(sp.s3 * prev));
        gaussmap_realize(stage_seed(master, 2), prev, sp.s3, o.proj.data());
        t.gauss_proj = o.proj.data();
    }
}

void check_tables(const Ctx& c, const krr_chain_tables& t) {
    validate_chain(krr_chain_spec{t.first, 0, t.s1, t.s2, t.s3});
    check_family(c, t.first);
    if (t.first == 0) {
        if (t.in_dim != c.d) fail(KRR_ERR_DIMENSION_MISMATCH, "RffMap: input dimension mismatch");
        if (!t.rff_w || !t.rff_b) fail(kInvalid, "chain tables: RFF tables missing");
    } else {
        if (t.in_dim != c.d + 1) fail(KRR_ERR_DIMENSION_MISMATCH, "TensorSketchMap: input dimension mismatch");
        if (t.degree != c.degree) fail(kInvalid, "chain tables: TensorSketch degree differs from the kernel's");
        if (!t.ts_hash || !t.ts_sign) fail(kInvalid, "chain tables: TensorSketch tables missing");
        for (int64_t i = 0; i < int64_t(t.degree) * t.in_dim; ++i)
            if (int64_t(t.ts_hash[i]) >= t.s1) fail(kInvalid, "TensorSketchMap: hash bucket out of range");
    }
    if (t.s2 > 0) {
        if (!t.srht_sign || !t.srht_rows) fail(kInvalid, "chain tables: SRHT tables missing");
        const int64_t P = next_pow2(t.s1);
        for (int64_t i = 0; i < t.s2; ++i)
            if (t.srht_rows[i] < 0 || t.srht_rows[i] >= P) fail(kInvalid, "SrhtMap: sampled row out of range");
    }
    if (t.s3 > 0 && !t.gauss_proj) fail(kInvalid, "chain tables: Gaussian projection missing");
}

template <typename T>
void upload(DevMem<T>& dst, const T* src, size_t count, cudaStream_t st) {
    dst.ensure(std::max<size_t>(1, count));
    if (count) KRR_CUDA(cudaMemcpyAsync(dst.get(), src, sizeof(T) * count, cudaMemcpyHostToDevice, st));
}

// Zout (m x out_dim, row-major) = SketchChain::apply_rows of the device rows Xrows (m x d).
void chain_apply_dev(Ctx& c, const krr_chain_tables& t, const double* Xrows, int64_t m, DevMem<double>& Zout) {
    check_tables(c, t);
    const int64_t out = chain_out_dim(t.s1, t.s2, t.s3);
    Zout.ensure(size_t(std::max<int64_t>(1, m * out)));
    if (m == 0) return;
    DevMem<double> z1, z2;
    DevMem<double>& d1 = (t.s2 == 0 && t.s3 == 0) ? Zout : z1;
    if (t.first == 0) {
        rf_features_dev(c, Xrows, m, t.rff_w, t.rff_b, t.s1, d1);  // K2
    } else {
        const int dp = c.plan.dp;
        DevMem<double> A;
        A.ensure(size_t(m * dp));
        poly_operands_launch(Xrows, m, c.d, m, dp, std::sqrt(c.gamma), std::sqrt(c.offset), c.degree, A.get(),
                             nullptr, nullptr, c.stream);
        DevMem<uint32_t> h;
        DevMem<double> g;
        upload(h, t.ts_hash, size_t(t.degree * t.in_dim), c.stream);
        upload(g, t.ts_sign, size_t(t.degree * t.in_dim), c.stream);
        const bool p2 = (t.s1 & (t.s1 - 1)) == 0;  // sketches.cpp:79-82
        const int64_t P = p2 ? t.s1 : next_pow2(int64_t(t.degree) * (t.s1 - 1) + 1);
        std::vector<double> tw(size_t(2 * std::max<int64_t>(1, P - 1)));
        DevMem<double2> twf, twi, scr;
        fft_twiddles(P, false, tw.data());
        upload(twf, reinterpret_cast<const double2*>(tw.data()), size_t(P - 1), c.stream);
        c.sync();  // tw is reused for the inverse table
        fft_twiddles(P, true, tw.data());
        upload(twi, reinterpret_cast<const double2*>(tw.data()), size_t(P - 1), c.stream);
        const size_t ns = tensorsketch_scratch(P, m);
        if (ns) scr.ensure(ns);
        d1.ensure(size_t(m * t.s1));
        tensorsketch_launch(h.get(), g.get(), twf.get(), twi.get(), t.in_dim, t.s1, P, t.degree, A.get(), dp, m,
                            d1.get(), ns ? scr.get() : nullptr, c.stream);
        c.sync();
    }
    DevMem<double>* cur = &d1;
    int64_t prev = t.s1;
    if (t.s2 > 0) {
        DevMem<double>& d2 = t.s3 == 0 ? Zout : z2;
        const int64_t P = next_pow2(prev);
        DevMem<double> sg, scr;
        DevMem<int64_t> rows;
        upload(sg, t.srht_sign, size_t(P), c.stream);
        upload(rows, t.srht_rows, size_t(t.s2), c.stream);
        const size_t ns = srht_scratch(P, m);
        if (ns) scr.ensure(ns);
        d2.ensure(size_t(m * t.s2));
        srht_launch(sg.get(), rows.get(), prev, P, t.s2, 1.0 / std::sqrt(double(t.s2)), cur->get(), m, d2.get(),
                    ns ? scr.get() : nullptr, c.stream);
        c.sync();
        cur = &d2;
        prev = t.s2;
    }
    if (t.s3 > 0) {
        DevMem<double> pj;
        upload(pj, t.gauss_proj, size_t(t.s3 * prev), c.stream);
        const double one = 1.0, zero = 0.0;
        cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
        // Z3^T (s3 x m, col-major) = proj (s3 x prev, row-major == col-major prev x s3, op T) . Z2^T
        cublas_check(cublasDgemm(c.blas, CUBLAS_OP_T, CUBLAS_OP_N, int(t.s3), int(m), int(prev), &one, pj.get(),
                                 int(prev), cur->get(), int(prev), &zero, Zout.get(), int(t.s3)),
                     "cublasDgemm(chain Gaussian stage)");
        div_launch(Zout.get(), m * t.s3, std::sqrt(double(t.s3)), c.stream);
        c.sync();
    }
}

// krr_rff_build generalised: the context's own rows [z0, z1) -> resident sketch Z.
void chain_build(Ctx& c, const krr_chain_tables& t) {
    require_data(c);
    c.set_device();
    check_tables(c, t);
    sketch_alloc(c, c.n, chain_out_dim(t.s1, t.s2, t.s3));
    chain_apply_dev(c, t, c.X.get() + c.z0 * c.d, c.z1 - c.z0, c.Z);
    c.sync();
    c.has_sketch = true;
}

void adaptive_dev(Ctx& c, const krr_chain_spec& tmpl, double lambda, double lambda_p, int64_t s0, int64_t s_max,
                  uint64_t master_seed, krr_quality_report* history, int max_history, int* n_history,
                  int64_t* final_size, int* passed, int* jitter_used) {
    require_data(c);
    if (s0 < 1) fail(kInvalid, "adaptive_build: s0 must be at least 1");
    if (s_max < s0) fail(kInvalid, "adaptive_build: s_max must be >= s0");
    validate_chain(tmpl);
    check_family(c, tmpl.first);
    const double lp = lambda_p > 0.0 ? lambda_p : lambda;
    int64_t s = s0;
    int nh = 0;
    bool ok = false;
    for (int attempt = 0;; ++attempt) {
        const uint64_t seed = master_seed + uint64_t(attempt) * kAttemptSeedStride;
        ChainOwned o;
        realize_chain_host(c, chain_scaled_to(tmpl, s), seed, o);
        chain_build(c, o.t);
        const krr_quality_report rep = quality_test_dev(c, lambda);
        if (history && nh < max_history) history[nh] = rep;
        ++nh;
        if (final_size) *final_size = s;
        if (rep.passed) {
            ok = true;
            break;
        }
        if (s >= s_max) break;
        s = std::min(2 * s, s_max);
    }
    if (n_history) *n_history = nh;
    if (passed) *passed = ok ? 1 : 0;
    precond_build(c, lp, jitter_used);
}

// solve_regularized (solver.cpp:69-94) on a caller-supplied dense K, the reference's own
// signature: A v = K v + lambda v by cuBLAS DGEMV (K is symmetric, so its row-major buffer is
// read as column-major) plus the lambda term; M = the context's Woodbury preconditioner.
void solve_dense_dev(Ctx& c, const double* K, int64_t n, const double* Y, int64_t t, double lambda, int use_precond,
                     double tau, int max_iter, double* C, krr_rhs_stats* stats, double* hist,
                     int64_t* total_matvecs) {
    if (n < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "solve_regularized: K must be non-empty");
    if (t < 1) fail(KRR_ERR_DIMENSION_MISMATCH, "solve_regularized: K and Y dimensions do not match");
    if (!(lambda > 0.0)) fail(KRR_ERR_NON_POSITIVE_LAMBDA, "solve_regularized: lambda must be positive");
    if (c.world != 1) fail(KRR_ERR_STATE, "the dense-K solve is single-rank");
    if (use_precond) {
        if (!c.has_pre) fail(KRR_ERR_STATE, "no preconditioner built");
        if (c.pn != n) fail(KRR_ERR_DIMENSION_MISMATCH, "Preconditioner: dimension mismatch");
    }
    c.set_device();
    DevMem<double> Kd;
    upload(Kd, K, size_t(n * n), c.stream);
    for (auto* v : {&c.vx, &c.vr, &c.vz, &c.vp, &c.vap, &c.vy}) v->ensure(size_t(n));
    c.red.ensure(size_t(4 * 1024));
    c.mat_a.ensure(size_t(n * t));
    c.mat_b.ensure(size_t(n * t));
    KRR_CUDA(cudaMemcpyAsync(c.mat_a.get(), Y, sizeof(double) * size_t(n * t), cudaMemcpyHostToDevice, c.stream));
    cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
    const double* kd = Kd.get();
    const DevOp A = [&c, kd, n, lambda](const double* din, double* dout) {
        const double one = 1.0, zero = 0.0;
        cublas_check(cublasDgemv(c.blas, CUBLAS_OP_N, int(n), int(n), &one, kd, int(n), din, 1, &zero, dout, 1),
                     "cublasDgemv(K v)");
        add_scaled_launch(dout, din, lambda, n, c.stream);
    };
    const DevOp M = precond_op(c);
    int64_t total = 0;
    for (int64_t j = 0; j < t; ++j) {
        gather_col_launch(c.mat_a.get(), n, t, j, c.vy.get(), c.stream);
        const PcgOut o = pcg_core(c, n, A, use_precond ? &M : nullptr, c.vy.get(), tau, max_iter,
                                  hist ? hist + j * max_iter : nullptr, nullptr, true);
        scatter_col_launch(c.vx.get(), n, t, j, c.mat_b.get(), c.stream);
        stats[j].iterations = o.iterations;
        stats[j].converged = o.converged;
        stats[j].final_residual = o.final_residual;
        total += o.iterations;
    }
    KRR_CUDA(cudaMemcpyAsync(C, c.mat_b.get(), sizeof(double) * size_t(n * t), cudaMemcpyDeviceToHost, c.stream));
    c.sync();
    if (total_matvecs) *total_matvecs = total;
}

}  // namespace
}  // namespace krr

extern "C" {

int krr_solve_regularized_dense(krr_ctx* ctx, const double* K, int64_t n, const double* Y, int64_t t, double lambda,
                                int use_precond, double tau, int max_iter, double* C, krr_rhs_stats* stats,
                                double* residual_history, int64_t* total_matvecs) {
    return guard([&] {
        krr::solve_dense_dev(*krr::as_ctx(ctx), K, n, Y, t, lambda, use_precond, tau, max_iter, C, stats,
                             residual_history, total_matvecs);
    });
}

int krr_set_data_kernel(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const krr_kernel_spec* kernel) {
    return guard([&] {
        if (!kernel) fail(KRR_ERR_INVALID_ARGUMENT, "null kernel spec");
        krr::set_data(*krr::as_ctx(ctx), X, n, d, *kernel);
    });
}

int krr_tensorsketch_realize(uint64_t seed, int64_t in_dim, int64_t s, int degree, uint32_t* hash, double* sign) {
    return guard([&] { krr::tensorsketch_realize(seed, in_dim, s, degree, hash, sign); });
}

int krr_srht_realize(uint64_t seed, int64_t in_dim, int64_t s, double* sign, int64_t* rows) {
    return guard([&] { krr::srht_realize(seed, in_dim, s, sign, rows); });
}

int krr_gaussmap_realize(uint64_t seed, int64_t in_dim, int64_t s, double* proj) {
    return guard([&] { krr::gaussmap_realize(seed, in_dim, s, proj); });
}

int krr_chain_apply(krr_ctx* ctx, const krr_chain_tables* tables, const double* Xq, int64_t m, double* Z) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (!tables) fail(KRR_ERR_INVALID_ARGUMENT, "null chain tables");
        if (m < 0) fail(KRR_ERR_DIMENSION_MISMATCH, "chain apply: bad shapes");
        c.set_device();
        krr::DevMem<double> q, z;
        krr::upload(q, Xq, size_t(m * c.d), c.stream);
        krr::chain_apply_dev(c, *tables, q.get(), m, z);
        const int64_t out = krr::chain_out_dim(tables->s1, tables->s2, tables->s3);
        if (m > 0)
            KRR_CUDA(cudaMemcpyAsync(Z, z.get(), sizeof(double) * size_t(m * out), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int krr_chain_build(krr_ctx* ctx, const krr_chain_tables* tables) {
    return guard([&] {
        if (!tables) fail(KRR_ERR_INVALID_ARGUMENT, "null chain tables");
        krr::chain_build(*krr::as_ctx(ctx), *tables);
    });
}

int krr_chain_build_seeded(krr_ctx* ctx, const krr_chain_spec* spec, uint64_t master_seed) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (!spec) fail(KRR_ERR_INVALID_ARGUMENT, "null chain spec");
        krr::ChainOwned o;
        krr::realize_chain_host(c, *spec, master_seed, o);
        krr::chain_build(c, o.t);
    });
}

int krr_chain_scaled_to(const krr_chain_spec* spec, int64_t target, krr_chain_spec* out) {
    return guard([&] {
        if (!spec || !out) fail(KRR_ERR_INVALID_ARGUMENT, "null chain spec");
        *out = krr::chain_scaled_to(*spec, target);
    });
}

int krr_train_ex(krr_ctx* ctx, const double* X, int64_t n, int64_t d, const double* Y, int64_t t,
                 const krr_kernel_spec* kernel, const krr_chain_spec* chain, double lambda, double lambda_p,
                 uint64_t master_seed, double tau, int max_iter, double* C, krr_rhs_stats* stats,
                 double* residual_history, int64_t* total_matvecs, double* phase_ms) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        if (!kernel || !chain) fail(KRR_ERR_INVALID_ARGUMENT, "null kernel or chain spec");
        if (n < 1) fail(KRR_ERR_INVALID_ARGUMENT, "train: dataset is empty");          // solver.cpp:97
        if (!(lambda > 0.0)) fail(KRR_ERR_NON_POSITIVE_LAMBDA, "train: lambda must be positive");
        const double lp = lambda_p > 0.0 ? lambda_p : lambda;                           // solver.cpp:102
        krr::validate_chain(*chain);
        krr::set_data(c, X, n, d, *kernel);
        krr::ChainOwned o;
        krr::realize_chain_host(c, *chain, master_seed, o);
        krr::Events ev(4);
        KRR_CUDA(cudaEventRecord(ev[0], c.stream));
        krr::chain_build(c, o.t);
        KRR_CUDA(cudaEventRecord(ev[1], c.stream));
        krr::precond_build(c, lp, nullptr);
        KRR_CUDA(cudaEventRecord(ev[2], c.stream));
        krr::solve_gaussian(c, lambda, Y, t, tau, max_iter, 1, C, stats, residual_history, total_matvecs);
        KRR_CUDA(cudaEventRecord(ev[3], c.stream));
        KRR_CUDA(cudaEventSynchronize(ev[3]));
        if (phase_ms) {
            float a = 0, b = 0, cc = 0, tot = 0;
            KRR_CUDA(cudaEventElapsedTime(&a, ev[0], ev[1]));
            KRR_CUDA(cudaEventElapsedTime(&b, ev[1], ev[2]));
            KRR_CUDA(cudaEventElapsedTime(&cc, ev[2], ev[3]));
            KRR_CUDA(cudaEventElapsedTime(&tot, ev[0], ev[3]));
            phase_ms[0] = a;
            phase_ms[1] = b;
            phase_ms[2] = cc;
            phase_ms[3] = tot;
        }
    });
}

int krr_adaptive_build_ex(krr_ctx* ctx, const krr_chain_spec* chain_template, double lambda, double lambda_p,
                          int64_t s0, int64_t s_max, uint64_t master_seed, krr_quality_report* history,
                          int max_history, int* n_history, int64_t* final_size, int* passed, int* jitter_used) {
    return guard([&] {
        if (!chain_template) fail(KRR_ERR_INVALID_ARGUMENT, "null chain spec");
        krr::adaptive_dev(*krr::as_ctx(ctx), *chain_template, lambda, lambda_p, s0, s_max, master_seed, history,
                          max_history, n_history, final_size, passed, jitter_used);
    });
}

int krr_adaptive_build(krr_ctx* ctx, double lambda, double lambda_p, int64_t s0, int64_t s_max,
                       uint64_t master_seed, krr_quality_report* history, int max_history, int* n_history,
                       int64_t* final_size, int* passed, int* jitter_used) {
    return guard([&] {
        krr_chain_spec rff{};  // the RandomFourier single-stage template (scaled_to(s) gives s1 = s)
        rff.first = 0;
        rff.s1 = std::max<int64_t>(1, s0);
        krr::adaptive_dev(*krr::as_ctx(ctx), rff, lambda, lambda_p, s0, s_max, master_seed, history, max_history,
                          n_history, final_size, passed, jitter_used);
    });
}

int krr_rf_baseline_train_ex(krr_ctx* ctx, const krr_chain_tables* tables, const double* Y, int64_t t,
                             double lambda, double* w_out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (!tables) fail(KRR_ERR_INVALID_ARGUMENT, "null chain tables");
        if (!(lambda > 0.0)) krr::fail(KRR_ERR_NON_POSITIVE_LAMBDA, "baseline: lambda must be positive");
        if (t < 1) krr::fail(KRR_ERR_DIMENSION_MISMATCH, "baseline: Y needs at least one column");
        if (c.world != 1) krr::fail(KRR_ERR_STATE, "the random-features baseline is single-rank");
        c.set_device();
        krr::DevMem<double> Z;
        krr::chain_apply_dev(c, *tables, c.X.get(), c.n, Z);
        krr::rf_baseline_solve(c, Z, krr::chain_out_dim(tables->s1, tables->s2, tables->s3), Y, t, lambda, w_out);
    });
}

int krr_rf_baseline_predict_ex(krr_ctx* ctx, const krr_chain_tables* tables, const double* Xq, int64_t m,
                               const double* w, int64_t t, double* out) {
    return guard([&] {
        Ctx& c = *krr::as_ctx(ctx);
        krr::require_data(c);
        if (!tables) fail(KRR_ERR_INVALID_ARGUMENT, "null chain tables");
        if (t < 1 || m < 0) krr::fail(KRR_ERR_DIMENSION_MISMATCH, "baseline predict: bad shapes");
        c.set_device();
        if (m == 0) return;
        const int64_t s = krr::chain_out_dim(tables->s1, tables->s2, tables->s3);
        krr::DevMem<double> q, Zq, wd, o;
        krr::upload(q, Xq, size_t(m * c.d), c.stream);
        krr::chain_apply_dev(c, *tables, q.get(), m, Zq);
        krr::upload(wd, w, size_t(s * t), c.stream);
        o.ensure(size_t(m * t));
        const double one = 1.0, zero = 0.0;
        krr::cublas_check(cublasSetStream(c.blas, c.stream), "cublasSetStream");
        krr::cublas_check(cublasDgemm(c.blas, CUBLAS_OP_N, CUBLAS_OP_N, int(t), int(m), int(s), &one, wd.get(), int(t),
                                      Zq.get(), int(s), &zero, o.get(), int(t)),
                          "cublasDgemm(Zq w)");
        KRR_CUDA(cudaMemcpyAsync(out, o.get(), sizeof(double) * size_t(m * t), cudaMemcpyDeviceToHost, c.stream));
        c.sync();
    });
}

int krr_model_save_ex(const char* path, const krr_kernel_spec* kernel, double lambda, uint64_t seed,
                      const double* label_map, int64_t nlabels, const double* X, int64_t n, int64_t d,
                      const double* C, int64_t t) {
    return guard([&] {
        if (!kernel) fail(KRR_ERR_INVALID_ARGUMENT, "null kernel spec");
        krr::validate_kernel(*kernel);
        krr::model_save(path, kernel->family, kernel->sigma, kernel->gamma, kernel->offset, kernel->degree, lambda,
                        seed, label_map, nlabels, X, n, d, C, t);
    });
}

int krr_model_kernel(const char* path, krr_kernel_spec* kernel) {
    return guard([&] {
        if (!kernel) fail(KRR_ERR_INVALID_ARGUMENT, "null kernel spec");
        const krr::ModelMeta m = krr::model_info(path);
        *kernel = krr_kernel_spec{};
        kernel->family = m.family;
        kernel->sigma = m.sigma;
        kernel->gamma = m.gamma;
        kernel->offset = m.offset;
        kernel->degree = m.degree;
    });
}

}  // extern "C"
