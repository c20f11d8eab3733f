// C++ caller of the C-ABI (include/krr_b200.h) without Python: the reference's own
// solver tests (test_solver.cpp:25-63, :126-147) rewritten against the B200 library.
// Built by __graft_entry__.build() into examples/cpp_dropin; run by
// tests/test_gpu_cpp_dropin.py.  Exit code 0 = all checks passed.
#include <krr_b200.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <vector>

namespace {

int failures = 0;

void check(bool ok, const char* what) {
    std::printf("%s %s\n", ok ? "PASS" : "FAIL", what);
    if (!ok) ++failures;
}

void must(int st, const char* what) {
    if (st != KRR_OK) {
        std::printf("FAIL %s: status %d: %s\n", what, st, krr_last_error());
        ++failures;
    }
}

struct Dense {
    std::vector<double> a;
    int64_t n;
};

int dense_op(void* user, const double* in, double* out, int64_t n) {
    const auto* m = static_cast<const Dense*>(user);
    for (int64_t i = 0; i < n; ++i) {
        double s = 0.0;
        for (int64_t j = 0; j < n; ++j) s += m->a[size_t(i * n + j)] * in[j];
        out[i] = s;
    }
    return 0;
}

std::vector<double> random_matrix(int64_t rows, int64_t cols, uint64_t seed) {
    std::mt19937_64 gen(seed);  // tests/support/oracles.cpp:87-94
    std::normal_distribution<double> normal(0.0, 1.0);
    std::vector<double> m(static_cast<size_t>(rows * cols));
    for (auto& v : m) v = normal(gen);
    return m;
}

}  // namespace

int main() {
    if (krr_device_count() < 1) {
        std::printf("no CUDA device\n");
        return 2;
    }
    krr_ctx* ctx = nullptr;
    must(krr_ctx_create(0, &ctx), "krr_ctx_create");
    if (!ctx) return 1;

    // pcg solves a 2x2 diagonal system in two iterations (test_solver.cpp:25-35)
    {
        Dense a{{3.0, 0.0, 0.0, 2.0}, 2};
        const double y[2] = {3.0, 2.0};
        double x[2] = {0, 0};
        krr_rhs_stats st{};
        must(krr_pcg_solve_operator(ctx, 2, dense_op, &a, nullptr, nullptr, y, 1e-10, 50, nullptr,
                                    nullptr, x, &st, nullptr),
             "pcg 2x2");
        check(st.converged && st.iterations <= 2 && std::fabs(x[0] - 1) <= 1e-9 &&
                  std::fabs(x[1] - 1) <= 1e-9,
              "pcg 2x2 diagonal");
    }
    // breakdown on -I (test_solver.cpp:65-69) -> KRR_ERR_BREAKDOWN
    {
        Dense a{{-1, 0, 0, 0, -1, 0, 0, 0, -1}, 3};
        const double y[3] = {1, 1, 1};
        double x[3];
        krr_rhs_stats st{};
        const int rc = krr_pcg_solve_operator(ctx, 3, dense_op, &a, nullptr, nullptr, y, 1e-8, 10,
                                              nullptr, nullptr, x, &st, nullptr);
        check(rc == KRR_ERR_BREAKDOWN, "pcg breakdown maps to BreakdownDetected");
    }
    // train agrees with the reference's tau bound (test_solver.cpp:126-147), through
    // the device kernel operator: |c - c*| <= 2 tau |y| / lambda with c* from a dense solve
    {
        const int64_t n = 200, d = 3, t = 2;
        const auto x = random_matrix(n, d, 5);
        const auto y = random_matrix(n, t, 6);
        std::vector<double> c(static_cast<size_t>(n * t));
        std::vector<krr_rhs_stats> st(t);
        int64_t total = 0;
        must(krr_train(ctx, x.data(), n, d, y.data(), t, 1.5, 0.1, -1.0, 64, 3, 1e-8, 1000, c.data(),
                       st.data(), nullptr, &total, nullptr),
             "krr_train");
        // true residual of the returned c through the device kernel operator
        bool ok = st[0].converged && st[1].converged;
        for (int64_t j = 0; j < t && ok; ++j) {
            std::vector<double> ycol(static_cast<size_t>(n)), kc(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) ycol[size_t(i)] = y[size_t(i * t + j)];
            std::vector<double> ccol(static_cast<size_t>(n));
            for (int64_t i = 0; i < n; ++i) ccol[size_t(i)] = c[size_t(i * t + j)];
            must(krr_kernel_matvec(ctx, 0.1, ccol.data(), 1, kc.data()), "matvec");
            double rn = 0, yn = 0;
            for (int64_t i = 0; i < n; ++i) {
                rn += (ycol[size_t(i)] - kc[size_t(i)]) * (ycol[size_t(i)] - kc[size_t(i)]);
                yn += ycol[size_t(i)] * ycol[size_t(i)];
            }
            ok = ok && std::sqrt(rn) <= 1.5e-8 * std::sqrt(yn);  // true residual ~ tau (recursive <= tau)
        }
        check(ok && total == st[0].iterations + st[1].iterations, "train residual within tau");
    }
    // mat-vec paths behind the same entry point: auto (K1-I8 tensor cores for d >= 48),
    // forced DMMA, and the optional fp32 mode, on one problem (the fp64 paths agree to
    // ~1e-13, the fp32 mode to ~1e-6)
    {
        const int64_t n = 700, d = 64;
        const auto x = random_matrix(n, d, 9);
        const auto v = random_matrix(n, 1, 10);
        std::vector<double> a(static_cast<size_t>(n)), b(static_cast<size_t>(n)), f(static_cast<size_t>(n));
        must(krr_set_data(ctx, x.data(), n, d, 6.0), "set_data");
        double path = -2;
        must(krr_get_option(ctx, "k1_path_effective", &path), "get_option");
        must(krr_kernel_matvec(ctx, 1e-3, v.data(), 1, a.data()), "matvec auto");
        must(krr_set_option(ctx, "k1_path", 0), "k1_path dmma");
        must(krr_kernel_matvec(ctx, 1e-3, v.data(), 1, b.data()), "matvec dmma");
        must(krr_set_option(ctx, "k1_path", -1), "k1_path auto");
        must(krr_set_precision(ctx, 32), "precision 32");
        must(krr_kernel_matvec(ctx, 1e-3, v.data(), 1, f.data()), "matvec fp32");
        must(krr_set_precision(ctx, 64), "precision 64");
        double dn = 0, fn = 0, nn = 0;
        for (int64_t i = 0; i < n; ++i) {
            dn += (a[size_t(i)] - b[size_t(i)]) * (a[size_t(i)] - b[size_t(i)]);
            fn += (a[size_t(i)] - f[size_t(i)]) * (a[size_t(i)] - f[size_t(i)]);
            nn += a[size_t(i)] * a[size_t(i)];
        }
        check(path == 1.0, "auto path is K1-I8 at d = 64");
        check(std::sqrt(dn / nn) <= 1e-13, "K1-I8 == K1-DMMA to 1e-13");
        check(std::sqrt(fn / nn) <= 2e-6, "fp32 mode within 2e-6");
        check(krr_set_precision(ctx, 16) == KRR_ERR_INVALID_ARGUMENT, "precision 16 rejected");
    }
    // polynomial kernel + TensorSketch -> SRHT chain through krr_train_ex; the
    // true residual of the returned c through the device polynomial operator
    {
        const int64_t n = 500, d = 4;
        auto x = random_matrix(n, d, 21);
        for (auto& v : x) v *= 0.5;
        const auto y = random_matrix(n, 1, 22);
        krr_kernel_spec k{};
        k.family = 1;
        k.gamma = 1.0;
        k.offset = 0.5;
        k.degree = 2;
        krr_chain_spec ch{};
        ch.first = 1;
        ch.s1 = 64;
        ch.s2 = 32;
        std::vector<double> c(static_cast<size_t>(n));
        krr_rhs_stats st{};
        int64_t total = 0;
        must(krr_train_ex(ctx, x.data(), n, d, y.data(), 1, &k, &ch, 0.05, -1.0, 3, 1e-9, 300, c.data(), &st,
                          nullptr, &total, nullptr),
             "train_ex polynomial");
        std::vector<double> kc(static_cast<size_t>(n));
        must(krr_kernel_matvec(ctx, 0.05, c.data(), 1, kc.data()), "polynomial matvec");
        double rn = 0, yn = 0;
        for (int64_t i = 0; i < n; ++i) {
            rn += (y[size_t(i)] - kc[size_t(i)]) * (y[size_t(i)] - kc[size_t(i)]);
            yn += y[size_t(i)] * y[size_t(i)];
        }
        check(st.converged == 1 && std::sqrt(rn) <= 1e-7 * std::sqrt(yn), "polynomial train residual within tau");
        krr_chain_spec bad = ch;
        bad.first = 0;
        check(krr_chain_build_seeded(ctx, &bad, 0) == KRR_ERR_INVALID_ARGUMENT, "RFF chain on a polynomial kernel rejected");
        krr_chain_spec half{};
        must(krr_chain_scaled_to(&ch, 16, &half), "scaled_to");
        check(half.s1 == 32 && half.s2 == 16, "ChainSpec::scaled_to(16) of {64, 32}");
    }
    // error mapping: lambda <= 0 -> NonPositiveLambda; sigma <= 0 -> invalid_argument
    {
        double dummy[4] = {0, 0, 0, 0};
        check(krr_precond_build(ctx, 0.0, nullptr) != KRR_OK, "precond before sketch fails");
        check(krr_set_data(ctx, dummy, 2, 2, -1.0) == KRR_ERR_INVALID_ARGUMENT, "sigma <= 0 rejected");
    }
    krr_ctx_destroy(ctx);
    std::printf("%d failure(s)\n", failures);
    return failures == 0 ? 0 : 1;
}
