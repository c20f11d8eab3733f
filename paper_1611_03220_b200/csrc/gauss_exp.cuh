// The fp64 Gaussian epilogue  e = exp(-max(0, d2) * scale)  (reference kernels.cpp:83-84).
//
// Two implementations:
//   mode 0 — libdevice exp():  the textbook form, ~23 FP64-pipe instructions.
//   mode 1 — table exp (default in the mat-vec): 10 FP64-pipe instructions.
//     k = round(y), y = d2 * (-scale * 64 / ln2), via the 1.5*2^52 shifter (1 DFMA + 1 DADD);
//     f = y - k exactly (1 DFMA), |f| <= 1/2, r = f ln2/64, |r| <= 0.0054;
//     q = expm1(r) by a degree-5 polynomial in f (4 DFMA + 1 DMUL; truncation
//     error <= 3.4e-17 relative);  e = T[k mod 64] * 2^(k div 64) * (1 + q)
//     = fma(T', q, T') (1 DFMA), where T' is the table entry 2^(j/64) with its
//     exponent field bumped by an integer add (INT pipe, no FP64 work).
//     Clamping d2 >= 0 and the underflow cut (e < 2^-1020 -> 0; the reference
//     would return a denormal or zero there, |difference| < 1e-307) are integer
//     compares on the high word of d2, also off the FP64 pipe.
//   Accuracy: <= ~1.5 ulp against a correctly rounded exp of the same rounded
//   argument (checked by tests/test_gpu_kernels.py against glibc).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace krr {

struct ExpConsts {
    double kscale;    // -scale * 64 / ln2
    double neg_scale; // -scale (mode 0)
    double a1, a2, a3, a4, a5;  // (ln2/64)^m / m!
    int hi_under;     // d2 high word above this -> result 0
    int degree;       // mode 2 (polynomial kernel): the exponent q
};

// Host-side construction (long double for the constants).
ExpConsts make_exp_consts(double scale);
// Mode 2 (polynomial kernel): only `degree` is used.
ExpConsts make_poly_consts(int degree);
// Host-side table 2^(j/64), j = 0..63, correctly rounded to double.
void make_exp_table(double* tab64);

__device__ __forceinline__ double gauss_exp_libdevice(double d2, const ExpConsts& c) {
    return exp(fmax(0.0, d2) * c.neg_scale);
}

__device__ __forceinline__ double gauss_exp_table(double d2, const ExpConsts& c,
                                                  const double* __restrict__ tab) {
    const int hi = __double2hiint(d2);
    d2 = hi < 0 ? 0.0 : d2;  // max(0, d2) without the FP64 pipe
    const double shifter = 6755399441055744.0;  // 1.5 * 2^52
    const double t = fma(d2, c.kscale, shifter);
    const double kd = t - shifter;
    const double f = fma(d2, c.kscale, -kd);
    double q = fma(f, c.a5, c.a4);
    q = fma(q, f, c.a3);
    q = fma(q, f, c.a2);
    q = fma(q, f, c.a1);
    q = q * f;
    const int k = __double2loint(t);
    const double tj = tab[k & 63];
    const int e = k >> 6;  // floor division (arithmetic shift)
    const double ts = __hiloint2double(__double2hiint(tj) + e * (1 << 20), __double2loint(tj));
    const double r = fma(ts, q, ts);
    return hi > c.hi_under ? 0.0 : r;
}

// Polynomial kernel entry ipow(p, q) (kernels.cpp:10-14: r = p, then q-1 times r *= p),
// p = gamma x_i.x_j + c arriving from the same tensor-core contraction as d2 (the operands
// are the augmented inputs [sqrt(gamma) x, sqrt(c)], kernels.cpp:56-62).
__device__ __forceinline__ double poly_ipow(double p, const ExpConsts& c) {
    double r = p;
    for (int i = 1; i < c.degree; ++i) r = __dmul_rn(r, p);
    return r;
}

// The same product chain with the degree known at compile time: straight-line code the
// scheduler interleaves across a tile's accumulators (a runtime-trip-count loop per element
// serialises the dependent DMULs and measured 1.5x slower than the Gaussian epilogue).
template <int Q>
__device__ __forceinline__ double poly_ipow_fixed(double p) {
    double r = p;
#pragma unroll
    for (int i = 1; i < Q; ++i) r = __dmul_rn(r, p);
    return r;
}

// K1 epilogue modes: 0/1 Gaussian (libdevice / table exp); 2 polynomial, runtime degree;
// 10 + q polynomial of compile-time degree q (q = 1..4).
constexpr int kPolyModeBase = 10;
constexpr int kPolyMaxFixed = 4;
inline int poly_mode(int degree) { return degree <= kPolyMaxFixed ? kPolyModeBase + degree : 2; }

template <int MODE>
__device__ __forceinline__ double gauss_exp(double d2, const ExpConsts& c,
                                            const double* __restrict__ tab) {
    if constexpr (MODE == 0) {
        return gauss_exp_libdevice(d2, c);
    } else if constexpr (MODE == 1) {
        return gauss_exp_table(d2, c, tab);
    } else if constexpr (MODE >= kPolyModeBase) {
        return poly_ipow_fixed<MODE - kPolyModeBase>(d2);
    } else {
        return poly_ipow(d2, c);
    }
}

}  // namespace krr
