"""Bit-level model of K1-I8X's integer Gaussian epilogue (csrc/gauss_matvec_i8x.cu).

K1-I8X evaluates exp(-scale d2_ij) without the FP64 pipe (which the INT8 tensor path
throttles ~4x on B200), so the exp phase of a tile can overlap the next tile's MMAs.  This
module restates that arithmetic step by step with Python integers (two's-complement 32/64-bit
semantics made explicit), so the constants and the error bound can be checked on the CPU
(tests/test_intexp.py) and so the device code has a readable specification.  It is not on any
product path.

Fixed-point pipeline for one pair (i, j), with z = sqrt(2 scale) x (so scale d2 = |z_i - z_j|^2 / 2),
one global exponent E (|z_ik| < 2^E 127.5/128, 1 <= E <= 8) and 8 signed digits per element
(round to nearest: |a_0| <= 127, |a_p| <= 64 after it):
    W_ij = sum_c 2^(49 - 7c) G_c          (G_c from the tensor cores, exact)
    P_ij = floor(W_ij / 2^8)              = z_i.z_j 2^G       (G = 55 - 2E)
    SQ_i = floor(|z~_i|^2 / 2 2^G)        (all digit products: the c <= 7 cut would bias the diagonal)
    u    = SQ_i + SQ_j - P_ij             = scale d2 2^G      (exact integer cancellation)
    k    = round(u 64 / ln2)  (from the high word),  s = k ln2/64 - u   (|s| <= ln2/128, units 2^-69)
    exp(-u) = 2^(-k/64) exp(s),  exp(s) = 1 + Q 2^-53,  Q from s, s^2/2 and s^3 D(s) in integers
    e    = fma(T_j 2^-53, X, T_j / 4) 2^-m,  X = 1.5 2^52 + Q (the bits 0x4338... + Q),  k = 64 m + j
The reference computes d2 = max(0, sq_i + sq_j - 2 p_ij) in fp64 (kernels.cpp:79-84), whose
rounding is ~2^-53 (|x_i|^2 + |x_j|^2) scale; here the cancellation is exact and the exp is
within ~1 ulp.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

LN2 = 0.6931471805599453094172321214581765680755
M64 = (1 << 64) - 1
M32 = (1 << 32) - 1


def s32(x: int) -> int:
    x &= M32
    return x - (1 << 32) if x >> 31 else x


def s64(x: int) -> int:
    x &= M64
    return x - (1 << 64) if x >> 63 else x


def mulhi32(a: int, b: int) -> int:
    """mul.hi.s32: the high 32 bits of the 64-bit signed product."""
    return s32((s32(a) * s32(b)) >> 32)


@dataclass(frozen=True)
class Consts:
    E: int           # global exponent of z (|z_ik| < 2^E)
    G: int           # fraction bits of u (u_fx = u 2^G)
    sh: int          # u 2^G -> u 2^69 shift
    K32H: int        # round(64/ln2 2^24): k = (hi32(-nt K32H) + 2^12) >> 13, nt = -u 2^21
    C69: int         # round(ln2/64 2^69)
    UHMAX: int       # high-word clamp: u <= ~700
    SHT: int         # u 2^G -> ut = u 2^21 (funnel shift right by G - 21)
    C3: int          # 1/6 - 1/8, 1/24, 1/120, 1/720 in units 2^-35
    C4: int
    C5: int
    C6: int
    ABIAS: int = 3 << 20   # rounding of (s^2/2 + s^3 D) 2^75 >> 22 (centres Q with TBIAS)
    RBIAS: int = 1 << 20   # rounding of M_j Q 2^-53
    TBIAS: int = 3         # centres the truncations of the s^3 term (units 2^-55)


def consts(E: int) -> Consts:
    if not 1 <= E <= 8:
        raise ValueError("K1-I8X needs 1 <= E <= 8")
    from fractions import Fraction
    import mpmath as mp
    mp.mp.prec = 200
    G = 55 - 2 * E
    ln2 = mp.log(2)
    K32H = int(mp.nint(64 / ln2 * mp.mpf(2) ** 24))
    C69 = int(mp.nint(ln2 / 64 * mp.mpf(2) ** 69))
    UHMAX = int(mp.floor(700 * mp.mpf(2) ** (G - 32)))
    c = [int(round(Fraction(2 ** 35, 24)))] + [int(round(Fraction(2 ** 35, math.factorial(n)))) for n in (4, 5, 6)]
    assert K32H < 2 ** 31 and C69 < 2 ** 63
    return Consts(E, G, 69 - G, K32H, C69, UHMAX, G - 21, *c)


def table(j: int) -> tuple[float, float]:
    """(T_j 2^-53, T_j / 4) with T_j = 2^(-j/64) correctly rounded."""
    import mpmath as mp
    mp.mp.prec = 200
    t = float(mp.mpf(2) ** (-mp.mpf(j) / 64))
    return math.ldexp(t, -53), math.ldexp(t, -2)


def fma(a: float, b: float, c: float) -> float:
    """fp64 fused multiply-add (CPython's Fraction -> float conversion rounds correctly)."""
    from fractions import Fraction
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def digits(z, E: int) -> list:
    """The 8 digit vectors of fl(c x) = z (numpy float64 array), rounded to nearest, as K1-I8X's prep."""
    import numpy as np
    w = np.ldexp(np.asarray(z, dtype=np.float64), 7 - E)
    out = []
    for _ in range(8):
        t = np.rint(w)
        out.append(t.astype(np.int64))
        w = (w - t) * 128.0
    return out


def pair_w(ai: list, aj: list) -> int:
    """W = sum_{c <= 7} 2^(49 - 7c) G_c: what the tensor cores accumulate for one pair."""
    g = [0] * 8
    for p in range(8):
        for q in range(8 - p):
            g[p + q] += sum(int(x) * int(y) for x, y in zip(ai[p], aj[q]))
    return sum(gc << (49 - 7 * c) for c, gc in enumerate(g))


def pair_p(b: tuple[int, int, int, int]) -> int:
    """P = floor(W / 2^8) from the drained b_k = 128 G_2k + G_2k+1 (device: two mad.wide + a high-word add)."""
    b0, b1, b2, b3 = (s32(x) for x in b)
    L = b2 * 64 + (b3 >> 8)
    L = b1 * (1 << 20) + L
    return s64(L + ((4 * b0) << 32))


def sq_from_digits(a: list) -> int:
    """SQ = floor(|z~|^2 / 2 2^G) from the 8 digit vectors of one row (every product p, q)."""
    g = [0] * 15
    for p in range(8):
        for q in range(8):
            g[p + q] += sum(int(x) * int(y) for x, y in zip(a[p], a[q]))
    return sum(gc << (98 - 7 * c) for c, gc in enumerate(g)) >> 58


def table_mant(j: int) -> int:
    """M_j = round(2^(-j/64) 2^53), in (2^52, 2^53]."""
    import mpmath as mp
    mp.mp.prec = 200
    return int(mp.nint(mp.mpf(2) ** (53 - mp.mpf(j) / 64)))


def table_mant_biased(j: int) -> int:
    """M'_j = round(M_j (1 - 2^-7)): absorbs the +2^46 that keeps Q non-negative."""
    from fractions import Fraction
    return round(Fraction(table_mant(j)) * Fraction(127, 128))


# 2^(-53 n) / n!, the FP64 phase-B polynomial coefficients (gauss_matvec_i8x.cu PB1..PB5)
PB = {n: float.fromhex(h) for n, h in
      {1: "0x1p-53", 2: "0x1p-107", 3: "0x1.5555555555555p-162", 4: "0x1.5555555555555p-217",
       5: "0x1.1111111111111p-272"}.items()}


def exp_neg(u: int, C: Consts, integer_poly: bool = False) -> tuple[float, dict]:
    """e = exp(-u 2^-G) for the int64 u = SQ_i + SQ_j - P_ij, exactly as the device computes it.

    integer_poly=False is the kernel's default (I8X_QA = 0): phase A forms k and round(s 2^53),
    phase B evaluates exp(s) - 1 in FP64; True restates the all-integer variant (I8X_QA = 1).
    """
    nu = s64(-u)                           # the device forms nu = P_ij - SQ_i - SQ_j
    nh, nl = nu >> 32, nu & M32
    nh = max(nh, -C.UHMAX)                 # u <= ~700: e >= 2^-1010 stays normal
    nu = (nh << 32) | nl
    nt = s32(nu >> C.SHT)                  # -u 2^21
    k = ((mulhi32(nt, -C.K32H) + 4096) & M32) >> 13
    s = s64(k * C.C69 + (nu << C.sh))      # s = k ln2/64 - u, units 2^-69
    if not integer_poly:
        sd = float((s + (1 << 15)) >> 16)  # round(s 2^53): phase A packs it (+2^46) with k
        q = fma(sd, PB[5], PB[4])
        for c in (3, 2, 1):
            q = fma(q, sd, PB[c])
        q = q * sd
        ts = math.ldexp(table(k & 63)[1] * 4.0, -(k >> 6))  # 2^-m T_j (exact scaling)
        return fma(ts, q, ts), dict(k=k, s=s, Q=None)
    sh32, sl = s >> 32, s & M32
    A = sh32 * sh32 + C.ABIAS              # s^2 2^74 (mad.wide, + the rounding bias of >> 22)
    cx = mulhi32(sh32, sl >> 1)            # cross term sh32 sl 2^-33
    A = A + 4 * cx                         # s^2 2^74 to ~2^-61 relative
    a2 = s32(A >> 28)                      # s^2 2^46
    s38 = s32(s >> 31)                     # s 2^38
    s3 = mulhi32(a2, s38)                  # s^3 2^52
    sq = sh32 >> 5                         # s 2^32
    t = C.C6
    t = mulhi32(t, sq) + C.C5
    t = mulhi32(t, sq) + C.C4
    D = mulhi32(t, sq) + C.C3              # (D(s) - 1/8) 2^35, D = 1/6 + s/24 + s^2/120 + s^3/720
    tail = s32(mulhi32(s3, D) + s3 + C.TBIAS)   # s^3 D 2^55
    A = A + tail * (1 << 20)               # (s^2/2 + s^3 D) 2^75
    Q = s64((s >> 16) + (A >> 22))         # (exp(s) - 1) 2^53; the device packs k << 47 | (Q + 2^46)
    # phase B (FP64): e = fma(T_j 2^-53, 1.5 2^52 + Q, T_j / 4) 2^-m   (T_j / 4 exact: one rounding)
    j, m = k & 63, k >> 6
    a, bb = table(j)
    X = 6755399441055744.0 + Q             # exact: |Q| < 2^46
    e = math.ldexp(fma(a, X, bb), -m)
    return e, dict(k=k, s=s, Q=Q)


def reference_exp(u: int, C: Consts) -> float:
    import mpmath as mp
    mp.mp.prec = 200
    uu = max(0, s64(u))
    return float(mp.exp(-mp.mpf(uu) / mp.mpf(2) ** C.G))
