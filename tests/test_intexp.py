"""CPU checks of K1-I8X's integer epilogue model (paper_1611_03220_b200/intexp.py) and of the
constants compiled into csrc/gauss_matvec_i8x.cu.  Reference semantics: kernels.cpp:79-86
(d2 = max(0, sq_i + sq_j - 2 p_ij), k = exp(-d2 scale))."""
import math
import random
import re
from fractions import Fraction
from pathlib import Path

import numpy as np
import pytest

from paper_1611_03220_b200 import intexp as ie

SRC = Path(__file__).resolve().parents[1] / "paper_1611_03220_b200" / "csrc" / "gauss_matvec_i8x.cu"


def _cu_int(name):
    m = re.search(rf"\b{name}\s*=\s*(\d+)u?\b", SRC.read_text())
    assert m, name
    return int(m.group(1))


def test_device_constants_match_the_model():
    c = ie.consts(1)
    assert _cu_int("K32H") == c.K32H
    assert _cu_int("C69LO") + (_cu_int("C69HI") << 32) == c.C69
    for nm in ("C3", "C4", "C5", "C6"):
        assert _cu_int(nm) == getattr(c, nm)
    for n in range(1, 6):
        m = re.search(rf"PB{n} = (0x[0-9a-fp.+-]+)", SRC.read_text())
        assert m and float.fromhex(m.group(1)) == ie.PB[n]
        assert ie.PB[n] == float(Fraction(1, math.factorial(n) * 2 ** (53 * n)))  # 2^-53n / n!, rounded


@pytest.mark.parametrize("integer_poly,bound", [(False, 1.0), (True, 2.0)])
@pytest.mark.parametrize("E", [1, 2, 5, 8])
def test_exp_within_ulps_of_exact(E, integer_poly, bound):
    """e = exp(-u 2^-G) within 1 ulp (FP64 polynomial in phase B, the default) or 2 ulp (the
    all-integer variant) of the correctly rounded exp of the exact fixed-point argument."""
    C = ie.consts(E)
    rng = random.Random(E)
    for t in range(1500):
        r = rng.random()
        uval = rng.random() * (1e-3 if r < 0.3 else (12.0 if r < 0.6 else 700.0))
        u = int(uval * 2 ** C.G) + rng.randint(0, 2 ** 20)
        e, _ = ie.exp_neg(u, C, integer_poly=integer_poly)
        ref = ie.reference_exp(u, C)
        assert abs(e - ref) <= bound * math.ulp(ref), (E, uval, e, ref)


def test_exp_edges():
    C = ie.consts(1)
    assert ie.exp_neg(0, C)[0] == 1.0
    # d2 < 0 by the slice truncation (u slightly negative): e = 1 + O(2^-50), never > 1 + 1e-14
    e, _ = ie.exp_neg(-50, C)
    assert 1.0 <= e <= 1.0 + 1e-14
    # u beyond the ~700 clamp: a tiny normal number, not a denormal or garbage
    e, _ = ie.exp_neg(int(900 * 2 ** C.G), C)
    assert 0.0 < e <= math.exp(-699) and e >= 2.0 ** -1022


def test_pair_p_is_floor_of_w():
    rng = random.Random(3)
    for _ in range(2000):
        b = [rng.randint(-(2 ** 27), 2 ** 27), rng.randint(-(2 ** 30), 2 ** 30), rng.randint(-(2 ** 30), 2 ** 30),
             rng.randint(-(2 ** 30), 2 ** 30)]
        w = b[0] * 2 ** 42 + b[1] * 2 ** 28 + b[2] * 2 ** 14 + b[3]
        assert ie.pair_p(tuple(b)) == w >> 8


def test_pipeline_entries_vs_exact_on_standardised_data():
    """Whole pair pipeline (digits -> SQ, W -> u -> e) on config-4-like rows: per-entry relative
    error vs exp(-scale |x_i - x_j|^2) in exact arithmetic, within the oracle's own error band."""
    mp = pytest.importorskip("mpmath")
    mp.mp.prec = 120
    rng = np.random.default_rng(4)
    n, d, sigma = 60, 90, 6.0
    x = rng.standard_normal((n, d))
    scale = 1.0 / (2.0 * sigma * sigma)
    ch = math.sqrt(2.0 * scale)
    cl = ie.fma(-ch, ch, 2.0 * scale) / (2.0 * ch)
    z = np.array([[ie.fma(a, ch, a * cl) for a in row] for row in x])
    zmax = float(np.abs(z).max())
    E = max(1, math.frexp(zmax)[1])
    while zmax >= math.ldexp(127.5 / 128.0, E):
        E += 1
    C = ie.consts(E)
    D = [ie.digits(z[i], E) for i in range(n)]
    SQ = [ie.sq_from_digits(D[i]) for i in range(n)]
    errs = []
    for i in range(0, n, 3):
        for j in range(i + 1, n, 5):
            u = SQ[i] + SQ[j] - (ie.pair_w(D[i], D[j]) >> 8)
            e, _ = ie.exp_neg(u, C)
            d2 = sum((mp.mpf(float(a)) - mp.mpf(float(b))) ** 2 for a, b in zip(x[i], x[j]))
            ex = mp.exp(-d2 * mp.mpf(scale))
            errs.append(float((e - ex) / ex))
    errs = np.array(errs)
    assert np.max(np.abs(errs)) <= 1.5e-15
    assert abs(errs.mean()) <= 3e-16
