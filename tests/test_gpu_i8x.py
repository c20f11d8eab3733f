"""K1-I8X — K1-I8's tensor-core dot products with the integer exp argument
(csrc/gauss_matvec_i8x.cu, opt-in k1_path = 3) vs the CPU oracle.

Reference: gram_matrix (kernels.cpp:72-88) + apply_a (solver.cpp:75-77).  The bit-level model of
the epilogue is paper_1611_03220_b200/intexp.py (checked on the CPU in tests/test_intexp.py).
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

CASES = [(1, 1, 1.0), (2, 3, 1.0), (5, 4, 0.7), (127, 3, 1.5), (129, 33, 2.0), (300, 4, 1.7), (1000, 90, 6.0),
         (4097, 16, 4.0), (5000, 54, 3.0), (9000, 96, 8.0), (40000, 90, 6.0)]


def _op(krr, ctx, x, sigma, lam=1e-3):
    ctx.set_option("k1_path", 3)
    return krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)


@pytest.mark.parametrize("n,d,sigma", CASES)
def test_i8x_matvec_matches_oracle_and_dmma(krr, oracle, ctx, n, d, sigma):
    x = oracle.random_matrix(n, d, 5 + n)
    v = oracle.random_vector(n, 7 + n)
    op = _op(krr, ctx, x, sigma)
    assert ctx.get_option("k1_path_effective") == 3
    assert 1 <= ctx.get_option("i8x_exponent") <= 8
    got = op(v)
    assert np.array_equal(op(v), got)  # deterministic run to run
    ctx.set_option("k1_path", 0)
    dmma = op(v)
    want = oracle.kernel_matvec(x, sigma, 1e-3, v)
    assert rel(got, want) <= 1e-13, rel(got, want)
    assert rel(got, dmma) <= 1e-13, rel(got, dmma)


def test_i8x_entries_symmetry_and_duplicates(krr, oracle, ctx):
    """Exact symmetry and unit diagonal, every entry within 1e-15 + 2^(2-G) e of exp(-scale
    |x_i - x_j|^2) evaluated directly in extended precision (u's fixed-point resolution is 2^-G,
    G = 55 - 2E: one global exponent E, here raised to 4 by the rows scaled by 4), with rows of
    very different scale and a duplicated row (d2 = 0).  The oracle's own entries carry the fp64
    cancellation error of sq_i + sq_j - 2 p_ij (kernels.cpp:84), ~2^-52 scale (sq_i + sq_j); K1-I8X
    cancels exactly in fixed point, so it is compared with the oracle within that budget."""
    n, d, sigma = 300, 6, 2.0
    x = oracle.random_matrix(n, d, 2)
    x[::7] *= 1e-3
    x[1::11] *= 4.0
    x[5] = x[6]
    op = _op(krr, ctx, x, sigma, 0.0)
    cols = list(range(0, n, 37)) + [5, 6]
    kk1 = np.column_stack([op(np.eye(n)[:, j]) for j in cols])
    xl = x.astype(np.longdouble)
    scale = 1.0 / (2.0 * sigma * sigma)
    exact = np.exp(-np.longdouble(scale) * ((xl[:, None, :] - xl[None, cols, :]) ** 2).sum(-1)).astype(np.float64)
    G = 55 - 2 * int(ctx.get_option("i8x_exponent"))
    assert np.all(np.abs(kk1 - exact) <= 1e-15 + 2.0 ** (2 - G) * exact)
    for c, j in enumerate(cols):
        assert kk1[j, c] == 1.0
    assert abs(kk1[6, cols.index(5)] - 1.0) <= 2e-15 and kk1[6, cols.index(5)] == kk1[5, cols.index(6)]
    want = oracle.gram_matrix(x, sigma)[:, cols]
    sq = (x * x).sum(1)
    budget = 2e-15 + (2.0 ** -51 * scale * (sq[:, None] + sq[None, cols]) + 2.0 ** (2 - G)) * want
    assert np.all(np.abs(kk1 - want) <= budget)


def test_i8x_wide_dynamic_range(krr, oracle, ctx):
    """Far-apart clusters: entries from ~1 down to below 1e-300 (u up to the ~700 clamp), all
    within the oracle's tolerance in K v."""
    n, d = 2000, 8
    x = oracle.random_matrix(n, d, 11)
    x[: n // 2] += 6.0
    v = oracle.random_vector(n, 12)
    for sigma in (0.35, 1.0, 3.0):
        op = _op(krr, ctx, x, sigma)
        assert ctx.get_option("k1_path_effective") == 3
        want = oracle.kernel_matvec(x, sigma, 1e-3, v)
        assert rel(op(v), want) <= 1e-13


def test_i8x_out_of_range_data_uses_another_kernel(krr, oracle, ctx):
    """|z| = |x| sqrt(2 scale) >= 2^8 is outside K1-I8X's fixed-point range: E = 0, the request
    falls back to the DMMA kernel (a GPU kernel, parity-tested), results unchanged."""
    n, d = 500, 12
    x = oracle.random_matrix(n, d, 4) * 1000.0
    v = oracle.random_vector(n, 5)
    op = _op(krr, ctx, x, 1.0)
    assert ctx.get_option("i8x_exponent") == 0
    assert ctx.get_option("k1_path_effective") != 3
    assert rel(op(v), oracle.kernel_matvec(x, 1.0, 1e-3, v)) <= 1e-13


def test_i8x_option_after_set_data(krr, oracle, ctx):
    """Requesting k1_path = 3 after the data is set prepares the operands then (outside capture)."""
    n, d = 700, 40
    x = oracle.random_matrix(n, d, 8)
    v = oracle.random_vector(n, 9)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(5.0), 1e-3, ctx=ctx)
    assert ctx.get_option("i8x_exponent") == 0  # opt-in: not prepared by default
    ctx.set_option("k1_path", 3)
    assert ctx.get_option("k1_path_effective") == 3
    assert rel(op(v), oracle.kernel_matvec(x, 5.0, 1e-3, v)) <= 1e-13


def test_i8x_train_matches_oracle(krr, oracle, ctx):
    """A full device PCG solve on K1-I8X: same iteration count and alpha as the oracle."""
    n, d, sigma, lam = 1000, 16, 4.0, 0.1
    x = oracle.random_matrix(n, d, 1)
    y = oracle.random_matrix(n, 1, 3)
    ctx.set_option("k1_path", 3)
    cfg = krr.SolverConfig(lambda_=lam, tau=1e-8, max_iter=500, chain=krr.ChainSpec(s1=256), seed=0)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == 3
    ref = oracle.train(x, y, sigma, lam, 256, 0, 1e-8, 500)
    st = res.report.per_rhs[0]
    assert st.converged and abs(st.iterations - ref.iterations[0]) <= 1
    assert rel(res.model.c, ref.c) <= 1e-8
