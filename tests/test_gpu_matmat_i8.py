"""K1T-I8 — the T = 16 multi-RHS mat-mat with tcgen05 INT8-slice dot products (K-streamed
operands) and DMMA E.V contractions (csrc/gauss_matmat_i8.cu), vs the CPU oracle and vs the
FP64 DMMA K1T.

Reference: gram_matrix (kernels.cpp:72-88) applied column by column as solve_regularized's
apply_a (solver.cpp:75-77).  Bar: ||dKV|| / ||KV|| <= 1e-13 (the K1 bar); the K entries are
K1-I8's bit patterns (same slices, drain and table exp), checked bitwise.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

CASES = [(1, 1, 1.0, 16), (5, 4, 0.7, 16), (300, 6, 1.7, 16), (1000, 90, 6.0, 11), (2048, 440, 20.0, 16),
         (4097, 440, 20.0, 16), (9000, 96, 8.0, 16), (20000, 440, 20.0, 16), (3000, 54, 3.0, 30)]


@pytest.mark.parametrize("n,d,sigma,t", CASES)
def test_i8_matmat_matches_oracle_and_dmma(krr, oracle, ctx, n, d, sigma, t):
    x = oracle.random_matrix(n, d, 3 + n)
    v = oracle.random_matrix(n, t, 4 + n)
    lam = 1e-3
    ctx.set_option("k1t_path", 1)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)
    assert ctx.get_option("k1t_path_effective") == 1
    got = op.matmat(v)
    ctx.set_option("k1t_path", 0)
    assert ctx.get_option("k1t_path_effective") == 0
    dmma = op.matmat(v)
    for r0, r1 in {(0, min(n, 40)), (max(0, n - 40), n)}:
        want = oracle.kernel_matvec(x, sigma, lam, v, rows=(r0, r1))
        assert rel(got[r0:r1], want) <= 1e-13, (r0, rel(got[r0:r1], want))
    assert rel(got, dmma) <= 1e-13, rel(got, dmma)


def test_i8_matmat_entries_bitwise_k1_i8(krr, oracle, ctx):
    """K V with V = identity columns: every entry is one e_ij (the E.V sums add exact zeros),
    so K1T-I8's Gram matrix is K1-I8's bit for bit, exactly symmetric, with a unit diagonal."""
    n, d = 300, 40
    x = oracle.random_matrix(n, d, 11)
    x[::7] *= 1e-2
    x[4] = x[9]  # duplicate rows: d2 clamped at 0 where rounding makes it negative
    ctx.set_option("k1t_path", 1)
    ctx.set_option("k1_path", 1)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(3.0), 0.0, ctx=ctx)
    kk = op.matmat(np.eye(n))
    cols = list(range(0, n, 23))
    k1 = np.column_stack([op(np.eye(n)[:, j]) for j in cols])
    assert np.array_equal(np.diag(kk), np.ones(n))
    assert np.array_equal(kk, kk.T)
    assert np.array_equal(kk[:, cols], k1)
    want = oracle.gram_matrix(x, 3.0)
    assert np.max(np.abs(kk - want)) <= 4e-15  # entries <= 1; |x|^2 up to ~40 at d = 40


def test_i8_matmat_rank_emulation_partials_sum(krr, oracle, ctx):
    """Per-rank K1T-I8 partials (emulated ranks of a W = 4 job) sum to the single-rank K V."""
    n, d, t = 9000, 90, 16
    x = oracle.random_matrix(n, d, 21)
    v = oracle.random_matrix(n, t, 22)
    ctx.set_option("k1t_path", 1)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 0.0, ctx=ctx)
    full = op.matmat(v)
    acc = np.zeros_like(full)
    for r in range(4):
        ctx.set_option("emulate_world", 4)
        ctx.set_option("emulate_rank", r)
        op_r = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 0.0, ctx=ctx)
        acc += op_r.matmat(v)
    ctx.set_option("emulate_world", 1)
    ctx.set_option("emulate_rank", 0)
    assert rel(acc, full) <= 1e-14, rel(acc, full)


@pytest.mark.parametrize("d,want", [(16, 0), (19, 0), (20, 1), (90, 1), (440, 1), (449, 0)])
def test_k1t_path_auto_selection(krr, oracle, ctx, d, want):
    """Auto K1T path: K1T-I8 from d = 20 (profiles/r2_k1t_i8_crossover.log) up to kp = 448."""
    x = oracle.random_matrix(600, d, 3)
    krr.GaussianOperator(x, krr.KernelSpec.gaussian(4.0), 0.0, ctx=ctx)
    assert ctx.get_option("k1t_path") == -1
    assert ctx.get_option("k1t_path_effective") == want


def test_k1t_i8_not_used_for_polynomial(krr, oracle, ctx):
    """The polynomial kernel's multi-RHS products stay on the DMMA K1T (Gaussian-only kernel)."""
    x = oracle.random_matrix(600, 90, 3)
    ctx.set_option("k1t_path", 1)
    krr.KernelOperator(x, krr.KernelSpec.polynomial(1.0 / 90, 1.0, 3), 0.0, ctx=ctx)
    assert ctx.get_option("k1t_path_effective") == 0


@pytest.mark.parametrize("n,d,sigma", [(700, 200, 12.0), (4097, 160, 10.0), (5000, 440, 20.0)])
def test_single_rhs_large_d_through_k1t_i8(krr, oracle, ctx, n, d, sigma):
    """d >= 160 (K1-I8 does not apply above d = 96): a single K v runs as column 0 of a
    16-column K1T-I8 pass (k1_path_effective = 2); same bar as every K1 path."""
    x = oracle.random_matrix(n, d, 8 + n)
    v = oracle.random_vector(n, 9 + n)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), 1e-3, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == 2
    got = op(v)
    for r0, r1 in {(0, min(n, 40)), (max(0, n - 40), n)}:
        want = oracle.kernel_matvec(x, sigma, 1e-3, v, rows=(r0, r1))
        assert rel(got[r0:r1], want) <= 1e-13, (r0, rel(got[r0:r1], want))
    ctx.set_option("k1_path", 0)
    try:
        assert ctx.get_option("k1_path_effective") == 0
        dmma = op(v)
    finally:
        ctx.set_option("k1_path", -1)
    assert rel(got, dmma) <= 1e-13


def test_train_large_d_graph_loop_matches_oracle(krr, oracle, ctx):
    """The graph-resident PCG loop with the large-d single-column K1T-I8 operator (prepared
    before capture) reproduces the oracle's train.  sigma = 8 at d = 200 keeps the solve well
    conditioned (a few tens of iterations), away from the round-off-sensitive regime where even
    two CPU summation orders disagree on the stopping iteration."""
    n, d, sigma, lam = 1200, 200, 8.0, 0.1
    x = oracle.random_matrix(n, d, 31)
    y = oracle.random_matrix(n, 1, 32)
    cfg = krr.SolverConfig(lambda_=lam, tau=1e-8, max_iter=500, chain=krr.ChainSpec(s1=256), seed=0)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == 2
    ref = oracle.train(x, y, sigma, lam, 256, 0, 1e-8, 500)
    st = res.report.per_rhs[0]
    assert st.converged and abs(st.iterations - ref.iterations[0]) <= 1, (st.iterations, ref.iterations[0])
    assert rel(res.model.c, ref.c) <= 1e-8, rel(res.model.c, ref.c)


@pytest.mark.parametrize("d", [440, 96])
def test_i8_matmat_worst_case_slice_sums(krr, oracle, ctx, d):
    """Inputs whose Ozaki digits are all +-127 (x = +-(1 - 2^-53)): the group sums reach
    8 x 127^2 x kp, which for kp = 448 overflows an int32 combination 128 G_2k + G_2k+1 — the
    drain combines in int64 (gauss_matmat_i8.cu).  Checked against the oracle and the DMMA K1T."""
    n, t = 512, 16
    rng = np.random.default_rng(5)
    x = np.where(rng.random((n, d)) < 0.9, 1.0, -1.0) * (1.0 - 2.0 ** -53)
    x[:, 0] = 1.0 - 2.0 ** -53  # every row's max |x| sets e = 0: all digits 127
    v = oracle.random_matrix(n, t, 8)
    sigma, lam = 30.0, 1e-3
    ctx.set_option("k1t_path", 1)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)
    assert ctx.get_option("k1t_path_effective") == 1
    got = op.matmat(v)
    want = oracle.kernel_matvec(x, sigma, lam, v)
    assert rel(got, want) <= 1e-13, rel(got, want)
    ctx.set_option("k1t_path", 0)
    assert rel(got, op.matmat(v)) <= 1e-13
