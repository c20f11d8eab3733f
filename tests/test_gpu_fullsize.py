"""Parity at BASELINE config 4's full size (n = 1,048,576, d = 90) through
size-independent properties — the dense oracle cannot run at this n:

  * sampled rows of (K + lambda I) v against the oracle's on-the-fly rows (first, middle and
    last rows, including the padded tail's neighbours);
  * the two independent fp64 K1 kernels (tcgen05 INT8 slices, FP64 DMMA) agree on the whole
    vector;
  * symmetry u'(K v) = v'(K u);
  * after a few PCG iterations of the full train (RFF s = 8192, Woodbury, device PCG), the
    recursive residual equals the explicitly recomputed y - (K + lambda I) x.

Each test is one or two minutes of B200 time at most.
"""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu

N, D, _T, SIGMA, LAM, S = 1048576, 90, 1, 6.0, 1e-6, 8192


@pytest.fixture(scope="module")
def c4(krr):
    x, y = krr.generate_config(4, N, D, 1, 0)
    return x, y[:, 0].copy()


def test_fullsize_matvec_rows_paths_symmetry(krr, oracle, ctx, c4):
    x, _ = c4
    rng = np.random.default_rng(7)
    v = rng.normal(size=N)
    u = rng.normal(size=N)
    op = krr.KernelOperator(x, krr.KernelSpec.gaussian(SIGMA), LAM, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == 1  # K1-I8 (auto, d = 90)
    kv = op(v)
    ku = op(u)
    for r0 in (0, N // 2 - 3, N - 8):
        want = oracle.kernel_matvec(x, SIGMA, LAM, v, rows=(r0, r0 + 8))
        got = kv[r0:r0 + 8]
        assert rel(got, want) <= 1e-13, (r0, rel(got, want))
    # symmetry of K (and of the fixed-order reductions): u'Kv == v'Ku
    a, b = float(u @ kv), float(v @ ku)
    assert abs(a - b) <= 1e-12 * (np.abs(u) @ np.abs(kv))
    # the DMMA K1 on the same data
    ctx.set_option("k1_path", 0)
    try:
        kv_dmma = op(v)
    finally:
        ctx.set_option("k1_path", -1)
    assert rel(kv_dmma, kv) <= 1e-13, rel(kv_dmma, kv)


def test_fullsize_pcg_recursive_vs_true_residual(krr, ctx, c4):
    x, y = c4
    cfg = krr.SolverConfig(lambda_=LAM, tau=1e-6, max_iter=3, chain=krr.ChainSpec(s1=S), seed=0)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(SIGMA), cfg, ctx=ctx)
    st = res.report.per_rhs[0]
    assert st.iterations == 3 and not st.converged
    assert all(np.isfinite(st.residual_history)) and st.residual_history[-1] < st.residual_history[0] * 10
    c = res.model.c[:, 0]
    op = krr.KernelOperator(x, krr.KernelSpec.gaussian(SIGMA), LAM, ctx=ctx)
    true_rel = float(np.linalg.norm(y - op(c)) / np.linalg.norm(y))
    assert abs(true_rel - st.final_residual) <= 1e-6 * st.final_residual + 1e-12, (true_rel, st.final_residual)


def test_config5_multi_rhs_rows_and_symmetry(krr, oracle, ctx):
    """BASELINE config 5 (n = 524288, d = 440, t = 16): the multi-RHS K1T over all 16 columns,
    sampled rows against the oracle, and U'(K V) symmetric in (U, V) column by column."""
    n, d, t, sigma, lam, _ = krr.CONFIGS[5]
    x, _y = krr.generate_config(5, n, d, t, 0)
    rng = np.random.default_rng(3)
    v = rng.normal(size=(n, t))
    u = rng.normal(size=(n, t))
    op = krr.KernelOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)
    kv = op.matmat(v)
    ku = op.matmat(u)
    for r0 in (0, n - 4):
        want = oracle.kernel_matvec(x, sigma, lam, v, rows=(r0, r0 + 4))
        assert rel(kv[r0:r0 + 4], want) <= 1e-13, rel(kv[r0:r0 + 4], want)
    a = np.einsum("ij,ij->j", u, kv)
    b = np.einsum("ij,ij->j", v, ku)
    assert np.all(np.abs(a - b) <= 1e-12 * np.einsum("ij,ij->j", np.abs(u), np.abs(kv)))
