"""quality_test and adaptive sketch sizing (precond.cpp:42-138) on the device
vs the oracle restatement."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,sigma,lam,s", [(600, 4, 1.5, 1e-1, 64), (900, 6, 2.0, 1e-2, 200),
                                             (800, 3, 0.8, 1e-2, 32)])
def test_quality_test_matches_oracle(krr, oracle, ctx, n, d, sigma, lam, s):
    x = oracle.random_matrix(n, d, 5)
    w, b = oracle.rff_realize(11, d, s, sigma)
    z = oracle.rff_apply_rows(x, w, b)
    got = krr.quality_test(x, krr.KernelSpec.gaussian(sigma), z, lam, ctx=ctx)
    want = oracle.quality_test(x, sigma, z, lam)
    assert got.rank_of_p == want["rank_of_p"]
    assert got.sketch_size == s and got.spectrum_cut == 0.05 * lam and got.cond1_threshold == 0.1 * lam
    # power iteration stops at tol 1e-4: the same start vector gives the same trajectory
    # up to reduction order, so the estimates agree to well inside the tolerance
    assert abs(got.cond1_value - want["cond1_value"]) <= 2e-4 * abs(want["cond1_value"]) + 1e-14
    assert abs(got.cond2_ratio_low - want["cond2_ratio_low"]) <= 1e-8
    assert abs(got.cond2_ratio_high - want["cond2_ratio_high"]) <= 1e-8
    assert got.passed == want["passed"]


def test_adaptive_build_and_train(krr, oracle, ctx):
    n, d, sigma, lam = 1000, 3, 1.0, 5e-2
    x = oracle.random_matrix(n, d, 9)
    y = oracle.random_matrix(n, 1, 10)
    ref = oracle.adaptive_sizes(x, sigma, lam, 64, n, 4)
    cfg = krr.SolverConfig(tau=1e-8, max_iter=400, lambda_=lam, chain=krr.ChainSpec(s1=64), adaptive=True,
                           s0=64, s_max=n, seed=4)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=ctx)
    assert [h.sketch_size for h in res.quality_history] == [s for s, _ in ref]
    assert [h.passed for h in res.quality_history] == [r["passed"] for _, r in ref]
    assert res.sketch_size == ref[-1][0] and res.quality_passed == ref[-1][1]["passed"]
    assert res.report.per_rhs[0].converged
    # the solution solves the system: residual through the device operator
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)
    r = y[:, 0] - op(res.model.c[:, 0])
    assert np.linalg.norm(r) <= 2e-8 * np.linalg.norm(y)


def test_default_initial_sketch_size(krr):
    assert krr.default_initial_sketch_size(100) == 64
    assert krr.default_initial_sketch_size(64 * 100 + 1) == 101
