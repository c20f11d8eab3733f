"""Parity at the BASELINE configs against oracle fixtures (tests/golden/make_config_fixtures.py:
the reference algorithm restated in oracle/, Eigen-like summation order, run on the same
generators).  Reference: solver.cpp:22-67 (PCG iterates), precond.cpp:20-40 (U = L^-1 Z^T),
sketches.cpp:37-41 (Z), kernels.cpp:72-88 with solver.cpp:75-77 ((K + lambda I) v rows).

C2 (n = 65536) and C3 (n = 262144): the device train stopped after k = 1..K iterations
matches the oracle's iterate x_k at the sampled rows and its residual history; U's first and
last 64 rows at the sampled columns match (the last rows depend on the whole Z^T Z, Cholesky
factor and TRSM).  C4 (n = 1M) and C5 (n = 524288, d = 440, s = 16384): U's leading 64-row
block (a function of Z's first 64 columns over all n rows), Z rows and (K + lambda I) Y rows.

Bars: 1e-9 relative on iterates / residual histories (the north star's alpha bar is 1e-8; the
two-order oracle floor at these sizes over this few iterations is ~1e-13, profiles/README.md),
1e-10 on U blocks, 1e-13 on (K + lambda I) Y rows, 1e-14 absolute on Z."""
from pathlib import Path

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"


def _fixture(cfg):
    p = GOLD / f"config{cfg}_fixture.npz"
    if not p.exists():
        pytest.fail(f"missing {p.name}: run tests/golden/make_config_fixtures.py {cfg}")
    return dict(np.load(p))


def _train(krr, ctx, cfg, max_iter):
    n, d, t, sigma, lam, s = krr.CONFIGS[cfg]
    x, y = krr.generate_config(cfg, n, d, t, 0)
    sc = krr.SolverConfig(tau=1e-6, max_iter=max_iter, lambda_=lam, chain=krr.ChainSpec(s1=s), seed=0)
    return x, y, krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), sc, ctx=ctx)


@pytest.mark.parametrize("cfg", [2, 3])
def test_config_pcg_iterates_match_oracle(krr, ctx, cfg):
    fx = _fixture(cfg)
    rows, its = fx["rows"], int(fx["iters"])
    s = int(fx["s"])
    for k in range(1, its + 1):
        x, y, res = _train(krr, ctx, cfg, k)
        st = res.report.per_rhs[0]
        assert st.iterations == k and not st.converged
        hist = np.asarray(st.residual_history)
        assert rel(hist, fx["residual_history"][:k]) <= 1e-9, (k, hist, fx["residual_history"][:k])
        got = res.model.c[rows, 0]
        assert rel(got, fx["x_rows"][k - 1]) <= 1e-9, (k, rel(got, fx["x_rows"][k - 1]))
    ctx_u_first = ctx.read_u(0, 64, rows)
    ctx_u_last = ctx.read_u(s - 64, 64, rows)
    assert rel(ctx_u_first, fx["u_first"]) <= 1e-10, rel(ctx_u_first, fx["u_first"])
    assert rel(ctx_u_last, fx["u_last"]) <= 1e-10, rel(ctx_u_last, fx["u_last"])
    assert rel(res.model.c[rows, 0], fx["alpha_rows"]) <= 1e-9


@pytest.mark.parametrize("cfg", [4, 5])
def test_config_build_block_matches_oracle(krr, cfg):
    fx = _fixture(cfg)
    rows = fx["rows"]
    n, d, t, sigma, lam, s = krr.CONFIGS[cfg]
    ctx = krr.Context(0)
    try:
        x, y, res = _train(krr, ctx, cfg, 1)
        u0 = ctx.read_u(0, 64, rows)
        assert rel(u0, fx["u_first"]) <= 1e-10, rel(u0, fx["u_first"])
        ctx.precond_drop()
        chain = krr.realize_chain(krr.ChainSpec(s1=s), krr.KernelSpec.gaussian(sigma), d, 0)
        z = chain.rff.apply_rows(x[rows], ctx=ctx)
        assert np.max(np.abs(z[:, :64] - fx["z_rows"])) <= 1e-14
        ky = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx).matmat(y)
        want = fx["ky_rows"]
        assert rel(ky[rows[:want.shape[0]]], want) <= 1e-13
    finally:
        ctx.close()


@pytest.mark.parametrize("lam", [3e-2, 1e-2])
def test_config1_shape_converging_full_solve(krr, oracle, lam):
    """The north-star bar on a BASELINE-shaped solve that converges: config 1's generator and
    sketch (n = 8192, d = 16, sigma = 4, s = 1024 RFF, tau = 1e-6) with lambda raised from 1e-3
    (where the reference algorithm stalls at max_iter) to 3e-2 / 1e-2 (~200 / ~430 iterations).
    Iterations within +-1 of the oracle's three summation orders; alpha within 1e-8 of the
    Eigen-like order when the counts match (else within the order-to-order spread)."""
    n, d, t, sigma, _, s = krr.CONFIGS[1]
    x, y = krr.generate_config(1, n, d, t, 0)
    fam = [oracle.train(x, y, sigma, lam, s, 0, 1e-6, 500, order=k) for k in (2, 0, 1)]
    cfg = krr.SolverConfig(lambda_=lam, tau=1e-6, max_iter=500, chain=krr.ChainSpec(s1=s), seed=0)
    res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg)
    st = res.report.per_rhs[0]
    its = [f.iterations[0] for f in fam]
    assert st.converged and all(f.converged[0] for f in fam)
    assert min(its) - 1 <= st.iterations <= max(its) + 1, (st.iterations, its)
    spread = max(rel(f.c, fam[0].c) for f in fam[1:])
    bar = 1e-8 if st.iterations == its[0] else max(1e-8, 4 * spread, 10 * 1e-6)
    assert rel(res.model.c, fam[0].c) <= bar, (rel(res.model.c, fam[0].c), st.iterations, its, spread)
