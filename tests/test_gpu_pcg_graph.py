"""The graph-resident PCG loop (one CUDA graph: a conditional WHILE node whose body is one
iteration, the stop / breakdown decision made on the device) against the host-driven loop:
same kernels in the same order, so iterates, residual histories and iteration counts are
bitwise identical (solver.cpp:22-67 semantics)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _solve(krr, ctx, x, y, kernel, lam, pre, tau, max_iter, graph):
    ctx.set_option("pcg_graph", 1 if graph else 0)
    try:
        p = None
        if pre:
            chain = krr.ChainSpec(s1=128) if kernel.family == "gaussian" else krr.ChainSpec("TensorSketch", 128)
            cfg = krr.SolverConfig(lambda_=lam, tau=tau, max_iter=max_iter, chain=chain, seed=3)
            return krr.train(krr.Dataset(x, y), kernel, cfg, ctx=ctx)
        c, rep = krr.solve_regularized(x, kernel, y, lam, p, tau, max_iter, ctx=ctx)
        return c, rep
    finally:
        ctx.set_option("pcg_graph", 1)


@pytest.mark.parametrize("d,kern,pre,prec", [(16, "g", False, 64), (54, "g", True, 64), (90, "g", True, 64),
                                            (8, "p", True, 64), (54, "g", True, 32), (20, "g", False, 64)])
def test_graph_loop_bitwise_equals_host_loop(krr, oracle, ctx, d, kern, pre, prec):
    n = 3000
    x = oracle.random_matrix(n, d, 4, 0.5 if kern == "p" else 1.0)
    y = oracle.random_vector(n, 5)
    kernel = krr.KernelSpec.gaussian(3.0) if kern == "g" else krr.KernelSpec.polynomial(1.0, 0.5, 2)
    ctx.set_precision(prec)
    try:
        a = _solve(krr, ctx, x, y, kernel, 1e-2, pre, 1e-10, 60, graph=True)
        b = _solve(krr, ctx, x, y, kernel, 1e-2, pre, 1e-10, 60, graph=False)
    finally:
        ctx.set_precision(64)
    if pre:
        ca, ra = a.model.c, a.report
        cb, rb = b.model.c, b.report
    else:
        (ca, ra), (cb, rb) = a, b
    sa, sb = ra.per_rhs[0], rb.per_rhs[0]
    assert sa.iterations == sb.iterations and sa.converged == sb.converged
    assert np.array_equal(np.asarray(sa.residual_history), np.asarray(sb.residual_history))
    assert sa.final_residual == sb.final_residual
    assert np.array_equal(ca, cb)


def test_graph_loop_converges_and_stops_at_max_iter(krr, oracle, ctx):
    x = oracle.random_matrix(1500, 10, 6)
    y = oracle.random_vector(1500, 7)
    kern = krr.KernelSpec.gaussian(2.0)
    c, rep = _solve(krr, ctx, x, y, kern, 1.0, False, 1e-6, 500, graph=True)
    st = rep.per_rhs[0]
    assert st.converged and st.final_residual <= 1e-6 and len(st.residual_history) == st.iterations
    c2, rep2 = _solve(krr, ctx, x, y, kern, 1e-6, False, 1e-14, 7, graph=True)
    assert rep2.per_rhs[0].iterations == 7 and not rep2.per_rhs[0].converged


def test_graph_loop_breakdown(krr, oracle, ctx):
    """p'Ap <= 0 -> BreakdownDetected from the device-side check (rank 1 of an emulated 2-rank
    schedule carries no diagonal term, so with y = e_0 the first p'Ap is exactly 0)."""
    x = oracle.random_matrix(700, 6, 8)
    y = np.zeros(700)
    y[0] = 1.0
    ctx.set_option("emulate_world", 2)
    ctx.set_option("emulate_rank", 1)
    try:
        for graph in (True, False):
            with pytest.raises(krr.BreakdownDetected):
                _solve(krr, ctx, x, y, krr.KernelSpec.gaussian(2.0), 1e-3, False, 1e-8, 10, graph)
    finally:
        ctx.set_option("emulate_world", 1)
        ctx.set_option("emulate_rank", 0)
