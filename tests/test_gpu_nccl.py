"""The NCCL plumbing on one GPU: a one-rank communicator (krr_ctx_create_dist with world = 1)
loads NCCL (dlopen) and builds the communicator (ncclCommCount = 1); the K1 data path is
unchanged by its presence.  (Multi-rank logic: tests/test_dist_gloo.py,
tests/test_gpu_rank_emulation.py.)"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def test_one_rank_nccl_comm_and_matvec(krr, oracle):
    import torch  # noqa: F401  (load torch's NCCL first, as bench.py does, so one NCCL is in the process)

    nid = krr.nccl_unique_id()
    assert len(nid) == 128
    ctx = krr.Context(0, 0, 1, nid)
    plain = krr.Context(0)
    try:
        assert ctx.get_option("nccl_nranks") == 1.0
        assert plain.get_option("nccl_nranks") == 1.0
        x = oracle.random_matrix(3000, 90, 4)
        v = oracle.random_vector(3000, 5)
        a = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 1e-3, ctx=ctx)(v)
        b = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 1e-3, ctx=plain)(v)
        assert np.array_equal(a, b)
    finally:
        ctx.close()
        plain.close()


@pytest.mark.parametrize("t", [1, 5])
def test_nccl_collectives_inside_graph_loop(krr, oracle, t):
    """The multi-rank data path on one GPU: a one-rank communicator with "nccl_always" runs every
    collective of the solve (K v and Woodbury all-reduces, the s x s Gram all-reduce), and for a
    single right-hand side the NCCL kernels are captured inside the graph-resident PCG loop (the
    conditional WHILE body).  An identity all-reduce changes no bit: the solve must equal the
    plain context's bitwise."""
    import torch  # noqa: F401  (one NCCL in the process, as bench.py)

    n, d, sigma, lam, s = 3000, 20, 3.0, 1e-1, 200
    x = oracle.random_matrix(n, d, 21)
    y = oracle.random_matrix(n, t, 22)
    cfg = krr.SolverConfig(lambda_=lam, tau=1e-5, max_iter=300, chain=krr.ChainSpec(s1=s), seed=0)
    ctx = krr.Context(0, 0, 1, krr.nccl_unique_id())
    plain = krr.Context(0)
    try:
        ctx.set_option("nccl_always", 1)
        assert ctx.get_option("pcg_graph") == 1.0
        a = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=ctx)
        b = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=plain)
        assert np.array_equal(a.model.c, b.model.c)
        assert [r.iterations for r in a.report.per_rhs] == [r.iterations for r in b.report.per_rhs]
        assert all(r.iterations > 3 for r in a.report.per_rhs)
    finally:
        ctx.close()
        plain.close()
