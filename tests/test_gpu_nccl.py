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
