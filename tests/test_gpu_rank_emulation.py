"""The multi-rank K1 / K1T on one GPU (B200_PROFILING: with fewer GPUs than ranks, emulate the
ranks): rank r of W builds its share of the symmetric super-tile schedule, writes only its
owned part slots and (rank 0 only) the diagonal term; the sum over ranks of the partial
(K + lambda I) V must equal the single-rank result — what the NCCL all-reduce computes on a
multi-GPU box (csrc/krr_capi.cu allreduce_sum)."""
import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n,d,world,t,path", [(1000, 16, 2, 1, 0), (5000, 90, 3, 1, -1), (40000, 90, 8, 1, -1),
                                              (40000, 20, 8, 1, 0), (9000, 54, 4, 16, -1), (3000, 7, 5, 8, 0)])
def test_rank_partials_sum_to_full_matvec(krr, oracle, ctx, n, d, world, t, path):
    x = oracle.random_matrix(n, d, 5)
    v = oracle.random_matrix(n, t, 6)
    kern = krr.KernelSpec.gaussian(4.0)
    ctx.set_option("k1_path", path)
    full = krr.KernelOperator(x, kern, 0.3, ctx=ctx).matmat(v)
    acc = np.zeros_like(full)
    try:
        ctx.set_option("emulate_world", world)
        for r in range(world):
            ctx.set_option("emulate_rank", r)
            part = krr.KernelOperator(x, kern, 0.3, ctx=ctx).matmat(v)
            assert not np.array_equal(part, full)
            acc += part
    finally:
        ctx.set_option("emulate_world", 1)
        ctx.set_option("emulate_rank", 0)
        ctx.set_option("k1_path", -1)
    assert rel(acc, full) <= 1e-14, rel(acc, full)


def test_rank_emulation_rejects_bad_values(krr, ctx):
    with pytest.raises(krr.InvalidArgument):
        ctx.set_option("emulate_world", 0)
    with pytest.raises(krr.InvalidArgument):
        ctx.set_option("emulate_rank", -1)
    with pytest.raises(krr.InvalidArgument):
        ctx.set_option("emulate_rank", 0.5)


@pytest.mark.parametrize("n,d,world", [(5000, 90, 3), (40000, 90, 8)])
def test_rank_partials_fp32_mode(krr, oracle, ctx, n, d, world):
    """The optional fp32 mode (K1-F32) on the multi-rank schedule: bench.py also measures it at
    N > 1, so rank r's partial must follow the same owned-slot / diagonal rules."""
    x = oracle.random_matrix(n, d, 7)
    v = oracle.random_matrix(n, 1, 8)
    kern = krr.KernelSpec.gaussian(6.0)
    ctx.set_precision(32)
    try:
        full = krr.KernelOperator(x, kern, 1e-3, ctx=ctx).matmat(v)
        acc = np.zeros_like(full)
        ctx.set_option("emulate_world", world)
        for r in range(world):
            ctx.set_option("emulate_rank", r)
            acc += krr.KernelOperator(x, kern, 1e-3, ctx=ctx).matmat(v)
    finally:
        ctx.set_option("emulate_world", 1)
        ctx.set_option("emulate_rank", 0)
        ctx.set_precision(64)
    # per-rank partials are fp32-accurate sums; their fp64 sum matches the one-rank result to
    # the fp32 mode's own accuracy
    assert rel(acc, full) <= 1e-6, rel(acc, full)
