"""K1 — fused symmetric Gaussian mat-vec on the B200 vs the CPU oracle.

Reference: gram_matrix (kernels.cpp:72-88) + apply_a (solver.cpp:75-77).
Tolerances: the device computes d2 with a DMMA contraction and a table exp (<= ~2 ulp);
per-entry relative differences are O(1e-15), so ||dKv|| / ||Kv|| <= 1e-13 is required.
"""
import math

import numpy as np
import pytest

from conftest import rel

pytestmark = pytest.mark.gpu


def _ulps(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    sp = np.spacing(np.maximum(np.abs(a), np.abs(b)))
    return np.abs(a - b) / np.where(sp > 0, sp, 1e-320)


@pytest.mark.parametrize("mode", [0, 1])
def test_gauss_exp_accuracy(krr, ctx, mode):
    """Device epilogue exp(-max(0, d2) scale) vs glibc exp on the same rounded argument."""
    from paper_1611_03220_b200 import _diag, _lib
    rng = np.random.default_rng(0)
    for scale in (1.0 / 32.0, 1.0 / 18.0, 1.0 / 72.0, 1.0 / 800.0, 0.5):
        d2 = np.concatenate([
            rng.uniform(0, 50, 20000), rng.uniform(0, 800 / scale * 1e-3, 20000),
            rng.exponential(1.0 / scale, 20000), np.array([0.0, -1e-14, -3.0, 1e-300, 5e-324]),
            np.linspace(0, 745.0 / scale, 5000)])
        out = np.empty_like(d2)
        _diag.check(_diag.LIB.krr_diag_gauss_exp(0, _lib.ptr(d2), d2.size, scale, mode, _lib.ptr(out)))
        y = -np.maximum(0.0, d2) * scale
        ref = np.exp(y)
        normal = ref >= 2.0 ** -1020
        u = _ulps(out[normal], ref[normal])
        if mode == 0:
            # same argument rounding as the reference (kernels.cpp:84) -> libm-grade exp
            assert u.max() <= 2.0, (scale, mode, u.max())
        else:
            # the table exp rounds y' = d2 * (-scale * 64 / ln2) instead of d2 * (-scale):
            # exp's own conditioning adds |y| * 2^-53 relative on top of <= 2 ulp.
            err = np.abs(out[normal] - ref[normal]) / ref[normal]
            bound = 2.0 ** -52 * (2.0 + 2.0 * np.abs(y[normal]))
            assert np.all(err <= bound), (scale, float(np.max(err / bound)))
            small = normal & (np.abs(y) <= 1.0)
            assert _ulps(out[small], ref[small]).max() <= 3.0
        # below 2^-1020 the table exp flushes to zero (|diff| < 1e-307)
        assert np.all(np.abs(out[~normal] - ref[~normal]) < 1e-306)
        assert out[d2 <= 0].tolist() == [1.0] * int((d2 <= 0).sum())


CASES = [
    # n, d, sigma
    (1, 1, 1.0), (2, 3, 1.0), (5, 4, 0.7), (127, 3, 1.5), (128, 16, 4.0), (129, 5, 2.0),
    (300, 4, 1.7), (513, 54, 3.0), (1000, 90, 6.0), (2048, 440, 20.0), (4097, 16, 4.0),
]


@pytest.mark.parametrize("n,d,sigma", CASES)
def test_matvec_matches_dense_oracle(krr, oracle, ctx, n, d, sigma):
    x = oracle.random_matrix(n, d, 5 + n)
    v = oracle.random_vector(n, 7 + n)
    lam = 1e-3
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=ctx)
    got = op(v)
    if n <= 4097:
        k = oracle.gram_matrix(x, sigma)
        want = k @ v + lam * v
    else:
        want = oracle.kernel_matvec(x, sigma, lam, v)
    assert rel(got, want) <= 1e-13, rel(got, want)


def test_matvec_multi_column(krr, oracle, ctx):
    n, d, sigma = 700, 7, 2.5
    x = oracle.random_matrix(n, d, 1)
    v = oracle.random_matrix(n, 3, 2)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), 0.25, ctx=ctx)
    got = op.matmat(v)
    want = oracle.kernel_matvec(x, sigma, 0.25, v)
    assert rel(got, want) <= 1e-13


def test_exact_symmetry_and_unit_diagonal(krr, oracle, ctx):
    """kernels.cpp:81-86: K_ii = 1 and K_ij == K_ji bitwise (one evaluation per pair)."""
    n, d = 300, 4
    x = oracle.random_matrix(n, d, 2)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(1.7), 0.0, ctx=ctx)
    kk = op.matmat(np.eye(n))  # column j = K e_j
    assert np.array_equal(np.diag(kk), np.ones(n))
    assert np.array_equal(kk, kk.T)
    want = oracle.gram_matrix(x, 1.7)
    assert np.max(np.abs(kk - want)) <= 1e-15  # entries <= 1: a few ulp


def test_duplicate_points_clamp(krr, oracle, ctx):
    """max(0, d2) clamp (kernels.cpp:83): duplicated rows give K_ij = 1 exactly."""
    x = oracle.random_matrix(64, 3, 9)
    x = np.vstack([x, x])
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(1.0), 0.0, ctx=ctx)
    kk = op.matmat(np.eye(128))
    assert np.all(np.abs(kk[np.arange(64), np.arange(64) + 64] - 1.0) <= 1e-14)
    want = oracle.gram_matrix(x, 1.0)
    assert np.max(np.abs(kk - want)) <= 1e-14


def test_far_points_underflow(krr, ctx):
    """Pairs whose kernel underflows contribute exactly zero; no NaN/inf."""
    x = np.array([[0.0], [1e3], [2e3], [1e150]])
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(1.0), 0.5, ctx=ctx)
    out = op(np.ones(4))
    assert np.array_equal(out, np.full(4, 1.5))


def test_device_matvec_entry_and_launch_count(krr, oracle, ctx):
    from paper_1611_03220_b200 import _lib
    import ctypes as C
    n, d = 1000, 10
    x = oracle.random_matrix(n, d, 3)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(3.0), 0.1, ctx=ctx)
    before = ctx.launches
    tot, k1 = C.c_double(), C.c_double()
    _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 0.1, 3, C.byref(tot), C.byref(k1)))
    assert ctx.launches - before == 3 * 2  # K1 + finish per mat-vec
    assert tot.value > 0 and 0 < k1.value <= tot.value


@pytest.mark.parametrize("n,d", [(1000, 16), (3000, 90), (700, 54), (5000, 20), (40000, 90), (33000, 5)])
def test_resident_and_streaming_variants_bitwise_equal(krr, oracle, ctx, n, d):
    """The DMMA K1 pipeline shapes do the same arithmetic in the same order."""
    x = oracle.random_matrix(n, d, 31)
    v = oracle.random_vector(n, 32)
    ctx.set_option("k1_path", 0)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(5.0), 1e-4, ctx=ctx)
    a = op(v)
    ctx.set_option("k1_grouped", 0)
    a2 = op(v)
    ctx.set_option("k1_grouped", 1)
    assert np.array_equal(a, a2)  # phase-offset warp groups: same arithmetic, same order
    ctx.set_option("k1_resident", 0)
    b = op(v)
    ctx.set_option("exp_mode", 0)
    c = op(v)
    ctx.set_option("k1_resident", 1)
    ctx.set_option("exp_mode", 1)
    ctx.set_option("k1_warps", 16)
    d16 = op(v)
    ctx.set_option("k1_resident", 0)
    e16 = op(v)
    ctx.set_option("k1_resident", 1)
    ctx.set_option("k1_warps", 8)
    assert np.array_equal(a, b)
    assert np.array_equal(d16, e16)
    assert rel(c, a) <= 1e-14
    assert rel(d16, a) <= 1e-14  # 16-warp layout reduces column sums over 4 warps, not 2
    assert np.array_equal(op(v), a)  # deterministic run to run
    want = oracle.kernel_matvec(x, 5.0, 1e-4, v)
    assert rel(d16, want) <= 1e-13


def test_set_option_rejects_unknown(krr, ctx):
    with pytest.raises(ValueError):
        ctx.set_option("no_such_knob", 1)
    with pytest.raises(ValueError):
        ctx.get_option("no_such_knob")
    with pytest.raises(ValueError):
        ctx.set_option("k1_path", 2)


@pytest.mark.parametrize("d,want", [(16, 0), (24, 0), (26, 0), (27, 1), (31, 1), (33, 1), (36, 1), (40, 1), (90, 1),
                                    (96, 1), (97, 0)])
def test_k1_path_auto_selection(krr, oracle, ctx, d, want):
    """Auto path: INT8-slice tensor-core K1 where the measured cost model says it is faster
    (27 <= d <= 96), FP64 DMMA otherwise; both match the oracle."""
    n = 600
    x = oracle.random_matrix(n, d, 7)
    v = oracle.random_vector(n, 8)
    assert ctx.get_option("k1_path") == -1
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 1e-3, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == want
    assert ctx.get_option("i8_supported") == (1 if d <= 96 else 0)
    assert rel(op(v), oracle.kernel_matvec(x, 6.0, 1e-3, v)) <= 1e-13


def test_i8_exponent_range_guard(krr, oracle, ctx):
    """Rows whose magnitudes would push the fused I8 scale factor out of the normal range
    (or the exp argument past the 1.5*2^52 rounding shifter) switch the auto path to the
    DMMA kernel at set_data; results stay exact either way."""
    n, d = 400, 64
    x = oracle.random_matrix(n, d, 3)
    x[7] *= 1e150
    v = oracle.random_vector(n, 4)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(2.0), 1e-3, ctx=ctx)
    assert ctx.get_option("i8_supported") == 0
    assert ctx.get_option("k1_path_effective") == 0
    assert rel(op(v), oracle.kernel_matvec(x, 2.0, 1e-3, v)) <= 1e-13
    x[7] /= 1e150
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(2.0), 1e-3, ctx=ctx)
    assert ctx.get_option("k1_path_effective") == 1


I8_CASES = [(1, 1, 1.0), (5, 4, 0.7), (127, 3, 1.5), (300, 4, 1.7), (1000, 90, 6.0), (4097, 16, 4.0),
            (5000, 54, 3.0), (40000, 90, 6.0), (9000, 96, 8.0)]


@pytest.mark.parametrize("n,d,sigma", I8_CASES)
def test_i8_slice_matvec_matches_oracle(krr, oracle, ctx, n, d, sigma):
    """K1-I8 (tcgen05 kind::i8 Ozaki slices): same bar as the FP64 DMMA kernel."""
    x = oracle.random_matrix(n, d, 5 + n)
    v = oracle.random_vector(n, 7 + n)
    ctx.set_option("k1_path", 1)
    try:
        op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), 1e-3, ctx=ctx)
        got = op(v)
    finally:
        ctx.set_option("k1_path", 0)
    dmma = op(v)
    want = oracle.kernel_matvec(x, sigma, 1e-3, v)
    assert rel(got, want) <= 1e-13, rel(got, want)
    assert rel(got, dmma) <= 1e-13


def test_i8_symmetry_diagonal_and_scaled_rows(krr, oracle, ctx):
    """Exact symmetry / unit diagonal on the I8 path, with rows of very different scale
    (per-row exponents) and duplicated rows (d2 clamp)."""
    n, d = 300, 6
    x = oracle.random_matrix(n, d, 2)
    x[::7] *= 1e-3
    x[1::11] *= 40.0
    x[5] = x[6]
    ctx.set_option("k1_path", 1)
    try:
        op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(2.0), 0.0, ctx=ctx)
        kk = op.matmat(np.eye(n))
        kk1 = np.column_stack([op(np.eye(n)[:, j]) for j in range(0, n, 37)])
    finally:
        ctx.set_option("k1_path", 0)
    assert np.array_equal(np.diag(kk), np.ones(n))
    assert np.array_equal(kk, kk.T)
    want = oracle.gram_matrix(x, 2.0)
    assert np.max(np.abs(kk - want)) <= 2e-15
    assert np.max(np.abs(kk1 - want[:, ::37])) <= 2e-15
    assert kk[5, 6] == 1.0


F32_CASES = [(1, 1, 1.0), (300, 4, 1.7), (1000, 90, 6.0), (4097, 16, 4.0), (5000, 54, 3.0), (40000, 90, 6.0),
             (3000, 128, 8.0), (2000, 100, 5.0)]


@pytest.mark.parametrize("n,d,sigma", F32_CASES)
def test_f32_mode_matvec(krr, oracle, ctx, n, d, sigma):
    """Optional fp32 mode (three bf16 parts on tcgen05 kind::f16, fp32 epilogue): K v within
    fp32-level error of the fp64 oracle; the default stays fp64."""
    x = oracle.random_matrix(n, d, 5 + n)
    v = oracle.random_vector(n, 7 + n)
    assert ctx.get_option("precision") == 64
    ctx.set_precision(32)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), 1e-3, ctx=ctx)
    got = op(v)
    assert ctx.get_option("precision") == 32
    want = oracle.kernel_matvec(x, sigma, 1e-3, v)
    assert rel(got, want) <= 2e-6, rel(got, want)
    assert np.array_equal(op(v), got)  # deterministic
    ctx.set_precision(64)
    assert rel(op(v), want) <= 1e-13


def test_f32_mode_gram_entries(krr, oracle, ctx):
    n, d = 300, 6
    x = oracle.random_matrix(n, d, 2)
    ctx.set_precision(32)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(2.0), 0.0, ctx=ctx)
    cols = np.column_stack([op(np.eye(n)[:, j]) for j in range(0, n, 29)])
    want = oracle.gram_matrix(x, 2.0)[:, ::29]
    assert np.max(np.abs(cols - want)) <= 2e-6
    assert np.all(np.abs(cols[np.arange(0, n, 29), np.arange(cols.shape[1])] - 1.0) == 0.0)  # K_ii = 1 exactly


def test_f32_mode_rejects_wide_d_and_bad_bits(krr, oracle, ctx):
    with pytest.raises(ValueError):
        ctx.set_precision(16)
    x = oracle.random_matrix(200, 129, 1)
    ctx.set_precision(32)
    op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(5.0), 1e-3, ctx=ctx)
    with pytest.raises(ValueError):
        op(np.ones(200))
