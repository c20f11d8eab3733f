"""tcgen05 (5th-gen tensor core) kind::i8 mechanics: descriptors, TMEM accumulators,
commit/mbarrier, tcgen05.ld — checked exactly against an integer matmul."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,N", [(32, 32), (96, 64), (256, 64), (64, 32)])
def test_i8_gemm_probe_exact(krr, ctx, K, N):
    from paper_1611_03220_b200 import _lib
    rng = np.random.default_rng(K + N)
    a = rng.integers(-127, 128, size=(128, K), dtype=np.int8)
    b = rng.integers(-127, 128, size=(N, K), dtype=np.int8)
    c = np.empty((128, N), dtype=np.int32)
    _lib.check(_lib.LIB.krr_debug_i8_gemm(ctx.handle, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), K, N))
    want = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(c.astype(np.int64), want)
