"""(libkrr_diag.so probes) tcgen05 (5th-gen tensor core) kind::i8 mechanics: descriptors, TMEM accumulators,
commit/mbarrier, tcgen05.ld — checked exactly against an integer matmul."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("K,N", [(32, 32), (96, 64), (256, 64), (64, 32)])
def test_i8_gemm_probe_exact(krr, ctx, K, N):
    from paper_1611_03220_b200 import _diag, _lib
    rng = np.random.default_rng(K + N)
    a = rng.integers(-127, 128, size=(128, K), dtype=np.int8)
    b = rng.integers(-127, 128, size=(N, K), dtype=np.int8)
    c = np.empty((128, N), dtype=np.int32)
    _diag.check(_diag.LIB.krr_diag_i8_gemm(0, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), K, N))
    want = a.astype(np.int64) @ b.astype(np.int64).T
    assert np.array_equal(c.astype(np.int64), want)


def _bf16_bits(x):
    """Round fp32 values to bf16 (nearest even) and return the uint16 bit patterns."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) >> 16
    return u.astype(np.uint16)


def _bf16_value(bits):
    return (bits.astype(np.uint32) << 16).view(np.float32).astype(np.float64)


@pytest.mark.parametrize("K,N", [(16, 32), (96, 64), (128, 64), (48, 32)])
def test_bf16_gemm_probe(krr, ctx, K, N):
    """kind::f16 with BF16 inputs and an FP32 TMEM accumulator (the fp32 mode's MMA)."""
    from paper_1611_03220_b200 import _diag, _lib
    rng = np.random.default_rng(3 * K + N)
    a = _bf16_bits(rng.standard_normal((128, K)))
    b = _bf16_bits(rng.standard_normal((N, K)))
    c = np.empty((128, N), dtype=np.float32)
    _diag.check(_diag.LIB.krr_diag_bf16_gemm(0, _lib.ptr(a), _lib.ptr(b), _lib.ptr(c), K, N))
    want = _bf16_value(a) @ _bf16_value(b).T  # bf16 products are exact in fp32; sums round
    assert np.max(np.abs(c - want)) <= 1e-5 * np.max(np.abs(want)) + 1e-6
