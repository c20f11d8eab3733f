"""pins the oracle's polynomial kernel and sketch-stage restatements against the
reference's own known-answer tests (tests/test_kernels.cpp:19-99, tests/test_sketches.cpp:42-285,
tests/support/oracles.cpp:60-85).  CPU only; the oracle is test infrastructure."""
import itertools
import math

import numpy as np
import pytest

from oracle import oracle_ffi as O


def explicit_tensorsketch(h, g, s, x):
    """tests/support/oracles.cpp:60-85: sum over all index tuples of the tensor power."""
    q, d = h.shape
    out = np.zeros(s)
    for tup in itertools.product(range(d), repeat=q):
        bucket, sign, prod = 0, 1.0, 1.0
        for j, i in enumerate(tup):
            bucket += int(h[j, i])
            sign *= g[j, i]
            prod *= x[i]
        out[bucket % s] += sign * prod
    return out


def tensor_power(v, q):
    out = np.array([1.0])
    for _ in range(q):
        out = np.kron(out, v)
    return out


# --------------------------------------------------------------------------- kernels
def test_poly_orthogonal_inputs_vanish():
    x = np.array([[1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    assert O.poly_cross(x[:1], x[1:], 1.0, 0.0, 3)[0, 0] == pytest.approx(0.0)


def test_poly_arithmetic_known_answer():
    x = np.array([[10.0]])
    assert O.poly_cross(x, x, 0.01, 1.0, 3)[0, 0] == pytest.approx(8.0)


def test_poly_spec_validation():
    x = np.ones((2, 2))
    for g, c, q in [(1.0, -1.0, 2), (1.0, 0.0, 0), (0.0, 1.0, 2)]:
        with pytest.raises(O.OracleError):
            O.poly_gram(x, g, c, q)


@pytest.mark.parametrize("q", [1, 2, 3])
def test_poly_gram_equals_monomial_feature_gram(q):
    x = O.random_matrix(10, 4, q)
    k = O.poly_gram(x, 0.5, 1.5, q)
    xa = O.poly_augment(x, 0.5, 1.5)
    vq = np.stack([tensor_power(r, q) for r in xa])
    expected = vq @ vq.T
    assert np.linalg.norm(k - expected) <= 1e-9 * np.linalg.norm(expected)


def test_poly_cross_and_matvec_agree_with_pairwise():
    a = O.random_matrix(7, 3, 11)
    b = O.random_matrix(5, 3, 12)
    k = O.poly_cross(a, b, 0.7, 0.4, 2)
    for i in range(7):
        for j in range(5):
            assert k[i, j] == pytest.approx((0.7 * a[i] @ b[j] + 0.4) ** 2, rel=1e-12)
    x = O.random_matrix(30, 4, 3)
    v = O.random_vector(30, 4)
    ref = O.poly_gram(x, 0.8, 0.2, 3) @ v + 0.5 * v
    np.testing.assert_allclose(O.poly_matvec(x, 0.8, 0.2, 3, 0.5, v), ref, rtol=1e-12, atol=1e-12)


# --------------------------------------------------------------------------- count sketch / TensorSketch
def test_countsketch_matches_definition():
    h = np.array([[0, 1, 0]], dtype=np.uint32)
    g = np.array([[1.0, -1.0, 1.0]])
    z = O.tensorsketch_apply_rows(h, g, 2, np.array([[1.0, 2.0, 3.0]]))[0]
    assert z.tolist() == [4.0, -2.0]
    assert np.linalg.norm(O.tensorsketch_apply_rows(h, g, 2, np.zeros((1, 3)))) == 0.0
    hid = np.array([[0, 1, 2]], dtype=np.uint32)
    x = np.array([[1.0, 2.0, 3.0]])
    assert np.array_equal(O.tensorsketch_apply_rows(hid, np.ones((1, 3)), 3, x), x)


def test_tensorsketch_degree_one_is_countsketch():
    h, g = O.tensorsketch_realize(21, 6, 5, 1)
    x = O.random_vector(6, 4)
    direct = np.zeros(5)
    for j in range(6):
        direct[h[0, j]] += g[0, j] * x[j]
    assert np.array_equal(O.tensorsketch_apply_rows(h, g, 5, x[None, :])[0], direct)


def test_tensorsketch_fft_path_equals_explicit_tensor_power():
    for d in range(2, 7):
        for q in (1, 2, 3):
            for s in (4, 8, 16):
                for seed in range(8):
                    h, g = O.tensorsketch_realize(10_000 + seed, d, s, q)
                    x = O.random_vector(d, 500 + seed)
                    fast = O.tensorsketch_apply_rows(h, g, s, x[None, :])[0]
                    assert np.abs(fast - explicit_tensorsketch(h, g, s, x)).max() <= 1e-12


def test_tensorsketch_non_power_of_two():
    h, g = O.tensorsketch_realize(9, 4, 7, 3)
    x = O.random_vector(4, 8)
    fast = O.tensorsketch_apply_rows(h, g, 7, x[None, :])[0]
    assert np.abs(fast - explicit_tensorsketch(h, g, 7, x)).max() <= 1e-12


def test_tensorsketch_mean_estimate_converges():
    q = 2
    x = O.random_vector(5, 30, 0.6)
    z = O.random_vector(5, 31, 0.6)
    target = float(x @ z) ** q
    est = []
    for m in range(200):
        h, g = O.tensorsketch_realize(5000 + m, 5, 64, q)
        zz = O.tensorsketch_apply_rows(h, g, 64, np.stack([x, z]))
        est.append(float(zz[0] @ zz[1]))
    est = np.array(est)
    assert abs(est.mean() - target) <= 3.0 * est.std(ddof=1) / math.sqrt(len(est)) + 1e-12


def test_tensorsketch_tables_are_deterministic():
    h1, g1 = O.tensorsketch_realize(77, 6, 32, 3)
    h2, g2 = O.tensorsketch_realize(77, 6, 32, 3)
    assert np.array_equal(h1, h2) and np.array_equal(g1, g2)
    assert h1.max() < 32 and set(np.unique(g1)) <= {-1.0, 1.0}


# --------------------------------------------------------------------------- SRHT
def test_srht_two_point_example_and_zero():
    sign = np.ones(2)
    rows = np.array([0])
    assert O.srht_apply_rows(sign, rows, 2, np.array([[2.0, 3.0]]))[0, 0] == pytest.approx(5.0)
    assert np.linalg.norm(O.srht_apply_rows(sign, rows, 2, np.zeros((1, 2)))) == 0.0


@pytest.mark.parametrize("in_dim", [8, 11])
def test_srht_dense_form_matches_apply(in_dim):
    sign, rows = O.srht_realize(17, in_dim, 5)
    dense = np.empty((5, in_dim))
    for i in range(5):
        for j in range(in_dim):
            parity = bin(int(rows[i]) & j).count("1") & 1
            dense[i, j] = (-1.0 if parity else 1.0) * sign[j] / math.sqrt(5)
    x = O.random_vector(in_dim, 18)
    np.testing.assert_allclose(dense @ x, O.srht_apply_rows(sign, rows, in_dim, x[None, :])[0], atol=1e-12)


def test_srht_preserves_norm_on_average():
    x = O.random_vector(64, 42)
    mean = np.mean([np.sum(O.srht_apply_rows(*O.srht_realize(900 + t, 64, 16), 64, x[None, :]) ** 2)
                    for t in range(500)])
    assert abs(mean - x @ x) <= 0.05 * (x @ x)


# --------------------------------------------------------------------------- Gaussian map
def test_gaussmap_forced_tables_and_norm():
    x = O.random_vector(4, 3)
    assert np.linalg.norm(O.gaussmap_apply_rows(np.zeros((3, 4)), O.random_vector(4, 2)[None, :])) == 0.0
    np.testing.assert_allclose(O.gaussmap_apply_rows(2.0 * np.eye(4), x[None, :])[0], x, atol=1e-15)
    y = O.random_vector(32, 5)
    mean = np.mean([np.sum(O.gaussmap_apply_rows(O.gaussmap_realize(700 + t, 32, 8), y[None, :]) ** 2)
                    for t in range(500)])
    assert abs(mean - y @ y) <= 0.05 * (y @ y)


def test_linear_stages_are_linear():
    h, g = O.tensorsketch_realize(2, 6, 8, 1)
    sg, rw = O.srht_realize(3, 6, 4)
    pj = O.gaussmap_realize(4, 6, 4)
    rng = np.random.default_rng(123)
    maps = [lambda v: O.tensorsketch_apply_rows(h, g, 8, v[None, :])[0],
            lambda v: O.srht_apply_rows(sg, rw, 6, v[None, :])[0],
            lambda v: O.gaussmap_apply_rows(pj, v[None, :])[0]]
    for trial in range(30):
        a, b = rng.normal(size=2)
        x = O.random_vector(6, 2 * trial)
        z = O.random_vector(6, 2 * trial + 1)
        for f in maps:
            rhs = a * f(x) + b * f(z)
            assert np.abs(f(a * x + b * z) - rhs).max() <= 1e-12 * (1.0 + np.abs(rhs).max())


# --------------------------------------------------------------------------- chains
POLY = {"family": "polynomial", "gamma": 0.8, "offset": 0.3, "degree": 2}


def test_chain_bitwise_deterministic():
    x = O.random_matrix(12, 5, 50)
    z1 = O.chain_apply_rows(O.chain_realize("TensorSketch", 32, 16, 8, POLY, 5, 1234), x)
    z2 = O.chain_apply_rows(O.chain_realize("TensorSketch", 32, 16, 8, POLY, 5, 1234), x)
    z3 = O.chain_apply_rows(O.chain_realize("TensorSketch", 32, 16, 8, POLY, 5, 1235), x)
    assert z1.shape == (12, 8)
    assert np.array_equal(z1, z2) and np.abs(z1 - z3).max() > 0.0


def test_chain_scaled_to():
    assert O.chain_scaled_to(1024, 256, 0, 128) == (512, 128, 0)
    assert O.chain_scaled_to(64, 0, 0, 256) == (256, 0, 0)


def test_rff_srht_chain_matches_dense_product():
    gk = {"family": "gaussian", "sigma": 1.0}
    t = O.chain_realize("RandomFourier", 64, 64, 0, gk, 3, 5)
    t["srht_sign"] = np.ones(64)
    t["srht_rows"] = np.arange(64, dtype=np.int64)
    x = O.random_matrix(6, 3, 7)
    z1 = O.rff_apply_rows(x, t["w"], t["b"])
    z = O.chain_apply_rows(t, x)
    h = np.array([[(-1.0) ** bin(i & j).count("1") for j in range(64)] for i in range(64)]) / 8.0
    np.testing.assert_allclose(z, z1 @ h.T, atol=1e-10)
    np.testing.assert_allclose(np.linalg.norm(z, axis=1), np.linalg.norm(z1, axis=1), rtol=1e-10)


def test_poly_train_reduces_residual():
    """A full polynomial-kernel train through the oracle (dense K, TS -> SRHT chain)."""
    x = O.random_matrix(120, 4, 9, 0.5)
    y = O.random_vector(120, 10)
    out = O.train_chain(x, y, {"family": "polynomial", "gamma": 1.0, "offset": 0.5, "degree": 2},
                        "TensorSketch", 64, 32, 0, 0.05, 3, 1e-8, 200)
    assert out.converged[0]
    k = O.poly_gram(x, 1.0, 0.5, 2)
    np.testing.assert_allclose((k + 0.05 * np.eye(120)) @ out.c[:, 0], y, atol=1e-6 * np.linalg.norm(y))
