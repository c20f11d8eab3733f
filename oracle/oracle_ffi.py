"""ctypes binding of oracle/liboracle.so — the CPU restatement of the reference path.

`order` selects the summation order (krr_oracle.cpp): 2 = Eigen-like (the default,
closest to the reference's SSE2/Eigen arithmetic), 0 = forward sequential,
1 = reverse sequential.

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs (cpu_baseline and --impl reference), never by the product package.
Every function cites the reference code it restates (see krr_oracle.cpp's header).
"""
from __future__ import annotations

import ctypes as C
import subprocess
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB_PATH = HERE / "liboracle.so"

DEFAULT_ORDER = 2

OK, DIMENSION_MISMATCH, NOT_POSITIVE_DEFINITE, SINGULAR_TRIANGULAR, BREAKDOWN, \
    NON_POSITIVE_LAMBDA, INVALID_ARGUMENT = range(7)


class OracleError(Exception):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def build() -> Path:
    subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
    return LIB_PATH


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        build()
    return C.CDLL(str(LIB_PATH))


_L = None
_vp, _i64, _d, _i = C.c_void_p, C.c_int64, C.c_double, C.c_int
OP_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)
OBS_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int64)


def lib() -> C.CDLL:
    global _L
    if _L is None:
        L = _load()
        sigs = {
            "oracle_num_threads": ([], _i),
            "oracle_set_num_threads": ([_i], None),
            "oracle_random_matrix": ([_i64, _i64, C.c_uint64, _d, _vp], None),
            "oracle_random_uniform": ([_i64, C.c_uint64, _d, _d, _vp], None),
            "oracle_rff_realize": ([C.c_uint64, _i64, _i64, _d, _vp, _vp], _i),
            "oracle_rff_apply_rows": ([_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i], _i),
            "oracle_gram_matrix": ([_vp, _i64, _i64, _d, _vp, _i], _i),
            "oracle_cross_gram": ([_vp, _i64, _vp, _i64, _i64, _d, _vp, _i], _i),
            "oracle_kernel_matvec": ([_vp, _i64, _i64, _d, _d, _vp, _i64, _vp, _i64, _i64, _i], _i),
            "oracle_dense_matvec": ([_vp, _i64, _d, _vp, _i64, _vp, _i], _i),
            "oracle_cholesky": ([_vp, _i64, _vp], _i),
            "oracle_triangular_solve": ([_vp, _i64, _vp, _i64, _i, _i, _vp], _i),
            "oracle_build_preconditioner": ([_vp, _i64, _i64, _d, _vp, C.POINTER(_i), _i], _i),
            "oracle_precond_apply": ([_vp, _i64, _i64, _d, _vp, _i64, _vp, _i], _i),
            "oracle_pcg_solve": ([_i64, OP_CB, _vp, OP_CB, _vp, _vp, _d, _i, OBS_CB, _vp, _vp,
                                  C.POINTER(_i), C.POINTER(_i), C.POINTER(_d), _vp, _i], _i),
            "oracle_solve_gaussian": ([_vp, _i64, _i64, _d, _d, _vp, _i64, _d, _vp, _i64, _d, _i, _i,
                                       _vp, _vp, _vp, _vp, _vp, C.POINTER(C.c_longlong), _i], _i),
            "oracle_train": ([_vp, _i64, _i64, _vp, _i64, _d, _d, _d, _i64, C.c_uint64, _d, _i, _i,
                              _vp, _vp, _vp, _vp, _vp, C.POINTER(C.c_longlong), _i], _i),
            "oracle_poly_gram": ([_vp, _i64, _i64, _d, _d, _i, _vp, _i], _i),
            "oracle_poly_cross": ([_vp, _i64, _vp, _i64, _i64, _d, _d, _i, _vp, _i], _i),
            "oracle_poly_matvec": ([_vp, _i64, _i64, _d, _d, _i, _d, _vp, _i64, _vp, _i], _i),
            "oracle_poly_augment": ([_vp, _i64, _i64, _d, _d, _vp], _i),
            "oracle_solve_dense": ([_vp, _i64, _d, _vp, _i64, _d, _vp, _i64, _d, _i, _vp, _vp, _vp, _vp, _vp,
                                    C.POINTER(C.c_longlong), _i], _i),
            "oracle_tensorsketch_realize": ([C.c_uint64, _i64, _i64, _i, _vp, _vp], _i),
            "oracle_tensorsketch_apply_rows": ([_vp, _vp, _i64, _i64, _i, _vp, _i64, _vp], _i),
            "oracle_srht_realize": ([C.c_uint64, _i64, _i64, _vp, _vp], _i),
            "oracle_srht_apply_rows": ([_vp, _vp, _i64, _i64, _vp, _i64, _vp], _i),
            "oracle_gaussmap_realize": ([C.c_uint64, _i64, _i64, _vp], _i),
            "oracle_gaussmap_apply_rows": ([_vp, _i64, _i64, _vp, _i64, _vp, _i], _i),
            "oracle_generate_config": ([_i, _i64, _i64, _i64, C.c_uint64, _vp, _vp], _i),
        }
        for name, (args, res) in sigs.items():
            fn = getattr(L, name)
            fn.argtypes = args
            fn.restype = res
        _L = L
    return _L


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def _chk(st: int, what: str) -> None:
    if st != OK:
        raise OracleError(st, what)


def f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def set_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


def random_matrix(rows: int, cols: int, seed: int, scale: float = 1.0) -> np.ndarray:
    out = np.empty((rows, cols))
    lib().oracle_random_matrix(rows, cols, seed, scale, _p(out))
    return out


def random_vector(n: int, seed: int, scale: float = 1.0) -> np.ndarray:
    return random_matrix(n, 1, seed, scale)[:, 0].copy()


def random_uniform(count: int, seed: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(count)
    lib().oracle_random_uniform(count, seed, lo, hi, _p(out))
    return out


def generate_config(cfg: int, n: int, d: int, t: int = 1, seed: int = 0):
    """BASELINE config generators, restated independently of the product
    library: bench.py's CPU legs and the config fixtures use this one.  Returns (X n x d, Y n x t)."""
    x = np.empty((n, d))
    y = np.empty((n, t))
    _chk(lib().oracle_generate_config(int(cfg), n, d, t, C.c_uint64(seed), _p(x), _p(y)), "generate_config")
    return x, y


def rff_realize(master_seed: int, d: int, s: int, sigma: float):
    w, b = np.empty((s, d)), np.empty(s)
    _chk(lib().oracle_rff_realize(master_seed, d, s, sigma, _p(w), _p(b)), "rff_realize")
    return w, b


def rff_apply_rows(x, w, b, order: int = DEFAULT_ORDER) -> np.ndarray:
    x, w, b = f64(x), f64(w), f64(b)
    z = np.empty((x.shape[0], w.shape[0]))
    _chk(lib().oracle_rff_apply_rows(_p(x), x.shape[0], x.shape[1], _p(w), _p(b), w.shape[0], _p(z),
                                     order), "rff_apply_rows")
    return z


def gram_matrix(x, sigma: float, order: int = DEFAULT_ORDER) -> np.ndarray:
    x = f64(x)
    k = np.empty((x.shape[0], x.shape[0]))
    _chk(lib().oracle_gram_matrix(_p(x), x.shape[0], x.shape[1], sigma, _p(k), order), "gram")
    return k


def cross_gram(a, b, sigma: float, order: int = DEFAULT_ORDER) -> np.ndarray:
    a, b = f64(a), f64(b)
    k = np.empty((a.shape[0], b.shape[0]))
    _chk(lib().oracle_cross_gram(_p(a), a.shape[0], _p(b), b.shape[0], a.shape[1], sigma, _p(k), order),
         "cross_gram")
    return k


def kernel_matvec(x, sigma: float, lam: float, v, rows=None, order: int = DEFAULT_ORDER) -> np.ndarray:
    """((K + lam I) V)[rows] with K on the fly (V n or n x t)."""
    x = f64(x)
    v = f64(v)
    vec = v.ndim == 1
    v2 = v[:, None] if vec else v
    n = x.shape[0]
    r0, r1 = (0, n) if rows is None else rows
    out = np.empty((r1 - r0, v2.shape[1]))
    _chk(lib().oracle_kernel_matvec(_p(x), n, x.shape[1], sigma, lam, _p(f64(v2)), v2.shape[1], _p(out),
                                    r0, r1, order), "kernel_matvec")
    return out[:, 0] if vec else out


def cholesky(a) -> np.ndarray:
    a = f64(a)
    out = np.empty_like(a)
    _chk(lib().oracle_cholesky(_p(a), a.shape[0], _p(out)), "cholesky")
    return out


def triangular_solve(l, b, side: str = "left", transpose: bool = False) -> np.ndarray:
    l, b = f64(l), f64(b)
    s = l.shape[0]
    m = b.shape[1] if side == "left" else b.shape[0]
    out = np.empty_like(b)
    _chk(lib().oracle_triangular_solve(_p(l), s, _p(b), m, 0 if side == "left" else 1, int(transpose),
                                       _p(out)), "triangular_solve")
    return out


def build_preconditioner(z, lambda_p: float, order: int = DEFAULT_ORDER):
    """Returns (U s x n, jitter_used)."""
    z = f64(z)
    n, s = z.shape
    u = np.empty((s, n))
    jit = C.c_int(0)
    _chk(lib().oracle_build_preconditioner(_p(z), n, s, lambda_p, _p(u), C.byref(jit), order),
         "build_preconditioner")
    return u, bool(jit.value)


def precond_apply(u, lambda_p: float, x, order: int = DEFAULT_ORDER) -> np.ndarray:
    u, x = f64(u), f64(x)
    vec = x.ndim == 1
    x2 = x[:, None] if vec else x
    out = np.empty_like(x2)
    _chk(lib().oracle_precond_apply(_p(u), u.shape[0], u.shape[1], lambda_p, _p(f64(x2)), x2.shape[1],
                                    _p(out), order), "precond_apply")
    return out[:, 0] if vec else out


@dataclass
class PcgOut:
    solution: np.ndarray
    iterations: int
    converged: bool
    final_residual: float
    residual_history: list = field(default_factory=list)


def pcg_solve(apply_a, apply_m, y, tau: float, max_iter: int, observer=None, order: int = DEFAULT_ORDER) -> PcgOut:
    """solver.cpp:22-67 with Python operators."""
    y = f64(y)
    n = y.shape[0]
    errs = []

    def wrap(fn):
        def cb(_u, inp, out, nn):
            try:
                v = np.ctypeslib.as_array(inp, shape=(nn,)).copy()
                np.ctypeslib.as_array(out, shape=(nn,))[:] = np.asarray(fn(v), dtype=np.float64)
                return 0
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                return 1
        return OP_CB(cb)

    ca = wrap(apply_a)
    cm = wrap(apply_m) if apply_m is not None else OP_CB()

    def ob(_u, it, xp, nn):
        observer(int(it), np.ctypeslib.as_array(xp, shape=(nn,)).copy())

    co = OBS_CB(ob) if observer is not None else OBS_CB()
    x = np.zeros(n)
    it, cv, fr = C.c_int(0), C.c_int(0), C.c_double(0)
    hist = np.zeros(max(1, max_iter))
    st = lib().oracle_pcg_solve(n, ca, None, cm, None, _p(y), tau, max_iter, co, None, _p(x),
                                C.byref(it), C.byref(cv), C.byref(fr), _p(hist), order)
    if errs:
        raise errs[0]
    _chk(st, "pcg_solve")
    return PcgOut(x, it.value, bool(cv.value), fr.value, list(hist[: it.value]))


@dataclass
class SolveOut:
    c: np.ndarray
    iterations: list
    converged: list
    final_residual: list
    residual_history: np.ndarray
    total_matvecs: int


def solve_gaussian(x, sigma, lam, u, lambda_p, y, tau, max_iter, dense_k=True, order=DEFAULT_ORDER) -> SolveOut:
    x, y = f64(x), f64(y)
    y2 = y[:, None] if y.ndim == 1 else y
    n, t = y2.shape
    c = np.empty((n, t))
    its = np.zeros(t, dtype=np.int32)
    cvs = np.zeros(t, dtype=np.int32)
    frs = np.zeros(t)
    hist = np.zeros((t, max(1, max_iter)))
    tot = C.c_longlong(0)
    uptr = None if u is None else _p(f64(u))
    s = 0 if u is None else u.shape[0]
    _chk(lib().oracle_solve_gaussian(_p(x), n, x.shape[1], sigma, lam, uptr, s, lambda_p, _p(f64(y2)), t,
                                     tau, max_iter, int(dense_k), _p(c), _p(its), _p(cvs), _p(frs),
                                     _p(hist), C.byref(tot), order), "solve_gaussian")
    return SolveOut(c, its.tolist(), [bool(v) for v in cvs], frs.tolist(), hist, int(tot.value))


def train(x, y, sigma, lam, s, seed, tau, max_iter, lambda_p=None, dense_k=True, order=DEFAULT_ORDER) -> SolveOut:
    """solver.cpp:96-133, non-adaptive RFF chain."""
    x, y = f64(x), f64(y)
    y2 = y[:, None] if y.ndim == 1 else y
    n, t = y2.shape
    c = np.empty((n, t))
    its = np.zeros(t, dtype=np.int32)
    cvs = np.zeros(t, dtype=np.int32)
    frs = np.zeros(t)
    hist = np.zeros((t, max(1, max_iter)))
    tot = C.c_longlong(0)
    lp = -1.0 if lambda_p is None else lambda_p
    _chk(lib().oracle_train(_p(x), n, x.shape[1], _p(f64(y2)), t, sigma, lam, lp, s, seed, tau, max_iter,
                            int(dense_k), _p(c), _p(its), _p(cvs), _p(frs), _p(hist), C.byref(tot), order),
         "train")
    return SolveOut(c, its.tolist(), [bool(v) for v in cvs], frs.tolist(), hist, int(tot.value))


def rf_baseline(x, y, sigma: float, lam: float, s: int, seed: int, order: int = DEFAULT_ORDER):
    """train_random_features_baseline (solver.cpp:175-193) composed from the restated pieces:
    Z = apply_rows (sketches.cpp:207-211), gram = Z^T Z + lambda I, L = cholesky
    (numerics.cpp:49-55), forward = L^-1 Z^T Y, w = L^-T forward (numerics.cpp:57-79).
    Returns (w, W, b).  Test infrastructure only."""
    x = f64(x)
    y = f64(y)
    y = y[:, None] if y.ndim == 1 else y
    w_rff, b_rff = rff_realize(seed, x.shape[1], s, sigma)
    z = rff_apply_rows(x, w_rff, b_rff, order)
    gram = z.T @ z
    gram[np.diag_indices(s)] += lam
    l = cholesky(gram)
    rhs = z.T @ y
    fwd = triangular_solve(l, rhs)
    w = triangular_solve(l, fwd, side="left", transpose=True)
    return w, w_rff, b_rff


def quality_test(x, sigma, z, lam: float, order: int = DEFAULT_ORDER, k=None) -> dict:
    """quality_test (precond.cpp:60-100) restated with the dense oracle K (small n only):
    retained_left_singular_basis (precond.cpp:42-58) through eig(Z'Z) (Eigen sorts ascending,
    the reference flips to descending, numerics.cpp:144-154), condition 1 by the reference's
    power iteration (numerics.cpp:156-190: mt19937_64(7) normal start, tol 1e-4, 500 its) on
    (I-P)K(I-P), condition 2 from eig(Sigma^-1 (B'KB) Sigma^-1).  Test infrastructure only."""
    x, z = f64(x), f64(z)
    n, s = z.shape
    if k is None:
        k = gram_matrix(x, sigma, order)
    rep = {"lambda": lam, "sketch_size": s, "spectrum_cut": 0.05 * lam, "cond1_threshold": 0.1 * lam,
           "cond2_ratio_low": 1.0, "cond2_ratio_high": 1.0}
    ev, vec = np.linalg.eigh(z.T @ z)
    ev, vec = ev[::-1], vec[:, ::-1]
    max_ev = max(0.0, ev[0]) if s else 0.0
    kk = 0
    while kk < s and ev[kk] > rep["spectrum_cut"] and ev[kk] > 1e-20 * max_ev:
        kk += 1
    rep["rank_of_p"] = kk
    b = z @ vec[:, :kk] / np.sqrt(ev[:kk])

    def deflated(v):
        w = v - b @ (b.T @ v)
        w = k @ w
        return w - b @ (b.T @ w)

    v = random_matrix(n, 1, 7)[:, 0]
    v = v / np.linalg.norm(v)
    prev, val = 0.0, 0.0
    for it in range(1, 501):
        w = deflated(v)
        rq = float(v @ w)
        val = rq
        nw = float(np.linalg.norm(w))
        if nw == 0.0:
            val = 0.0
            break
        if it > 1 and abs(rq - prev) <= 1e-4 * abs(rq):
            break
        prev = rq
        v = w / nw
    rep["cond1_value"] = val
    if kk > 0:
        inv = 1.0 / np.sqrt(ev[:kk])
        m = (b.T @ k @ b) * inv[:, None] * inv[None, :]
        m = (m + m.T) / 2.0
        e2 = np.linalg.eigvalsh(m)
        rep["cond2_ratio_high"], rep["cond2_ratio_low"] = float(e2[-1]), float(e2[0])
    rep["passed"] = (rep["cond1_value"] <= rep["cond1_threshold"] and rep["cond2_ratio_low"] >= 0.9
                     and rep["cond2_ratio_high"] <= 1.1)
    return rep


ATTEMPT_SEED_STRIDE = 0xD1B54A32D192ED03  # sketches.hpp:16


def adaptive_sizes(x, sigma: float, lam: float, s0: int, s_max: int, master_seed: int) -> list:
    """adaptive_build's doubling loop (precond.cpp:107-138) with the oracle quality test:
    returns [(s, report), ...] per attempt."""
    out, s = [], s0
    for attempt in range(64):
        seed = (master_seed + attempt * ATTEMPT_SEED_STRIDE) % (1 << 64)
        w, b = rff_realize(seed, x.shape[1], s, sigma)
        rep = quality_test(x, sigma, rff_apply_rows(x, w, b), lam)
        out.append((s, rep))
        if rep["passed"] or s >= s_max:
            break
        s = min(2 * s, s_max)
    return out


# ============================================================================= SURVEY 8f4
# Polynomial kernel and the TensorSketch / SRHT / Gaussian sketch chain.  Kernels are
# passed as dicts {"family": "gaussian", "sigma": S} or {"family": "polynomial",
# "gamma": G, "offset": C, "degree": Q} (kernels.hpp:15-27).

STAGE_SEED_STRIDE = 0x9E3779B97F4A7C15  # sketches.hpp:14


def stage_seed(master: int, stage: int) -> int:
    """sketches.cpp:18-20."""
    return (int(master) + (stage + 1) * STAGE_SEED_STRIDE) % (1 << 64)


def poly_gram(x, gamma: float, offset: float, degree: int, order: int = DEFAULT_ORDER) -> np.ndarray:
    """kernels.cpp:89-99."""
    x = f64(x)
    k = np.empty((x.shape[0], x.shape[0]))
    _chk(lib().oracle_poly_gram(_p(x), x.shape[0], x.shape[1], gamma, offset, degree, _p(k), order), "poly_gram")
    return k


def poly_cross(q, x, gamma: float, offset: float, degree: int, order: int = DEFAULT_ORDER) -> np.ndarray:
    """kernels.cpp:103-121 (polynomial branch)."""
    q, x = f64(q), f64(x)
    k = np.empty((q.shape[0], x.shape[0]))
    _chk(lib().oracle_poly_cross(_p(q), q.shape[0], _p(x), x.shape[0], x.shape[1], gamma, offset, degree, _p(k),
                                 order), "poly_cross")
    return k


def poly_matvec(x, gamma, offset, degree, lam, v, order: int = DEFAULT_ORDER) -> np.ndarray:
    x, v = f64(x), f64(v)
    v2 = v[:, None] if v.ndim == 1 else v
    out = np.empty_like(v2)
    _chk(lib().oracle_poly_matvec(_p(x), x.shape[0], x.shape[1], gamma, offset, degree, lam, _p(v2), v2.shape[1],
                                  _p(out), order), "poly_matvec")
    return out[:, 0].copy() if v.ndim == 1 else out


def poly_augment(x, gamma: float, offset: float) -> np.ndarray:
    """kernels.cpp:56-62."""
    x = f64(x)
    out = np.empty((x.shape[0], x.shape[1] + 1))
    _chk(lib().oracle_poly_augment(_p(x), x.shape[0], x.shape[1], gamma, offset, _p(out)), "poly_augment")
    return out


def kernel_gram(x, kernel: dict, order: int = DEFAULT_ORDER) -> np.ndarray:
    if kernel["family"] == "gaussian":
        return gram_matrix(x, kernel["sigma"], order)
    return poly_gram(x, kernel["gamma"], kernel["offset"], kernel["degree"], order)


def tensorsketch_realize(seed: int, in_dim: int, s: int, degree: int):
    """TensorSketchMap ctor (sketches.cpp:51-69) with the map's own seed."""
    h = np.empty((degree, in_dim), dtype=np.uint32)
    g = np.empty((degree, in_dim))
    _chk(lib().oracle_tensorsketch_realize(seed % (1 << 64), in_dim, s, degree, _p(h), _p(g)), "tensorsketch_realize")
    return h, g


def tensorsketch_apply_rows(h, g, s: int, x) -> np.ndarray:
    """TensorSketchMap::apply (sketches.cpp:71-93) row by row."""
    h = np.ascontiguousarray(h, dtype=np.uint32)
    g, x = f64(g), f64(x)
    z = np.empty((x.shape[0], s))
    _chk(lib().oracle_tensorsketch_apply_rows(_p(h), _p(g), h.shape[1], s, h.shape[0], _p(x), x.shape[0], _p(z)),
         "tensorsketch_apply_rows")
    return z


def srht_realize(seed: int, in_dim: int, s: int):
    """SrhtMap ctor (sketches.cpp:95-109)."""
    p = 1
    while p < in_dim:
        p <<= 1
    sign = np.empty(p)
    rows = np.empty(s, dtype=np.int64)
    _chk(lib().oracle_srht_realize(seed % (1 << 64), in_dim, s, _p(sign), _p(rows)), "srht_realize")
    return sign, rows


def srht_apply_rows(sign, rows, in_dim: int, x) -> np.ndarray:
    """SrhtMap::apply (sketches.cpp:111-121)."""
    sign, x = f64(sign), f64(x)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    z = np.empty((x.shape[0], rows.shape[0]))
    _chk(lib().oracle_srht_apply_rows(_p(sign), _p(rows), in_dim, rows.shape[0], _p(x), x.shape[0], _p(z)),
         "srht_apply_rows")
    return z


def gaussmap_realize(seed: int, in_dim: int, s: int) -> np.ndarray:
    """GaussianMap ctor (sketches.cpp:128-135)."""
    proj = np.empty((s, in_dim))
    _chk(lib().oracle_gaussmap_realize(seed % (1 << 64), in_dim, s, _p(proj)), "gaussmap_realize")
    return proj


def gaussmap_apply_rows(proj, x, order: int = DEFAULT_ORDER) -> np.ndarray:
    """GaussianMap::apply (sketches.cpp:137-140)."""
    proj, x = f64(proj), f64(x)
    z = np.empty((x.shape[0], proj.shape[0]))
    _chk(lib().oracle_gaussmap_apply_rows(_p(proj), proj.shape[1], proj.shape[0], _p(x), x.shape[0], _p(z), order),
         "gaussmap_apply_rows")
    return z


def chain_realize(first: str, s1: int, s2: int, s3: int, kernel: dict, d: int, master_seed: int) -> dict:
    """realize_chain (sketches.cpp:213-242): stage 0 RFF (Gaussian) or TensorSketch on the
    d+1 augmented inputs (polynomial), stage 1 SRHT, stage 2 Gaussian map."""
    t = {"first": first, "s1": s1, "s2": s2, "s3": s3, "kernel": dict(kernel), "d": d}
    if first == "RandomFourier":
        t["w"], t["b"] = rff_realize(master_seed, d, s1, kernel["sigma"])
    else:
        t["hash"], t["sign"] = tensorsketch_realize(stage_seed(master_seed, 0), d + 1, s1, kernel["degree"])
    prev = s1
    if s2 > 0:
        t["srht_sign"], t["srht_rows"] = srht_realize(stage_seed(master_seed, 1), prev, s2)
        t["srht_in"] = prev
        prev = s2
    if s3 > 0:
        t["proj"] = gaussmap_realize(stage_seed(master_seed, 2), prev, s3)
        prev = s3
    return t


def chain_apply_rows(t: dict, x, order: int = DEFAULT_ORDER) -> np.ndarray:
    """SketchChain::apply_rows (sketches.cpp:194-211)."""
    x = f64(x)
    k = t["kernel"]
    if t["first"] == "RandomFourier":
        z = rff_apply_rows(x, t["w"], t["b"], order)
    else:
        z = tensorsketch_apply_rows(t["hash"], t["sign"], t["s1"], poly_augment(x, k["gamma"], k["offset"]))
    if t["s2"] > 0:
        z = srht_apply_rows(t["srht_sign"], t["srht_rows"], t["srht_in"], z)
    if t["s3"] > 0:
        z = gaussmap_apply_rows(t["proj"], z, order)
    return z


def chain_scaled_to(s1: int, s2: int, s3: int, target: int):
    """ChainSpec::scaled_to (sketches.cpp:173-192)."""
    import math
    out_dim = s3 or s2 or s1
    factor = float(target) / float(out_dim)

    def scale(v):
        return max(target, int(math.ceil(float(v) * factor)))

    n1 = scale(s1)
    n2 = scale(s2) if s2 > 0 else 0
    n3 = scale(s3) if s3 > 0 else 0
    if n3 > 0:
        n3 = target
    elif n2 > 0:
        n2 = target
    else:
        n1 = target
    return n1, n2, n3


def solve_dense(k, lam, u, lambda_p, y, tau, max_iter, order=DEFAULT_ORDER) -> SolveOut:
    """solve_regularized (solver.cpp:69-94) on a given dense K."""
    k, y = f64(k), f64(y)
    y2 = y[:, None] if y.ndim == 1 else y
    n, t = y2.shape
    c = np.empty((n, t))
    its = np.zeros(t, dtype=np.int32)
    cvs = np.zeros(t, dtype=np.int32)
    frs = np.zeros(t)
    hist = np.zeros((t, max(1, max_iter)))
    tot = C.c_longlong(0)
    uptr = None if u is None else _p(f64(u))
    s = 0 if u is None else u.shape[0]
    _chk(lib().oracle_solve_dense(_p(k), n, lam, uptr, s, lambda_p, _p(f64(y2)), t, tau, max_iter, _p(c), _p(its),
                                  _p(cvs), _p(frs), _p(hist), C.byref(tot), order), "solve_dense")
    return SolveOut(c, its.tolist(), [bool(v) for v in cvs], frs.tolist(), hist, int(tot.value))


def train_chain(x, y, kernel: dict, first: str, s1: int, s2: int, s3: int, lam: float, seed: int, tau: float,
                max_iter: int, lambda_p=None, order=DEFAULT_ORDER) -> SolveOut:
    """train (solver.cpp:96-133) for any kernel family and chain, dense K (small n)."""
    lp = lam if lambda_p is None else lambda_p
    t = chain_realize(first, s1, s2, s3, kernel, f64(x).shape[1], seed)
    z = chain_apply_rows(t, x, order)
    u, _ = build_preconditioner(z, lp, order)
    return solve_dense(kernel_gram(x, kernel, order), lam, u, lp, y, tau, max_iter, order)


def adaptive_sizes_chain(x, kernel: dict, first: str, s1: int, s2: int, s3: int, lam: float, s0: int, s_max: int,
                         master_seed: int) -> list:
    """adaptive_build (precond.cpp:107-138) for any chain template: attempt a realizes
    chain_template.scaled_to(s) with master + a * kAttemptSeedStride."""
    k = kernel_gram(x, kernel)
    out, s = [], s0
    for attempt in range(64):
        seed = (master_seed + attempt * ATTEMPT_SEED_STRIDE) % (1 << 64)
        a1, a2, a3 = chain_scaled_to(s1, s2, s3, s)
        t = chain_realize(first, a1, a2, a3, kernel, f64(x).shape[1], seed)
        rep = quality_test(x, None, chain_apply_rows(t, x), lam, k=k)
        out.append((s, rep))
        if rep["passed"] or s >= s_max:
            break
        s = min(2 * s, s_max)
    return out
