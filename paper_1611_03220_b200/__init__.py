"""B200-native sketch-preconditioned kernel ridge regression (arXiv 1611.03220 hot path).

Host-side mirror of the reference's C++ operator / preconditioner / solver API
(/root/reference/proj/core/include/krr/{kernels,sketches,precond,solver}.hpp), backed
by the CUDA library libkrr_b200.so through its C-ABI (include/krr_b200.h).  Same names,
same argument meaning, same error behaviour (exceptions map 1:1 onto types.hpp).
All compute runs on the GPU; there is no CPU fallback.

Reference -> here
  krr::kernels::KernelSpec::gaussian          KernelSpec.gaussian
  krr::kernels::Dataset                       Dataset
  krr::sketches::RffMap / ChainSpec / realize_chain / SketchChain::apply_rows
  krr::precond::build_preconditioner / Preconditioner::{apply, apply_columns}
  krr::solver::pcg_solve(LinearOperator...)   pcg_solve  (device vector algebra, host operators)
  krr::solver::solve_regularized(K, ...)      solve_regularized(x, kernel, ...)  (K on the fly)
  krr::solver::train / predict_scores / predict_labels / rlsc_encode / rlsc_decode
  apply_a lambda over gram_matrix             GaussianOperator (fused on-the-fly K1 kernel)
"""
from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import (  # noqa: F401  (re-exported exception types)
    BreakdownDetected,
    CallbackError,
    Context,
    CudaError,
    DimensionMismatch,
    InvalidArgument,
    KrrError,
    ModelFileError,
    NcclError,
    NoConvergence,
    NonPositiveLambda,
    NotPositiveDefinite,
    SingularTriangular,
    StateError,
    device_count,
    nccl_unique_id,
)

__all__ = [
    "KernelSpec", "Dataset", "RffMap", "TensorSketchMap", "SrhtMap", "GaussianMap", "ChainSpec", "SketchChain",
    "realize_chain", "KernelOperator",
    "Preconditioner", "build_preconditioner", "GaussianOperator", "SolverConfig", "RhsStats",
    "PcgReport", "PcgResult", "KrrModel", "TrainResult", "pcg_solve", "solve_regularized", "solve_regularized_dense",
    "train", "predict_scores", "predict_labels", "rlsc_encode", "rlsc_decode",
    "generate_config", "schedule", "Context", "device_count",
    "save_model", "load_model", "ModelFileError", "NoConvergence",
    "QualityReport", "quality_test", "AdaptiveResult", "adaptive_build", "default_initial_sketch_size",
    "RandomFeaturesModel", "train_random_features_baseline", "baseline_predict_scores", "baseline_predict_labels",
]

K_STAGE_SEED_STRIDE = 0x9E3779B97F4A7C15  # sketches.hpp:14


# ----------------------------------------------------------------------------- kernels.hpp
@dataclass
class KernelSpec:
    """KernelSpec (kernels.hpp:15-27): the Gaussian kernel exp(-|x-z|^2 / 2 sigma^2) or the
    polynomial kernel (gamma x.z + offset)^degree."""

    family: str = "gaussian"
    sigma: float = 1.0
    gamma: float = 1.0
    offset: float = 0.0
    degree: int = 2

    @staticmethod
    def gaussian(sigma: float) -> "KernelSpec":
        spec = KernelSpec("gaussian", float(sigma))
        spec.validate()
        return spec

    @staticmethod
    def polynomial(gamma: float, offset: float, degree: int) -> "KernelSpec":
        spec = KernelSpec("polynomial", 1.0, float(gamma), float(offset), int(degree))
        spec.validate()
        return spec

    def validate(self) -> None:  # kernels.cpp:36-44
        if self.family == "gaussian":
            if not (self.sigma > 0.0):
                raise InvalidArgument("KernelSpec: sigma must be positive")
        elif self.family == "polynomial":
            if self.degree < 1:
                raise InvalidArgument("KernelSpec: degree must be at least 1")
            if self.offset < 0.0:
                raise InvalidArgument("KernelSpec: offset must be non-negative")
            if not (self.gamma > 0.0):
                raise InvalidArgument("KernelSpec: gamma must be positive")
        else:
            raise InvalidArgument(f"KernelSpec: unknown kernel family '{self.family}'")

    def _c(self) -> "_lib.KernelSpecC":
        return _lib.KernelSpecC(0 if self.family == "gaussian" else 1, int(self.degree), float(self.sigma),
                                float(self.gamma), float(self.offset))


def _set_data(ctx: Context, x: np.ndarray, kernel: KernelSpec) -> None:
    kc = kernel._c()
    _lib.check(_lib.LIB.krr_set_data_kernel(ctx.handle, _lib.ptr(x), x.shape[0], x.shape[1], C.byref(kc)))


@dataclass
class Dataset:
    """kernels.hpp:33-43: x n x d, y n x t (RLSC +/-1 for classification)."""

    x: np.ndarray
    y: np.ndarray
    labels: list = field(default_factory=list)
    label_map: list = field(default_factory=list)

    def classification(self) -> bool:
        return len(self.label_map) > 0

    def n(self) -> int:
        return int(np.asarray(self.x).shape[0])

    def dim(self) -> int:
        return int(np.asarray(self.x).shape[1])

    def targets(self) -> int:
        y = np.asarray(self.y)
        return 1 if y.ndim == 1 else int(y.shape[1])


# ----------------------------------------------------------------------------- sketches.hpp
class RffMap:
    """Random Fourier features (sketches.hpp:21-31).  W, b drawn on the host with the
    reference's libstdc++ RNG (sketches.cpp:24-35), so they are bitwise identical."""

    def __init__(self, input_dim: int, features: int, sigma: float, seed: int):
        if features < 1:
            raise InvalidArgument("RffMap: need at least one feature")
        if not (sigma > 0.0):
            raise InvalidArgument("RffMap: sigma must be positive")
        self.w = np.empty((features, input_dim))
        self.b = np.empty(features)
        self.seed = int(seed)
        self.sigma = float(sigma)
        # krr_rff_realize applies stage_seed(master, 0) = master + stride; pass seed - stride.
        master = (int(seed) - K_STAGE_SEED_STRIDE) % (1 << 64)
        _lib.check(_lib.LIB.krr_rff_realize(master, input_dim, features, sigma,
                                            _lib.ptr(self.w), _lib.ptr(self.b)))

    def input_dim(self) -> int:
        return self.w.shape[1]

    def output_dim(self) -> int:
        return self.w.shape[0]

    def apply_rows(self, x: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
        """Z with row i = sqrt(2/s) cos(W x_i + b), built on the device (K2)."""
        x = _lib.f64(x)
        if x.ndim != 2 or x.shape[1] != self.input_dim():
            raise DimensionMismatch("RffMap: input dimension mismatch")
        n, s = x.shape[0], self.output_dim()
        if n == 0:
            return np.zeros((0, s))
        own = ctx is None
        ctx = ctx or Context()
        try:
            _lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, x.shape[1], self.sigma))
            _lib.check(_lib.LIB.krr_rff_build(ctx.handle, _lib.ptr(self.w), _lib.ptr(self.b), s))
            z = np.empty((n, s))
            _lib.check(_lib.LIB.krr_rff_download(ctx.handle, _lib.ptr(z)))
            return z
        finally:
            if own:
                ctx.close()

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = _lib.f64(x)
        if x.ndim != 1 or x.shape[0] != self.input_dim():
            raise DimensionMismatch("RffMap: input dimension mismatch")
        return self.apply_rows(x[None, :])[0]


class TensorSketchMap:
    """TensorSketchMap (sketches.hpp:45-62): per mode a hash table (buckets in [0, s)) and a
    +-1 sign table, drawn on the host with the reference's libstdc++ distributions in its
    order (sketches.cpp:51-69).  Tables are public and may be overwritten, as in the
    reference's tests; the device applies them through SketchChain.apply_rows."""

    def __init__(self, input_dim: int, features: int, degree: int, seed: int):
        if features < 1:
            raise InvalidArgument("TensorSketchMap: need at least one feature")
        if degree < 1:
            raise InvalidArgument("TensorSketchMap: degree must be >= 1")
        self.in_dim, self.out_dim, self.degree, self.seed = int(input_dim), int(features), int(degree), int(seed)
        self.hash = np.empty((degree, input_dim), dtype=np.uint32)
        self.sign = np.empty((degree, input_dim))
        _lib.check(_lib.LIB.krr_tensorsketch_realize(int(seed) % (1 << 64), input_dim, features, degree,
                                                     _lib.ptr(self.hash), _lib.ptr(self.sign)))


class SrhtMap:
    """SrhtMap (sketches.hpp:64-79): sign (next_pow2(in) entries) then sampled rows, drawn
    as sketches.cpp:95-109 does."""

    def __init__(self, input_dim: int, features: int, seed: int):
        if features < 1:
            raise InvalidArgument("SrhtMap: need at least one feature")
        if input_dim < 1:
            raise InvalidArgument("SrhtMap: input dimension must be positive")
        self.in_dim, self.out_dim, self.seed = int(input_dim), int(features), int(seed)
        self.padded_dim = 1 << max(0, (int(input_dim) - 1).bit_length())
        self.sign = np.empty(self.padded_dim)
        self.rows = np.empty(features, dtype=np.int64)
        _lib.check(_lib.LIB.krr_srht_realize(int(seed) % (1 << 64), input_dim, features, _lib.ptr(self.sign),
                                             _lib.ptr(self.rows)))

    def dense(self) -> np.ndarray:
        """SrhtMap::dense (sketches.cpp:123-135)."""
        i = self.rows[:, None].astype(np.uint64)
        j = np.arange(self.in_dim, dtype=np.uint64)[None, :]
        bits = np.unpackbits((i & j).view(np.uint8).reshape(len(self.rows), self.in_dim, 8), axis=2).sum(axis=2)
        return np.where(bits & 1, -1.0, 1.0) * self.sign[None, :self.in_dim] / math.sqrt(self.out_dim)


class GaussianMap:
    """GaussianMap (sketches.hpp:81-92): proj (s x in) standard normals (sketches.cpp:128-135)."""

    def __init__(self, input_dim: int, features: int, seed: int):
        if features < 1:
            raise InvalidArgument("GaussianMap: need at least one feature")
        self.seed = int(seed)
        self.proj = np.empty((features, input_dim))
        _lib.check(_lib.LIB.krr_gaussmap_realize(int(seed) % (1 << 64), input_dim, features, _lib.ptr(self.proj)))

    def dense(self) -> np.ndarray:
        return self.proj / math.sqrt(self.proj.shape[0])


_FIRST = {"RandomFourier": 0, "TensorSketch": 1}


@dataclass
class ChainSpec:
    """ChainSpec (sketches.hpp:96-107): first stage RandomFourier (Gaussian kernel) or
    TensorSketch (polynomial kernel), optional SRHT (s2) and Gaussian (s3) stages."""

    first: str = "RandomFourier"
    s1: int = 0
    s2: int = 0
    s3: int = 0

    def validate(self) -> None:  # sketches.cpp:155-165
        if self.first not in _FIRST:
            raise InvalidArgument(f"ChainSpec: unknown first stage '{self.first}'")
        if self.s1 < 1:
            raise InvalidArgument("ChainSpec: s1 must be at least 1")
        if self.s2 < 0 or self.s3 < 0:
            raise InvalidArgument("ChainSpec: stage sizes must be non-negative")
        prev = self.s1
        if self.s2 > 0:
            if self.s2 > prev:
                raise InvalidArgument("ChainSpec: stage sizes must be non-increasing")
            prev = self.s2
        if self.s3 > 0 and self.s3 > prev:
            raise InvalidArgument("ChainSpec: stage sizes must be non-increasing")

    def output_dim(self) -> int:
        return self.s3 or self.s2 or self.s1

    def scaled_to(self, target: int) -> "ChainSpec":
        """sketches.cpp:173-192."""
        out = _lib.ChainSpecC()
        _lib.check(_lib.LIB.krr_chain_scaled_to(C.byref(self._c()), int(target), C.byref(out)))
        return ChainSpec(self.first, int(out.s1), int(out.s2), int(out.s3))

    def _c(self) -> "_lib.ChainSpecC":
        if self.first not in _FIRST:
            raise InvalidArgument(f"ChainSpec: unknown first stage '{self.first}'")
        return _lib.ChainSpecC(_FIRST[self.first], 0, int(self.s1), int(self.s2), int(self.s3))

    def rff_only(self) -> bool:
        return self.first == "RandomFourier" and self.s2 == 0 and self.s3 == 0


@dataclass
class SketchChain:
    """SketchChain (sketches.hpp:109-127): the realized stages; apply_rows runs on the device."""

    kernel: KernelSpec
    in_dim: int
    out_dim: int
    rff: Optional[RffMap] = None
    tensor: Optional[TensorSketchMap] = None
    srht: Optional[SrhtMap] = None
    gauss: Optional[GaussianMap] = None

    def input_dim(self) -> int:
        return self.in_dim

    def output_dim(self) -> int:
        return self.out_dim

    def _tables(self):
        """krr_chain_tables view (the arrays stay referenced by self while the call runs)."""
        t = _lib.ChainTablesC()
        if self.rff is not None:
            t.first, t.in_dim, t.s1 = 0, self.rff.w.shape[1], self.rff.w.shape[0]
            t.rff_w, t.rff_b = _lib.ptr(self.rff.w), _lib.ptr(self.rff.b)
        else:
            ts = self.tensor
            ts.hash = np.ascontiguousarray(ts.hash, dtype=np.uint32)
            ts.sign = _lib.f64(ts.sign)
            t.first, t.degree, t.in_dim, t.s1 = 1, ts.degree, ts.in_dim, ts.out_dim
            t.ts_hash, t.ts_sign = _lib.ptr(ts.hash), _lib.ptr(ts.sign)
        if self.srht is not None:
            self.srht.sign = _lib.f64(self.srht.sign)
            self.srht.rows = np.ascontiguousarray(self.srht.rows, dtype=np.int64)
            t.s2, t.srht_sign, t.srht_rows = len(self.srht.rows), _lib.ptr(self.srht.sign), _lib.ptr(self.srht.rows)
        if self.gauss is not None:
            self.gauss.proj = _lib.f64(self.gauss.proj)
            t.s3, t.gauss_proj = self.gauss.proj.shape[0], _lib.ptr(self.gauss.proj)
        return t

    def apply_rows(self, x: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
        """SketchChain::apply_rows (sketches.cpp:207-211) on the device."""
        x = _lib.f64(x)
        if x.ndim != 2 or x.shape[1] != self.in_dim:
            raise DimensionMismatch("SketchChain: input dimension mismatch")
        if x.shape[0] == 0:
            return np.zeros((0, self.out_dim))
        own = ctx is None
        ctx = ctx or Context()
        try:
            _set_data(ctx, x, self.kernel)
            z = np.empty((x.shape[0], self.out_dim))
            t = self._tables()
            _lib.check(_lib.LIB.krr_chain_apply(ctx.handle, C.byref(t), _lib.ptr(x), x.shape[0], _lib.ptr(z)))
            return z
        finally:
            if own:
                ctx.close()

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = _lib.f64(x)
        if x.ndim != 1 or x.shape[0] != self.in_dim:
            raise DimensionMismatch("SketchChain: input dimension mismatch")
        return self.apply_rows(x[None, :])[0]


def _stage_seed(master: int, stage: int) -> int:
    return (int(master) + (stage + 1) * K_STAGE_SEED_STRIDE) % (1 << 64)


def realize_chain(spec: ChainSpec, kernel: KernelSpec, input_dim: int, master_seed: int) -> SketchChain:
    """realize_chain (sketches.cpp:213-242): stage k drawn with stage_seed(master, k)."""
    spec.validate()
    kernel.validate()
    if spec.first == "RandomFourier" and kernel.family != "gaussian":
        raise InvalidArgument("realize_chain: random Fourier features serve the Gaussian kernel")
    if spec.first == "TensorSketch" and kernel.family != "polynomial":
        raise InvalidArgument("realize_chain: TensorSketch serves the polynomial kernel")
    chain = SketchChain(kernel, int(input_dim), spec.output_dim())
    if spec.first == "RandomFourier":
        chain.rff = RffMap(input_dim, spec.s1, kernel.sigma, _stage_seed(master_seed, 0))
    else:
        chain.tensor = TensorSketchMap(input_dim + 1, spec.s1, kernel.degree, _stage_seed(master_seed, 0))
    prev = spec.s1
    if spec.s2 > 0:
        chain.srht = SrhtMap(prev, spec.s2, _stage_seed(master_seed, 1))
        prev = spec.s2
    if spec.s3 > 0:
        chain.gauss = GaussianMap(prev, spec.s3, _stage_seed(master_seed, 2))
    return chain


# ----------------------------------------------------------------------------- precond.hpp
class Preconditioner:
    """Woodbury (Z Z^T + lambda_p I)^-1 = (I - U^T U)/lambda_p, U = L^-1 Z^T s x n, resident
    on the device (precond.hpp:15-23)."""

    def __init__(self, ctx: Context, n: int, s: int, lambda_p: float, jitter_used: bool, owns: bool):
        self._ctx, self._n, self._s = ctx, n, s
        self.lambda_p = float(lambda_p)
        self.jitter_used = bool(jitter_used)
        self._owns = owns

    def sketch_size(self) -> int:
        return self._s

    def dim(self) -> int:
        return self._n

    @property
    def u(self) -> np.ndarray:
        out = np.empty((self._s, self._n))
        _lib.check(_lib.LIB.krr_precond_download_u(self._ctx.handle, _lib.ptr(out)))
        return out

    def apply_columns(self, x: np.ndarray) -> np.ndarray:
        x = _lib.f64(x)
        if x.ndim != 2 or x.shape[0] != self._n:
            raise DimensionMismatch("Preconditioner: dimension mismatch")
        out = np.empty_like(x)
        _lib.check(_lib.LIB.krr_precond_apply(self._ctx.handle, _lib.ptr(x), x.shape[1], _lib.ptr(out)))
        return out

    def apply(self, x: np.ndarray) -> np.ndarray:
        x = _lib.f64(x)
        if x.ndim != 1 or x.shape[0] != self._n:
            raise DimensionMismatch("Preconditioner: dimension mismatch")
        return self.apply_columns(x[:, None])[:, 0]

    __call__ = apply

    def close(self):
        if self._owns:
            self._ctx.close()


def build_preconditioner(z: np.ndarray, lambda_p: float, ctx: Optional[Context] = None) -> Preconditioner:
    """precond.cpp:20-40 on the device (SYRK, Cholesky with one jitter retry, TRSM)."""
    if not (lambda_p > 0.0):
        raise NonPositiveLambda("build_preconditioner: lambda_p must be positive")
    z = _lib.f64(z)
    if z.ndim != 2:
        raise DimensionMismatch("build_preconditioner: Z must be a matrix")
    own = ctx is None
    ctx = ctx or Context()
    try:
        _lib.check(_lib.LIB.krr_sketch_upload(ctx.handle, _lib.ptr(z), z.shape[0], z.shape[1]))
        jit = C.c_int(0)
        _lib.check(_lib.LIB.krr_precond_build(ctx.handle, float(lambda_p), C.byref(jit)))
    except Exception:
        if own:
            ctx.close()
        raise
    return Preconditioner(ctx, z.shape[0], z.shape[1], lambda_p, bool(jit.value), own)


# ----------------------------------------------------------------------------- operator
class GaussianOperator:
    """v -> (K + lambda I) v with K never stored: the fused sm_100a K1 kernel (Gaussian, or
    the polynomial kernel of SURVEY 8f4 — see KernelOperator).  Callable like the
    reference's LinearOperator (solver.hpp:15)."""

    def __init__(self, x: np.ndarray, kernel: KernelSpec, lambda_: float = 0.0,
                 ctx: Optional[Context] = None):
        kernel.validate()
        x = _lib.f64(x)
        if x.ndim != 2 or x.shape[0] < 1:
            raise DimensionMismatch("GaussianOperator: x must be a non-empty n x d matrix")
        self._own = ctx is None
        self.ctx = ctx or Context()
        self.n, self.d = x.shape
        self.lambda_ = float(lambda_)
        self.kernel = kernel
        _set_data(self.ctx, x, kernel)

    def matmat(self, v: np.ndarray) -> np.ndarray:
        v = _lib.f64(v)
        if v.ndim != 2 or v.shape[0] != self.n:
            raise DimensionMismatch("GaussianOperator: dimension mismatch")
        out = np.empty_like(v)
        _lib.check(_lib.LIB.krr_kernel_matvec(self.ctx.handle, self.lambda_, _lib.ptr(v), v.shape[1],
                                              _lib.ptr(out)))
        return out

    def __call__(self, v: np.ndarray) -> np.ndarray:
        v = _lib.f64(v)
        if v.ndim != 1:
            raise DimensionMismatch("GaussianOperator: expected a vector")
        return self.matmat(v[:, None])[:, 0]

    def close(self):
        if self._own:
            self.ctx.close()


KernelOperator = GaussianOperator  # either kernel family


# ----------------------------------------------------------------------------- solver.hpp
@dataclass
class SolverConfig:
    """solver.hpp:17-27 (`lambda` is spelled `lambda_`)."""

    tau: float = 1e-5
    max_iter: int = 1000
    lambda_: float = 1e-2
    lambda_p: Optional[float] = None
    chain: ChainSpec = field(default_factory=ChainSpec)
    adaptive: bool = False
    s0: int = 0
    s_max: int = 0
    seed: int = 0


@dataclass
class RhsStats:
    iterations: int = 0
    final_residual: float = 0.0
    converged: bool = False
    residual_history: list = field(default_factory=list)


@dataclass
class PcgReport:
    per_rhs: list = field(default_factory=list)
    total_matvecs: int = 0
    wall_time_sec: float = 0.0
    phase_ms: dict = field(default_factory=dict)

    def all_converged(self) -> bool:
        return all(s.converged for s in self.per_rhs)

    def max_iterations(self) -> int:
        return max((s.iterations for s in self.per_rhs), default=0)


@dataclass
class PcgResult:
    solution: np.ndarray
    stats: RhsStats


@dataclass
class KrrModel:
    kernel: KernelSpec
    x: np.ndarray
    c: np.ndarray
    label_map: list = field(default_factory=list)
    lambda_: float = 0.0
    seed: int = 0

    def classification(self) -> bool:
        return len(self.label_map) > 0


@dataclass
class TrainResult:
    model: KrrModel
    report: PcgReport
    sketch_size: int = 0
    quality_passed: bool = True
    quality_history: list = field(default_factory=list)


def _stats_from(c_stats, hist: Optional[np.ndarray], j: int) -> RhsStats:
    s = c_stats[j]
    h = [] if hist is None else [float(v) for v in hist[j, : s.iterations]]
    return RhsStats(int(s.iterations), float(s.final_residual), bool(s.converged), h)


def pcg_solve(apply_a: Callable[[np.ndarray], np.ndarray],
              preconditioner: Optional[Callable[[np.ndarray], np.ndarray]],
              y: np.ndarray, tau: float, max_iter: int,
              observer: Optional[Callable[[int, np.ndarray], None]] = None,
              ctx: Optional[Context] = None) -> PcgResult:
    """solver.hpp:55-57 / solver.cpp:22-67.  The PCG vector algebra runs on the device;
    apply_a / preconditioner are caller operators (host callables), exactly as the
    reference's LinearOperator.  Throws BreakdownDetected when p'Ap <= 0."""
    y = _lib.f64(y)
    if y.ndim != 1:
        raise DimensionMismatch("pcg_solve: y must be a vector")
    n = y.shape[0]
    errors: list = []

    def wrap(fn):
        def cb(_user, inp, out, nn):
            try:
                v = np.ctypeslib.as_array(inp, shape=(nn,)).copy()
                r = np.asarray(fn(v), dtype=np.float64).reshape(-1)
                if r.shape[0] != nn:
                    raise DimensionMismatch("operator returned a vector of the wrong length")
                np.ctypeslib.as_array(out, shape=(nn,))[:] = r
                return 0
            except BaseException as e:  # noqa: BLE001 - propagated after the C call
                errors.append(e)
                return 1
        return _lib.OPERATOR_CB(cb)

    cb_a = wrap(apply_a)
    cb_m = wrap(preconditioner) if preconditioner is not None else _lib.OPERATOR_CB()

    def obs(_user, it, xptr, nn):
        try:
            observer(int(it), np.ctypeslib.as_array(xptr, shape=(nn,)).copy())
        except BaseException as e:  # noqa: BLE001
            errors.append(e)

    cb_o = _lib.OBSERVER_CB(obs) if observer is not None else _lib.OBSERVER_CB()
    x = np.zeros(n)
    st = (_lib.RhsStatsC * 1)()
    hist = np.zeros((1, max(1, int(max_iter))))
    own = ctx is None
    ctx = ctx or Context()
    try:
        status = _lib.LIB.krr_pcg_solve_operator(ctx.handle, n, cb_a, None, cb_m, None, _lib.ptr(y),
                                                 float(tau), int(max_iter), cb_o, None, _lib.ptr(x),
                                                 st, _lib.ptr(hist))
    finally:
        if own:
            ctx.close()
    if errors:
        raise errors[0]
    _lib.check(status)
    return PcgResult(x, _stats_from(st, hist, 0))


def solve_regularized(x: np.ndarray, kernel: KernelSpec, y: np.ndarray, lambda_: float,
                      preconditioner: Optional[Preconditioner], tau: float, max_iter: int,
                      ctx: Optional[Context] = None):
    """solver.cpp:69-94 with the Gaussian operator computed on the fly (the reference
    takes a dense K; here K is never stored).  `preconditioner` must have been built
    on the same context (pass ctx), or be None for plain CG."""
    kernel.validate()
    x = _lib.f64(x)
    y = _lib.f64(y)
    y2 = y[:, None] if y.ndim == 1 else y
    if x.ndim != 2 or y2.shape[0] != x.shape[0]:
        raise DimensionMismatch("solve_regularized: K and Y dimensions do not match")
    own = ctx is None
    if preconditioner is not None:
        ctx = preconditioner._ctx
        own = False
    ctx = ctx or Context()
    try:
        n, t = y2.shape
        _set_data(ctx, x, kernel)
        c = np.empty((n, t))
        st = (_lib.RhsStatsC * t)()
        hist = np.zeros((t, max(1, int(max_iter))))
        tot = C.c_int64()
        t0 = time.perf_counter()
        _lib.check(_lib.LIB.krr_pcg_solve(ctx.handle, float(lambda_), _lib.ptr(_lib.f64(y2)), t,
                                          float(tau), int(max_iter),
                                          1 if preconditioner is not None else 0, _lib.ptr(c), st,
                                          _lib.ptr(hist), C.byref(tot)))
        wall = time.perf_counter() - t0
    finally:
        if own:
            ctx.close()
    report = PcgReport([_stats_from(st, hist, j) for j in range(t)], int(tot.value), wall)
    return c, report


def solve_regularized_dense(k: np.ndarray, y: np.ndarray, lambda_: float, preconditioner: Optional[Preconditioner],
                            tau: float, max_iter: int, ctx: Optional[Context] = None):
    """solve_regularized (solver.hpp:82-84, solver.cpp:69-94) with the reference's own signature:
    a dense K (the on-the-fly `solve_regularized(x, kernel, ...)` is the scalable form).  The
    preconditioner, if given, must have been built on the same context (pass its ctx)."""
    k = _lib.f64(k)
    y = _lib.f64(y)
    y2 = y[:, None] if y.ndim == 1 else y
    if k.ndim != 2 or k.shape[0] != k.shape[1] or y2.shape[0] != k.shape[0]:
        raise DimensionMismatch("solve_regularized: K and Y dimensions do not match")
    own = ctx is None
    if preconditioner is not None:
        ctx = preconditioner._ctx
        own = False
    ctx = ctx or Context()
    try:
        n, t = y2.shape
        c = np.empty((n, t))
        st = (_lib.RhsStatsC * t)()
        hist = np.zeros((t, max(1, int(max_iter))))
        tot = C.c_int64()
        t0 = time.perf_counter()
        _lib.check(_lib.LIB.krr_solve_regularized_dense(ctx.handle, _lib.ptr(k), n, _lib.ptr(y2), t, float(lambda_),
                                                        1 if preconditioner is not None else 0, float(tau),
                                                        int(max_iter), _lib.ptr(c), st, _lib.ptr(hist),
                                                        C.byref(tot)))
        wall = time.perf_counter() - t0
    finally:
        if own:
            ctx.close()
    return c, PcgReport([_stats_from(st, hist, j) for j in range(t)], int(tot.value), wall)


def train(data: Dataset, kernel: KernelSpec, cfg: SolverConfig, ctx: Optional[Context] = None) -> TrainResult:
    """solver.cpp:96-133 — the whole hot path on the device (RFF chain for the Gaussian kernel,
    TensorSketch chains for the polynomial kernel, optional SRHT / Gaussian stages)."""
    if data.n() < 1:
        raise InvalidArgument("train: dataset is empty")
    if not (cfg.lambda_ > 0.0):
        raise NonPositiveLambda("train: lambda must be positive")
    if cfg.adaptive:
        return _train_adaptive(data, kernel, cfg, ctx)
    kernel.validate()
    cfg.chain.validate()
    x = _lib.f64(data.x)
    y = _lib.f64(data.y)
    y2 = y[:, None] if y.ndim == 1 else y
    n, d = x.shape
    t = y2.shape[1]
    s = cfg.chain.output_dim()
    c = np.empty((n, t))
    st = (_lib.RhsStatsC * t)()
    hist = np.zeros((t, max(1, int(cfg.max_iter))))
    tot = C.c_int64()
    phase = np.zeros(4)
    lp = cfg.lambda_p if cfg.lambda_p is not None else -1.0
    own = ctx is None
    ctx = ctx or Context()
    try:
        t0 = time.perf_counter()
        if kernel.family == "gaussian" and cfg.chain.rff_only():
            _lib.check(_lib.LIB.krr_train(ctx.handle, _lib.ptr(x), n, d, _lib.ptr(_lib.f64(y2)), t,
                                          kernel.sigma, float(cfg.lambda_), float(lp), s, int(cfg.seed),
                                          float(cfg.tau), int(cfg.max_iter), _lib.ptr(c), st,
                                          _lib.ptr(hist), C.byref(tot), _lib.ptr(phase)))
        else:  # any kernel family / sketch chain
            kc, cc = kernel._c(), cfg.chain._c()
            _lib.check(_lib.LIB.krr_train_ex(ctx.handle, _lib.ptr(x), n, d, _lib.ptr(_lib.f64(y2)), t,
                                             C.byref(kc), C.byref(cc), float(cfg.lambda_), float(lp),
                                             int(cfg.seed) % (1 << 64), float(cfg.tau), int(cfg.max_iter),
                                             _lib.ptr(c), st, _lib.ptr(hist), C.byref(tot), _lib.ptr(phase)))
        wall = time.perf_counter() - t0
    finally:
        if own:
            ctx.close()
    report = PcgReport([_stats_from(st, hist, j) for j in range(t)], int(tot.value), wall,
                       {"sketch_build": phase[0], "rff_build": phase[0], "precond_build": phase[1], "solve": phase[2],
                        "total": phase[3]})
    model = KrrModel(kernel, x.copy(), c, list(data.label_map), float(cfg.lambda_), int(cfg.seed))
    return TrainResult(model, report, s)


def _train_adaptive(data: Dataset, kernel: KernelSpec, cfg: SolverConfig, ctx: Optional[Context]) -> TrainResult:
    """solver.cpp:106-116: adaptive sketch size, then the same device PCG."""
    kernel.validate()
    cfg.chain.validate()
    x = _lib.f64(data.x)
    n = x.shape[0]
    s0 = cfg.s0 if cfg.s0 > 0 else default_initial_sketch_size(n)
    s_max = min(cfg.s_max, n) if cfg.s_max > 0 else max(n, s0)
    lp = cfg.lambda_p if cfg.lambda_p is not None else cfg.lambda_
    own = ctx is None
    ctx = ctx or Context()
    try:
        t0 = time.perf_counter()
        ad = adaptive_build(x, cfg.chain, kernel, cfg.lambda_, lp, min(s0, s_max), s_max, cfg.seed, ctx=ctx)
        c, rep = solve_regularized(x, kernel, data.y, cfg.lambda_, ad.preconditioner, cfg.tau, cfg.max_iter)
        rep.wall_time_sec = time.perf_counter() - t0
    finally:
        if own:
            ctx.close()
    model = KrrModel(kernel, x.copy(), c, list(data.label_map), float(cfg.lambda_), int(cfg.seed))
    return TrainResult(model, rep, ad.final_size, ad.passed, ad.history)


def predict_scores(model: KrrModel, xq: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
    """solver.cpp:135-139: cross_gram(Xq, X) C on the device (no diagonal forcing)."""
    xq = _lib.f64(xq)
    if xq.ndim != 2 or xq.shape[1] != model.x.shape[1]:
        raise DimensionMismatch("predict: query dimension does not match the model")
    c = _lib.f64(model.c)
    c2 = c[:, None] if c.ndim == 1 else c
    own = ctx is None
    ctx = ctx or Context()
    try:
        x = _lib.f64(model.x)
        _set_data(ctx, x, model.kernel)
        out = np.empty((xq.shape[0], c2.shape[1]))
        _lib.check(_lib.LIB.krr_predict_scores(ctx.handle, _lib.ptr(xq), xq.shape[0], _lib.ptr(c2),
                                               c2.shape[1], _lib.ptr(out)))
    finally:
        if own:
            ctx.close()
    return out


def rlsc_encode(class_indices, num_classes: int) -> np.ndarray:
    """solver.cpp:152-161."""
    cls = np.ascontiguousarray(class_indices, dtype=np.int32)
    y = np.empty((cls.shape[0], num_classes))
    _lib.check(_lib.LIB.krr_rlsc_encode(_lib.ptr(cls), cls.shape[0], int(num_classes), _lib.ptr(y)))
    return y


def rlsc_decode(scores: np.ndarray) -> list:
    """solver.cpp:163-173: row-wise argmax, ties to the lowest index (host bookkeeping)."""
    s = np.asarray(scores)
    return [int(np.argmax(row)) for row in s]  # np.argmax returns the first maximum


def predict_labels(model: KrrModel, xq: np.ndarray) -> list:
    if not model.classification():
        raise KrrError("predict_labels: model has no label map")
    scores = predict_scores(model, xq)
    if scores.shape[1] != len(model.label_map):
        raise KrrError("predict_labels: score width does not match the label map")
    return [model.label_map[i] for i in rlsc_decode(scores)]


# ----------------------------------------------------------------------------- f3: quality test / adaptive sizing
@dataclass
class QualityReport:
    """precond.hpp:35-47."""
    passed: bool = False
    cond1_value: float = 0.0
    cond2_ratio_low: float = 1.0
    cond2_ratio_high: float = 1.0
    rank_of_p: int = 0
    sketch_size: int = 0
    lambda_: float = 0.0
    cond1_threshold: float = 0.0
    spectrum_cut: float = 0.0
    ratio_low_threshold: float = 0.9
    ratio_high_threshold: float = 1.1


def _qr(r) -> QualityReport:
    return QualityReport(bool(r.passed), r.cond1_value, r.cond2_ratio_low, r.cond2_ratio_high, int(r.rank_of_p),
                         int(r.sketch_size), r.lambda_, r.cond1_threshold, r.spectrum_cut, r.ratio_low_threshold,
                         r.ratio_high_threshold)


def default_initial_sketch_size(n: int) -> int:
    """precond.cpp:102-104."""
    return max(64, (int(n) + 63) // 64)


def quality_test(x: np.ndarray, kernel: KernelSpec, z: np.ndarray, lambda_: float,
                 ctx: Optional[Context] = None) -> QualityReport:
    """quality_test (precond.cpp:60-100) with K the Gaussian kernel of X (never stored):
    eig(Z'Z), power iteration on (I-P)K(I-P) through the fused K1, B'KB through K1T."""
    kernel.validate()
    x = _lib.f64(x)
    z = _lib.f64(z)
    if z.ndim != 2 or z.shape[0] != x.shape[0]:
        raise DimensionMismatch("quality_test: K and Z dimensions do not match")
    if not (lambda_ > 0.0):
        raise NonPositiveLambda("quality_test: lambda must be positive")
    own = ctx is None
    ctx = ctx or Context()
    try:
        _set_data(ctx, x, kernel)
        _lib.check(_lib.LIB.krr_sketch_upload(ctx.handle, _lib.ptr(z), z.shape[0], z.shape[1]))
        r = _lib.QualityReportC()
        _lib.check(_lib.LIB.krr_quality_test(ctx.handle, float(lambda_), C.byref(r)))
    finally:
        if own:
            ctx.close()
    return _qr(r)


@dataclass
class AdaptiveResult:
    """precond.hpp AdaptiveResult (the sketch itself stays on the device)."""
    passed: bool
    preconditioner: "Preconditioner"
    final_size: int
    history: list


def adaptive_build(x: np.ndarray, chain_template: ChainSpec, kernel: KernelSpec, lambda_: float, lambda_p: float,
                   s0: int, s_max: int, master_seed: int, ctx: Optional[Context] = None) -> AdaptiveResult:
    """adaptive_build (precond.cpp:107-138): double s from s0 until quality_test passes or s_max,
    each attempt re-seeded with master + attempt * 0xD1B54A32D192ED03; the preconditioner from the
    final sketch stays resident on the device (pass ctx to keep using it)."""
    kernel.validate()
    chain_template.validate()
    if s0 < 1:
        raise InvalidArgument("adaptive_build: s0 must be at least 1")
    if s_max < s0:
        raise InvalidArgument("adaptive_build: s_max must be >= s0")
    x = _lib.f64(x)
    own = ctx is None
    ctx = ctx or Context()
    hist = (_lib.QualityReportC * 64)()
    nh, fs, ok, jit = C.c_int(), C.c_int64(), C.c_int(), C.c_int()
    try:
        _set_data(ctx, x, kernel)
        cc = chain_template._c()
        _lib.check(_lib.LIB.krr_adaptive_build_ex(ctx.handle, C.byref(cc), float(lambda_), float(lambda_p), int(s0),
                                                  int(s_max), int(master_seed) % (1 << 64), hist, 64, C.byref(nh),
                                                  C.byref(fs), C.byref(ok), C.byref(jit)))
    except BaseException:
        if own:
            ctx.close()
        raise
    pre = Preconditioner(ctx, x.shape[0], int(fs.value), float(lambda_p), bool(jit.value), own)
    return AdaptiveResult(bool(ok.value), pre, int(fs.value), [_qr(hist[i]) for i in range(min(nh.value, 64))])


# ----------------------------------------------------------------------------- f2: KRRM model file
def save_model(path, model: KrrModel) -> None:
    """io.cpp:192-215: the reference's KRRM file (byte-identical layout), written by the
    library's host code; readable by the reference's `krr predict` / `krr eval`."""
    x = _lib.f64(model.x)
    c = _lib.f64(model.c)
    c2 = c[:, None] if c.ndim == 1 else c
    lm = np.ascontiguousarray(model.label_map, dtype=np.float64)
    kc = model.kernel._c()
    _lib.check(_lib.LIB.krr_model_save_ex(str(path).encode(), C.byref(kc), float(model.lambda_),
                                          int(model.seed) % (1 << 64), _lib.ptr(lm) if lm.size else None, lm.size,
                                          _lib.ptr(x), x.shape[0], x.shape[1], _lib.ptr(c2), c2.shape[1]))


def load_model(path) -> KrrModel:
    """io.cpp:217-261 (same checks and messages; Gaussian and polynomial models)."""
    n, d, t, nl = C.c_int64(), C.c_int64(), C.c_int64(), C.c_int64()
    sigma, lam, seed = C.c_double(), C.c_double(), C.c_uint64()
    p = str(path).encode()
    _lib.check(_lib.LIB.krr_model_info(p, C.byref(n), C.byref(d), C.byref(t), C.byref(nl), C.byref(sigma),
                                       C.byref(lam), C.byref(seed)))
    lm = np.empty(max(1, nl.value))
    x = np.empty((n.value, d.value))
    c = np.empty((n.value, t.value))
    _lib.check(_lib.LIB.krr_model_load(p, _lib.ptr(lm), _lib.ptr(x), _lib.ptr(c)))
    kc = _lib.KernelSpecC()
    _lib.check(_lib.LIB.krr_model_kernel(p, C.byref(kc)))
    kernel = (KernelSpec.gaussian(kc.sigma) if kc.family == 0
              else KernelSpec.polynomial(kc.gamma, kc.offset, int(kc.degree)))
    return KrrModel(kernel, x, c, list(lm[:nl.value]), lam.value, int(seed.value))


# ----------------------------------------------------------------------------- f1: RF baseline
@dataclass
class RandomFeaturesModel:
    """solver.hpp RandomFeaturesModel: the realized sketch chain, weights w (s x t), lambda."""
    chain: SketchChain
    w: np.ndarray
    lambda_: float
    label_map: list = field(default_factory=list)

    def classification(self) -> bool:
        return len(self.label_map) > 0


def train_random_features_baseline(data: Dataset, kernel: KernelSpec, chain: ChainSpec, lambda_: float,
                                   seed: int = 0, ctx: Optional[Context] = None) -> RandomFeaturesModel:
    """Sketch-and-solve baseline of `krr bench` (solver.cpp:175-193): Z = chain(X),
    w = (Z^T Z + lambda I)^{-1} Z^T Y on the device (chain stages as SketchChain.apply_rows,
    cuBLAS SYRK/GEMM, cuSOLVER potrf/potrs; no jitter)."""
    kernel.validate()
    if not (lambda_ > 0.0):
        raise NonPositiveLambda("baseline: lambda must be positive")
    x = _lib.f64(data.x)
    y = _lib.f64(data.y)
    y2 = y[:, None] if y.ndim == 1 else y
    sk = realize_chain(chain, kernel, x.shape[1], seed)
    s, t = sk.output_dim(), y2.shape[1]
    own = ctx is None
    ctx = ctx or Context()
    try:
        _set_data(ctx, x, kernel)
        w = np.empty((s, t))
        tab = sk._tables()
        _lib.check(_lib.LIB.krr_rf_baseline_train_ex(ctx.handle, C.byref(tab), _lib.ptr(y2), t, float(lambda_),
                                                     _lib.ptr(w)))
    finally:
        if own:
            ctx.close()
    return RandomFeaturesModel(sk, w, float(lambda_), list(data.label_map))


def baseline_predict_scores(model: RandomFeaturesModel, xq: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
    """solver.cpp:195-197: chain(Xq) w."""
    xq = _lib.f64(xq)
    if xq.ndim != 2 or xq.shape[1] != model.chain.input_dim():
        raise DimensionMismatch("baseline predict: query dimension mismatch")
    s, t = model.w.shape
    own = ctx is None
    ctx = ctx or Context()
    try:
        # the context needs a data set for d / the kernel: the queries themselves
        _set_data(ctx, xq, model.chain.kernel)
        out = np.empty((xq.shape[0], t))
        tab = model.chain._tables()
        _lib.check(_lib.LIB.krr_rf_baseline_predict_ex(ctx.handle, C.byref(tab), _lib.ptr(xq), xq.shape[0],
                                                       _lib.ptr(_lib.f64(model.w)), t, _lib.ptr(out)))
    finally:
        if own:
            ctx.close()
    return out


def baseline_predict_labels(model: RandomFeaturesModel, xq: np.ndarray) -> list:
    if not model.classification():
        raise KrrError("baseline: model has no label map")
    return [model.label_map[i] for i in rlsc_decode(baseline_predict_scores(model, xq))]


# ----------------------------------------------------------------------------- synthetic data
def generate_config(cfg: int, n: int, d: int, t: int = 1, seed: int = 0):
    """BASELINE.json configs 1-5 generators, host C++ in the library."""
    x = np.empty((n, d))
    y = np.empty((n, t))
    _lib.check(_lib.LIB.krr_generate_config(int(cfg), n, d, t, int(seed), _lib.ptr(x), _lib.ptr(y)))
    return x, y


def schedule(n: int, world: int = 1, rank: int = 0):
    """Symmetric super-tile schedule of K1 (host only): (st, ns, tiles[(a, b)])."""
    st, ns, nt = C.c_int64(), C.c_int64(), C.c_int64()
    _lib.check(_lib.LIB.krr_schedule(n, world, rank, C.byref(st), C.byref(ns), None, 0, C.byref(nt)))
    tiles = np.empty((max(1, nt.value), 2), dtype=np.int32)
    _lib.check(_lib.LIB.krr_schedule(n, world, rank, C.byref(st), C.byref(ns), _lib.ptr(tiles),
                                     nt.value, C.byref(nt)))
    return int(st.value), int(ns.value), tiles[: nt.value].copy()


def shard_rows(n: int, world: int, rank: int):
    """Rows [begin, end) of the sketch owned by `rank` (host only)."""
    a, b = C.c_int64(), C.c_int64()
    _lib.check(_lib.LIB.krr_shard_rows(n, world, rank, C.byref(a), C.byref(b)))
    return int(a.value), int(b.value)


CONFIGS = {
    # cfg: (n, d, t, sigma, lambda, s)  -- BASELINE.json configs[0..4]
    1: (8192, 16, 1, 4.0, 1e-3, 1024),
    2: (65536, 54, 1, 3.0, 1e-4, 2048),
    3: (262144, 90, 1, 6.0, 1e-5, 4096),
    4: (1048576, 90, 1, 6.0, 1e-6, 8192),
    5: (524288, 440, 16, 20.0, 1e-5, 16384),
}
