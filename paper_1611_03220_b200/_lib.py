"""ctypes binding of libkrr_b200.so (the C-ABI in include/krr_b200.h).

The product path is the CUDA library; there is no Python/NumPy compute fallback.
If the shared library is missing, importing the binding raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

_HERE = Path(__file__).resolve().parent
LIB_PATH = Path(os.environ.get("KRR_B200_LIB", _HERE / "libkrr_b200.so"))

# Status codes (include/krr_b200.h)
OK = 0
ERR_DIMENSION_MISMATCH = 1
ERR_NOT_POSITIVE_DEFINITE = 2
ERR_SINGULAR_TRIANGULAR = 3
ERR_BREAKDOWN = 4
ERR_NON_POSITIVE_LAMBDA = 5
ERR_INVALID_ARGUMENT = 6
ERR_CUDA = 7
ERR_NCCL = 8
ERR_STATE = 9
ERR_CALLBACK = 10
ERR_IO = 11
ERR_NO_CONVERGENCE = 12


class KrrError(Exception):
    """Base of every error raised through the C-ABI."""


# Exception types mirror reference types.hpp:18-64 (invalid_argument-derived ones
# also derive from ValueError, runtime_error-derived ones from RuntimeError).
class DimensionMismatch(KrrError, ValueError):
    pass


class NotPositiveDefinite(KrrError, RuntimeError):
    pass


class SingularTriangular(KrrError, RuntimeError):
    pass


class BreakdownDetected(KrrError, RuntimeError):
    pass


class NonPositiveLambda(KrrError, ValueError):
    pass


class InvalidArgument(KrrError, ValueError):
    pass


class CudaError(KrrError, RuntimeError):
    pass


class NcclError(KrrError, RuntimeError):
    pass


class StateError(KrrError, RuntimeError):
    pass


class CallbackError(KrrError, RuntimeError):
    pass


class NoConvergence(KrrError, RuntimeError):
    """types.hpp:34 (symmetric_eigen's eigensolver did not converge)."""


class ModelFileError(KrrError, RuntimeError):
    """io.cpp model file errors (std::runtime_error in the reference)."""


_EXC = {
    ERR_DIMENSION_MISMATCH: DimensionMismatch,
    ERR_NOT_POSITIVE_DEFINITE: NotPositiveDefinite,
    ERR_SINGULAR_TRIANGULAR: SingularTriangular,
    ERR_BREAKDOWN: BreakdownDetected,
    ERR_NON_POSITIVE_LAMBDA: NonPositiveLambda,
    ERR_INVALID_ARGUMENT: InvalidArgument,
    ERR_CUDA: CudaError,
    ERR_NCCL: NcclError,
    ERR_STATE: StateError,
    ERR_CALLBACK: CallbackError,
    ERR_IO: ModelFileError,
    ERR_NO_CONVERGENCE: NoConvergence,
}


class QualityReportC(C.Structure):
    _fields_ = [("passed", C.c_int32), ("pad_", C.c_int32), ("cond1_value", C.c_double),
                ("cond2_ratio_low", C.c_double), ("cond2_ratio_high", C.c_double), ("rank_of_p", C.c_int64),
                ("sketch_size", C.c_int64), ("lambda_", C.c_double), ("cond1_threshold", C.c_double),
                ("spectrum_cut", C.c_double), ("ratio_low_threshold", C.c_double),
                ("ratio_high_threshold", C.c_double)]


class RhsStatsC(C.Structure):
    _fields_ = [("iterations", C.c_int32), ("converged", C.c_int32), ("final_residual", C.c_double)]


class KernelSpecC(C.Structure):
    _fields_ = [("family", C.c_int32), ("degree", C.c_int32), ("sigma", C.c_double), ("gamma", C.c_double),
                ("offset", C.c_double)]


class ChainSpecC(C.Structure):
    _fields_ = [("first", C.c_int32), ("pad_", C.c_int32), ("s1", C.c_int64), ("s2", C.c_int64),
                ("s3", C.c_int64)]


class ChainTablesC(C.Structure):
    _fields_ = [("first", C.c_int32), ("degree", C.c_int32), ("in_dim", C.c_int64), ("s1", C.c_int64),
                ("s2", C.c_int64), ("s3", C.c_int64), ("rff_w", C.c_void_p), ("rff_b", C.c_void_p),
                ("ts_hash", C.c_void_p), ("ts_sign", C.c_void_p), ("srht_sign", C.c_void_p),
                ("srht_rows", C.c_void_p), ("gauss_proj", C.c_void_p)]


OPERATOR_CB = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int64)
OBSERVER_CB = C.CFUNCTYPE(None, C.c_void_p, C.c_int, C.POINTER(C.c_double), C.c_int64)

_vp = C.c_void_p
_i64 = C.c_int64
_d = C.c_double
_i = C.c_int

# name -> argtypes (restype int unless stated)
_SIGS = {
    "krr_abi_version": [],
    "krr_device_count": [],
    "krr_ctx_create": [_i, C.POINTER(_vp)],
    "krr_nccl_unique_id": [_vp],
    "krr_ctx_create_dist": [_i, _i, _i, _vp, C.POINTER(_vp)],
    "krr_ctx_destroy": [_vp],
    "krr_ctx_launch_count": [_vp, C.POINTER(_i64)],
    "krr_set_option": [_vp, C.c_char_p, _d],
    "krr_get_option": [_vp, C.c_char_p, C.POINTER(_d)],
    "krr_set_precision": [_vp, _i],
    "krr_quality_test": [_vp, _d, C.POINTER(QualityReportC)],
    "krr_adaptive_build": [_vp, _d, _d, _i64, _i64, C.c_uint64, _vp, _i, C.POINTER(_i), C.POINTER(_i64),
                           C.POINTER(_i), C.POINTER(_i)],
    "krr_model_save": [C.c_char_p, _d, _d, C.c_uint64, _vp, _i64, _vp, _i64, _i64, _vp, _i64],
    "krr_model_info": [C.c_char_p, C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64), C.POINTER(_i64),
                       C.POINTER(_d), C.POINTER(_d), C.POINTER(C.c_uint64)],
    "krr_model_load": [C.c_char_p, _vp, _vp, _vp],
    "krr_rf_baseline_train": [_vp, _vp, _vp, _i64, _vp, _i64, _d, _vp],
    "krr_rf_baseline_predict": [_vp, _vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp],
    "krr_set_data": [_vp, _vp, _i64, _i64, _d],
    "krr_kernel_matvec": [_vp, _d, _vp, _i64, _vp],
    "krr_kernel_matvec_device": [_vp, _d, _vp, _i64, _vp],
    "krr_predict_scores": [_vp, _vp, _i64, _vp, _i64, _vp],
    "krr_rff_realize": [C.c_uint64, _i64, _i64, _d, _vp, _vp],
    "krr_rff_build": [_vp, _vp, _vp, _i64],
    "krr_rff_download": [_vp, _vp],
    "krr_sketch_upload": [_vp, _vp, _i64, _i64],
    "krr_precond_build": [_vp, _d, C.POINTER(_i)],
    "krr_precond_apply": [_vp, _vp, _i64, _vp],
    "krr_precond_download_u": [_vp, _vp],
    "krr_precond_read_u": [_vp, _i64, _i64, _vp, _i64, _vp],
    "krr_precond_drop": [_vp],
    "krr_pcg_solve": [_vp, _d, _vp, _i64, _d, _i, _i, _vp, _vp, _vp, C.POINTER(_i64)],
    "krr_pcg_solve_operator": [_vp, _i64, OPERATOR_CB, _vp, OPERATOR_CB, _vp, _vp, _d, _i,
                               OBSERVER_CB, _vp, _vp, _vp, _vp],
    "krr_train": [_vp, _vp, _i64, _i64, _vp, _i64, _d, _d, _d, _i64, C.c_uint64, _d, _i, _vp,
                  _vp, _vp, C.POINTER(_i64), _vp],
    "krr_schedule": [_i64, _i, _i, C.POINTER(_i64), C.POINTER(_i64), _vp, _i64, C.POINTER(_i64)],
    "krr_shard_rows": [_i64, _i, _i, C.POINTER(_i64), C.POINTER(_i64)],
    "krr_generate_config": [_i, _i64, _i64, _i64, C.c_uint64, _vp, _vp],
    "krr_rlsc_encode": [_vp, _i64, C.c_int32, _vp],
    "krr_bench_matvec": [_vp, _d, _i, C.POINTER(_d), C.POINTER(_d)],
    "krr_solve_regularized_dense": [_vp, _vp, _i64, _vp, _i64, _d, _i, _d, _i, _vp, _vp, _vp, C.POINTER(_i64)],
    # SURVEY 8f4
    "krr_set_data_kernel": [_vp, _vp, _i64, _i64, C.POINTER(KernelSpecC)],
    "krr_tensorsketch_realize": [C.c_uint64, _i64, _i64, _i, _vp, _vp],
    "krr_srht_realize": [C.c_uint64, _i64, _i64, _vp, _vp],
    "krr_gaussmap_realize": [C.c_uint64, _i64, _i64, _vp],
    "krr_chain_apply": [_vp, C.POINTER(ChainTablesC), _vp, _i64, _vp],
    "krr_chain_build": [_vp, C.POINTER(ChainTablesC)],
    "krr_chain_build_seeded": [_vp, C.POINTER(ChainSpecC), C.c_uint64],
    "krr_chain_scaled_to": [C.POINTER(ChainSpecC), _i64, C.POINTER(ChainSpecC)],
    "krr_train_ex": [_vp, _vp, _i64, _i64, _vp, _i64, C.POINTER(KernelSpecC), C.POINTER(ChainSpecC), _d, _d,
                     C.c_uint64, _d, _i, _vp, _vp, _vp, C.POINTER(_i64), _vp],
    "krr_adaptive_build_ex": [_vp, C.POINTER(ChainSpecC), _d, _d, _i64, _i64, C.c_uint64, _vp, _i, C.POINTER(_i),
                              C.POINTER(_i64), C.POINTER(_i), C.POINTER(_i)],
    "krr_rf_baseline_train_ex": [_vp, C.POINTER(ChainTablesC), _vp, _i64, _d, _vp],
    "krr_rf_baseline_predict_ex": [_vp, C.POINTER(ChainTablesC), _vp, _i64, _vp, _i64, _vp],
    "krr_model_save_ex": [C.c_char_p, C.POINTER(KernelSpecC), _d, C.c_uint64, _vp, _i64, _vp, _i64, _i64, _vp,
                          _i64],
    "krr_model_kernel": [C.c_char_p, C.POINTER(KernelSpecC)],
}


def _load() -> C.CDLL:
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python paper_1611_03220_b200/_build.py` "
            "(there is no CPU fallback)")
    lib = C.CDLL(str(LIB_PATH))
    lib.krr_last_error.restype = C.c_char_p
    lib.krr_last_error.argtypes = []
    for name, args in _SIGS.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = C.c_int
    return lib


LIB = _load()


def declared_symbols() -> list[str]:
    return ["krr_last_error"] + list(_SIGS)


def check(status: int) -> None:
    if status != OK:
        msg = LIB.krr_last_error().decode(errors="replace")
        raise _EXC.get(status, KrrError)(msg)


def ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def f64(a, shape=None) -> np.ndarray:
    """Contiguous row-major float64 view/copy (reference Matrix is RowMajor fp64)."""
    out = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        out = out.reshape(shape)
    return out


def device_count() -> int:
    return int(LIB.krr_device_count())


class Context:
    """One device context (one GPU, one stream; NCCL comm when world > 1)."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_id: bytes | None = None):
        h = C.c_void_p()
        if world > 1 or nccl_id is not None:  # world 1 + id: a one-rank NCCL communicator
            if nccl_id is None or len(nccl_id) != 128:
                raise InvalidArgument("a 128-byte NCCL unique id is required when world > 1")
            buf = C.create_string_buffer(nccl_id, 128)
            check(LIB.krr_ctx_create_dist(device, rank, world, buf, C.byref(h)))
        else:
            check(LIB.krr_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device, self.rank, self.world = device, rank, world

    def close(self) -> None:
        if getattr(self, "handle", None) and self.handle.value:
            LIB.krr_ctx_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):  # pragma: no cover - interpreter shutdown order
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_option(self, key: str, value: float) -> None:
        check(LIB.krr_set_option(self.handle, key.encode(), float(value)))

    def set_precision(self, bits: int) -> None:
        """64: fp64 oracle-matching K v (default); 32: the optional fp32-accuracy mode."""
        check(LIB.krr_set_precision(self.handle, int(bits)))

    def get_option(self, key: str) -> float:
        out = C.c_double()
        check(LIB.krr_get_option(self.handle, key.encode(), C.byref(out)))
        return out.value

    def read_u(self, row0: int, nrows: int, cols) -> np.ndarray:
        """U[row0:row0+nrows, cols] of the context's preconditioner (krr_precond_read_u)."""
        cols = np.ascontiguousarray(cols, dtype=np.int64)
        out = np.empty((nrows, cols.size))
        check(LIB.krr_precond_read_u(self.handle, row0, nrows, ptr(cols), cols.size, ptr(out)))
        return out

    def precond_drop(self) -> None:
        """Free the context's sketch / preconditioner buffers (krr_precond_drop)."""
        check(LIB.krr_precond_drop(self.handle))

    @property
    def launches(self) -> int:
        v = C.c_int64()
        check(LIB.krr_ctx_launch_count(self.handle, C.byref(v)))
        return int(v.value)


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    check(LIB.krr_nccl_unique_id(buf))
    return buf.raw
