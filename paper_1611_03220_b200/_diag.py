"""ctypes binding of libkrr_diag.so (include/krr_diag.h): micro-benchmarks, tcgen05 probes and
kernel clock traces used by bench.py's roofline bookkeeping, tools/ and tests/.  Measurement
tooling only; the drop-in library is libkrr_b200.so (_lib.py)."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _lib  # loads libkrr_b200.so first (libkrr_diag.so links against it)

LIB_PATH = Path(__file__).resolve().parent / "libkrr_diag.so"
if not LIB_PATH.exists():
    raise ImportError(f"{LIB_PATH} is missing: build it with python paper_1611_03220_b200/_build.py")
LIB = C.CDLL(str(LIB_PATH))

_vp, _i64, _d, _i = C.c_void_p, C.c_int64, C.c_double, C.c_int
_SIGS = {
    "krr_diag_microbench": [_i, _vp],
    "krr_diag_gauss_exp": [_i, _vp, _i64, _d, _i, _vp],
    "krr_diag_i8_gemm": [_i, _vp, _vp, _vp, _i, _i],
    "krr_diag_bf16_gemm": [_i, _vp, _vp, _vp, _i, _i],
    "krr_diag_i8_mma_rate": [_i, _i, _i, _i, _i, C.POINTER(_d)],
    "krr_diag_tmem_ld_rate": [_i, _i, _i, C.POINTER(_d)],
    "krr_diag_tmem_ld_under_mma": [_i, _i, _i, C.POINTER(_d), C.POINTER(_d)],
    "krr_diag_i8_trace": [_vp, _i],
    "krr_diag_i8x_trace": [_vp, _i],
    "krr_diag_i8t_trace": [_vp, _i],
}
for _name, _args in _SIGS.items():
    _f = getattr(LIB, _name)
    _f.argtypes = _args
    _f.restype = C.c_int
LIB.krr_diag_last_error.argtypes = []
LIB.krr_diag_last_error.restype = C.c_char_p


def check(status: int) -> None:
    if status != _lib.OK:
        raise _lib._EXC.get(status, _lib.KrrError)(LIB.krr_diag_last_error().decode(errors="replace"))


def declared_symbols() -> list[str]:
    return ["krr_diag_last_error"] + list(_SIGS)


def microbench(device: int = 0) -> np.ndarray:
    """[dmma_tflops, dfma_tflops, mixed, exp_libdevice_gevals, exp_table_gevals, sms, clock_mhz,
    split_tflops, imma_tops] measured live on `device`."""
    out = np.zeros(9)
    check(LIB.krr_diag_microbench(device, _lib.ptr(out)))
    return out


def i8_mma_rate(N: int, reps: int, kbytes: int, mode: int, device: int = 0) -> float:
    v = C.c_double()
    check(LIB.krr_diag_i8_mma_rate(device, N, reps, kbytes, mode, C.byref(v)))
    return v.value
