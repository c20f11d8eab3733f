"""K1-I8 per-tile timeline of CTA 0 (clock64 stamps; i8_debug bit 2).

python tools/i8_trace.py [n] [d] [extra debug bits] [poly]
"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib
from paper_1611_03220_b200 import _diag  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
d = int(sys.argv[2]) if len(sys.argv) > 2 else 90
extra = int(sys.argv[3]) if len(sys.argv) > 3 else 0
poly = len(sys.argv) > 4 and sys.argv[4] == "poly"
ctx = krr.Context(0)
x = np.random.default_rng(0).standard_normal((n, d))
if poly:  # the polynomial kernel's epilogue (no exp) on the same K1-I8 skeleton
    krr._set_data(ctx, x, krr.KernelSpec.polynomial(1.0 / d, 1.0, 3))
else:
    _lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, 6.0))
ctx.set_option("k1_path", 1)
tot, k1 = C.c_double(), C.c_double()
_lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))
ctx.set_option("i8_debug", 4 | extra)
_lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))
buf = np.zeros(64 * 16, dtype=np.int64)
_diag.check(_diag.LIB.krr_diag_i8_trace(buf.ctypes.data_as(C.c_void_p), buf.size))
t = buf.reshape(64, 16)
t0 = t[0, 0]
names = ["start", "st65", "st43", "st21", "st0", "cd", "exp", "bar", "m:epiw", "m:bfull", "m:g6", "m:g4", "m:g0",
         "elem", "colsum", "g0done"]
print("tile " + " ".join(f"{nm:>8s}" for nm in names))
for q in range(1, 40):
    row = t[q]
    print(f"{q:4d} " + " ".join(f"{(row[i] - t[q, 0]):8d}" for i in range(16)), f" dt={t[q + 1, 0] - t[q, 0]}")
