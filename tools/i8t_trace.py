"""K1T-I8 per-tile timeline of CTA 0 (clock64 stamps; i8_debug bit 2), config-5 shape.

python tools/i8t_trace.py [n] [d]
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
d = int(sys.argv[2]) if len(sys.argv) > 2 else 440
x, _ = krr.generate_config(5, n, d, 16, 0) if d == 440 else (np.random.default_rng(0).standard_normal((n, d)), None)
v = np.random.default_rng(0).standard_normal((n, 16))
ctx = krr.Context(0)
ctx.set_option("k1t_path", 1)
op = krr.KernelOperator(x, krr.KernelSpec.gaussian(20.0 if d == 440 else 6.0), 0.0, ctx=ctx)
op.matmat(v)
ctx.set_option("i8_debug", 4)
op.matmat(v)
buf = np.zeros(32 * 16, dtype=np.int64)
_diag.check(_diag.LIB.krr_diag_i8t_trace(buf.ctypes.data_as(C.c_void_p), buf.size))
t = buf.reshape(32, 16)
names = ["start", "st6", "drained", "exp", "barA", "dmmaR", "dmmaC", "barB", "m:go", "m:ks0", "m:ksM", "m:ksL",
         "p:ks0", "p:efree", "-", "-"]
print("tile " + " ".join(f"{nm:>8s}" for nm in names))
for q in range(1, 31):
    row = t[q]
    print(f"{q:4d} " + " ".join(f"{(row[i] - t[q, 0]) if row[i] else 0:8d}" for i in range(16)),
          f" dt={t[q + 1, 0] - t[q, 0]}")
