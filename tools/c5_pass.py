"""One (K + lambda I) V pass at BASELINE config 5 (n = 524288, d = 440, t = 16: the K1T
multi-RHS kernel), timed end to end through krr_kernel_matvec (host buffers)."""
import json
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402

n, d, t, sigma, lam, s = krr.CONFIGS[5]
if len(sys.argv) > 1:
    n = int(sys.argv[1])
k1t = int(sys.argv[2]) if len(sys.argv) > 2 else -1  # K1T path: -1 auto, 0 DMMA, 1 K1T-I8
ctx = krr.Context(0)
ctx.set_option("k1t_path", k1t)
x, y = krr.generate_config(5, n, d, t, 0)
_lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, sigma))
v = np.ascontiguousarray(y)
out = np.empty_like(v)
_lib.check(_lib.LIB.krr_kernel_matvec(ctx.handle, lam, _lib.ptr(v), t, _lib.ptr(out)))  # warm
t0 = time.perf_counter()
_lib.check(_lib.LIB.krr_kernel_matvec(ctx.handle, lam, _lib.ptr(v), t, _lib.ptr(out)))
dt = time.perf_counter() - t0
print(json.dumps({"config": 5, "n": n, "d": d, "t": t, "k1t_path": ctx.get_option("k1t_path_effective"),
                  "seconds_per_pass": dt,
                  "gevals_per_s": float(n) * n / dt / 1e9, "rhs_gevals_per_s": float(n) * n * t / dt / 1e9,
                  "finite": bool(np.isfinite(out).all())}))
