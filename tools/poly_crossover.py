"""Polynomial-kernel K1 path crossover: DMMA vs K1-I8 (ms per K v, n = 65536, q = 3)."""
import ctypes as C
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402

n = 65536
ctx = krr.Context(0)
for d in [int(a) for a in sys.argv[1:]] or (8, 16, 24, 32, 40, 48, 64, 90):
    x = np.random.default_rng(d).standard_normal((n, d)) / np.sqrt(d)
    row = {"d": d}
    for path in (0, 1):
        ctx.set_option("k1_path", path)
        krr._set_data(ctx, x, krr.KernelSpec.polynomial(1.0, 1.0, 3))
        tot, k1 = C.c_double(), C.c_double()
        _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 0.0, 3, C.byref(tot), C.byref(k1)))
        row[["dmma_ms", "i8_ms"][path]] = tot.value / 3
    print(json.dumps(row), flush=True)
