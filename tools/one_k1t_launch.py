"""One K1T launch (multi-RHS, t = 16) at config-5 shape (d = 440) for ncu captures.

python tools/one_k1t_launch.py [n] [k1t_path: -1 auto, 0 DMMA K1T, 1 K1T-I8]
"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 65536
path = int(sys.argv[2]) if len(sys.argv) > 2 else -1
x, _ = krr.generate_config(5, n, 440, 16, 0)
v = np.random.default_rng(0).standard_normal((n, 16))
ctx = krr.Context(0)
ctx.set_option("k1t_path", path)
op = krr.KernelOperator(x, krr.KernelSpec.gaussian(20.0), 1e-5, ctx=ctx)
out = op.matmat(v)
print("ok", float(out[0, 0]))
