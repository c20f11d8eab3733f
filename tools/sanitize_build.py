"""Small Woodbury builds + applies checked against numpy (K3-I8 Gram, K4 Cholesky, K5 TRSM over
several column blocks with a ragged last block, K6 and K6T): a quick stand-alone check, and the
workload for compute-sanitizer where that tool is available (it is closed on this GPU pool).

  python tools/sanitize_build.py
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402

rng = np.random.default_rng(0)
for n, s, t in ((700, 300, 16), (257, 130, 8), (90, 33, 16)):
    z = rng.standard_normal((n, s)) * 0.1
    p = krr.build_preconditioner(z, 1e-2)
    x = rng.standard_normal((n, t))
    y = p.apply_columns(x)
    y1 = p.apply(x[:, 0].copy())
    g = z.T @ z + 1e-2 * np.eye(s)
    u = np.linalg.solve(np.linalg.cholesky(g), z.T)
    want = (x - u.T @ (u @ x)) / 1e-2
    print(n, s, t, float(np.abs(y - want).max() / np.abs(want).max()), float(np.abs(y1 - want[:, 0]).max()))
