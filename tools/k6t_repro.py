"""Bisect helper for the K6T kernels: runs apply_columns for one (n, s, t) given on the command line."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_1611_03220_b200 as krr  # noqa: E402
from oracle import oracle_ffi as oracle  # noqa: E402

n, s, t = (int(a) for a in sys.argv[1:4])
z = oracle.random_matrix(n, s, 31) * 0.1
p = krr.build_preconditioner(z, 1e-2)
x = oracle.random_matrix(n, t, 32)
got = p.apply_columns(x)
u, _ = oracle.build_preconditioner(z, 1e-2)
want = oracle.precond_apply(u, 1e-2, x)
print(n, s, t, np.linalg.norm(got - want) / np.linalg.norm(want), flush=True)
