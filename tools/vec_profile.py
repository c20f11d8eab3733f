"""HBM-bound kernels of one PCG iteration (Woodbury apply K6, vector algebra K7): a small
train at BASELINE config-3 shape (n = 262144, s = 4096) for a few iterations, meant to run
under ncu with a kernel-name filter, e.g.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
      --clock-control none -k regex:'gemvT|reduce_rows|precond_z|dot_partial|pcg_update|sum_partials' \
      --csv --log-file gpurun_out/vec.csv python tools/vec_profile.py

Without ncu it prints the per-iteration time for reference.
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 262144
s = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
its = int(sys.argv[3]) if len(sys.argv) > 3 else 3
n_, d, t, sigma, lam, _ = krr.CONFIGS[3]
x, y = krr.generate_config(3, n, d, 1, 0)
ctx = krr.Context(0)
cfg = krr.SolverConfig(lambda_=lam, tau=1e-12, max_iter=its, chain=krr.ChainSpec(s1=s), seed=0)
t0 = time.perf_counter()
res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg, ctx=ctx)
print(json.dumps({"n": n, "s": s, "iterations": res.report.per_rhs[0].iterations,
                  "phase_ms": res.report.phase_ms, "wall_s": time.perf_counter() - t0}))
ctx.close()
