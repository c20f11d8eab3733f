"""Woodbury build split and the multi-column apply at a BASELINE shape: set data, RFF features
(K2), krr_precond_build (Z^T Z, Cholesky, U = L^-1 Z^T: CUDA-event split from
krr_get_option build_*_ms), then `reps` apply_columns of t = 16 columns (K6T) with host buffers.
Meant to run alone and under ncu with a kernel filter, e.g.

  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      -k regex:'k6t|syrk|trsm|chol|reduce' --csv --log-file gpurun_out/build.csv python tools/build_profile.py 5

  python tools/build_profile.py CFG [n] [reps]
"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 5
n_, d, t, sigma, lam, s = krr.CONFIGS[cfg]
n = int(sys.argv[2]) if len(sys.argv) > 2 else n_
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
x, y = krr.generate_config(cfg, n, d, t, 0)
ctx = krr.Context(0)
chain = krr.realize_chain(krr.ChainSpec(s1=s), krr.KernelSpec.gaussian(sigma), d, 0)
_lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, sigma))
t0 = time.perf_counter()
_lib.check(_lib.LIB.krr_rff_build(ctx.handle, _lib.ptr(chain.rff.w), _lib.ptr(chain.rff.b), s))
t_rff = time.perf_counter() - t0
jit = _lib.C.c_int(0)
t0 = time.perf_counter()
_lib.check(_lib.LIB.krr_precond_build(ctx.handle, lam, _lib.C.byref(jit)))
t_build = time.perf_counter() - t0
split = {k: ctx.get_option(f"build_{k}_ms") for k in ("gram", "cholesky", "trsm")}
r = np.random.default_rng(1).standard_normal((n, 16))
o = np.empty_like(r)
_lib.check(_lib.LIB.krr_precond_apply(ctx.handle, _lib.ptr(r), 16, _lib.ptr(o)))
t0 = time.perf_counter()
for _ in range(reps):
    _lib.check(_lib.LIB.krr_precond_apply(ctx.handle, _lib.ptr(r), 16, _lib.ptr(o)))
t_apply = (time.perf_counter() - t0) / reps
print(json.dumps({"cfg": cfg, "n": n, "d": d, "s": s, "rff_s": t_rff, "precond_build_s": t_build,
                  "build_split_ms": split, "jitter": jit.value, "apply16_host_s": t_apply,
                  "u_bytes": 8.0 * n * s,
                  "apply_sha1": __import__("hashlib").sha1(o.tobytes()).hexdigest()[:16]}))
ctx.close()
