"""A/B timing of K1T variants at config-5 shape: python tools/ab_k1t.py [--n N] lib1.so ...
Each library in its own process (KRR_B200_LIB); device time of one (K + lambda I) V pass
(t = 16) via CUDA events around krr_kernel_matvec on device buffers is not exposed, so this
times the host call (H2D/D2H of n x 16 doubles included, identical across variants)."""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
CHILD = r"""
import sys, time, json, numpy as np
sys.path.insert(0, %(root)r)
import paper_1611_03220_b200 as krr
n, path, reps, d, dbg = %(n)d, %(path)d, %(reps)d, %(d)d, %(dbg)d
x = krr.generate_config(5, n, 440, 16, 0)[0] if d == 440 else np.random.default_rng(0).standard_normal((n, d))
v = np.random.default_rng(0).standard_normal((n, 16))
ctx = krr.Context(0)
ctx.set_option("k1t_path", path)
op = krr.KernelOperator(x, krr.KernelSpec.gaussian(20.0 if d == 440 else 6.0), 1e-5, ctx=ctx)
out = op.matmat(v)
if dbg:
    ctx.set_option("i8_debug", dbg)
ts = []
for _ in range(reps):
    t0 = time.perf_counter(); out = op.matmat(v); ts.append(time.perf_counter() - t0)
np.save(%(out)r, out)
print(json.dumps({"s": ts}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=131072)
    ap.add_argument("--path", default="1", help="comma list of k1t_path values, crossed with the libraries")
    ap.add_argument("--d", default="440", help="comma list of d values")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--debug", default="0", help="comma list of i8_debug profiling modes (results invalid)")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    import numpy as np
    ref = None
    runs = [(lib, int(dd), int(pp), int(g)) for dd in a.d.split(",") for lib in a.libs for pp in a.path.split(",")
            for g in a.debug.split(",")]
    for i, (lib, d, path, dbg) in enumerate(runs):
        if i and runs[i - 1][1] != d:
            ref = None
        out = f"/tmp/abk1t_{i}.npy"
        env = dict(os.environ, KRR_B200_LIB=str(Path(lib).resolve()))
        r = subprocess.run([sys.executable, "-c", CHILD % dict(root=str(ROOT), n=a.n, path=path, reps=a.reps, out=out, d=d, dbg=dbg)],
                           capture_output=True, text=True, env=env, timeout=900)
        if r.returncode:
            print(json.dumps({"lib": lib, "error": r.stderr[-600:]}), flush=True)
            continue
        s = json.loads(r.stdout.strip().splitlines()[-1])["s"]
        kv = np.load(out)
        ref = kv if ref is None else ref
        print(json.dumps({"lib": Path(lib).name, "n": a.n, "d": d, "k1t_path": path, "debug": dbg, "s": s, "best_s": min(s),
                          "rel_vs_first": float(np.linalg.norm(kv - ref) / np.linalg.norm(ref))}), flush=True)


if __name__ == "__main__":
    main()
