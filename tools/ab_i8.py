"""A/B timing of K1 variants: python tools/ab_i8.py [--n N --d D --reps R] lib1.so lib2.so ...

Each library runs in its own process (KRR_B200_LIB), times krr_bench_matvec on the same
seeded X, and checks K.v against the first library's result (relative error).
"""
import argparse
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

CHILD = r"""
import sys, json, ctypes as C, numpy as np
sys.path.insert(0, %(root)r)
import paper_1611_03220_b200 as krr
from paper_1611_03220_b200 import _lib
n, d, reps, path, out, dbg = %(n)d, %(d)d, %(reps)d, %(path)d, %(out)r, %(dbg)d
x = np.random.default_rng(0).standard_normal((n, d))
ctx = krr.Context(0)
ctx.set_option("k1_path", path)
op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(6.0), 1e-6, ctx=ctx)
v = np.random.default_rng(1).standard_normal(n)
kv = op(v)
np.save(out, kv)
if dbg:
    ctx.set_option("i8_debug", dbg)
tot, k1 = C.c_double(), C.c_double()
_lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 2, C.byref(tot), C.byref(k1)))
ts = []
for _ in range(reps):
    _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 3, C.byref(tot), C.byref(k1)))
    ts.append(k1.value)
print(json.dumps({"k1_ms": ts}))
"""


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=262144)
    ap.add_argument("--d", type=int, default=90)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--path", type=int, default=1)
    ap.add_argument("--debug", default="0", help="comma list of i8_debug values (profiling modes) per lib")
    ap.add_argument("libs", nargs="+")
    a = ap.parse_args()
    import numpy as np
    ref = None
    runs = [(lib, int(g)) for lib in a.libs for g in a.debug.split(",")]
    for i, (lib, dbg) in enumerate(runs):
        out = f"/tmp/ab_kv_{i}.npy"
        code = CHILD % dict(root=str(ROOT), n=a.n, d=a.d, reps=a.reps, path=a.path, out=out, dbg=dbg)
        env = dict(os.environ, KRR_B200_LIB=str(Path(lib).resolve()))
        r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env, timeout=600)
        if r.returncode:
            print(json.dumps({"lib": lib, "error": r.stderr[-800:]}), flush=True)
            continue
        res = json.loads(r.stdout.strip().splitlines()[-1])
        kv = np.load(out)
        if ref is None:
            ref = kv
        rel = float(np.linalg.norm(kv - ref) / np.linalg.norm(ref))
        pairs = a.n * (a.n - 1) / 2
        best = min(res["k1_ms"])
        print(json.dumps({"lib": Path(lib).name, "debug": dbg, "n": a.n, "d": a.d, "k1_ms": res["k1_ms"], "best_ms": best,
                          "gevals": a.n * a.n / (best * 1e-3) / 1e9, "rel_vs_first": rel}), flush=True)


if __name__ == "__main__":
    main()
