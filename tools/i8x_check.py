"""K1-I8X vs K1-I8 / DMMA K1: parity (vs the oracle at small n, vs the DMMA K1 at large n) and
K1 time per mat-vec.  python tools/i8x_check.py [--sizes 65536:90,...] [--paths 3,1,0] [--steps 3]
"""
import argparse
import ctypes as C
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402


def matvec(ctx, v):
    out = np.empty_like(v)
    _lib.check(_lib.LIB.krr_kernel_matvec(ctx.handle, 1e-3, _lib.ptr(v), 1, _lib.ptr(out)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="4096:90:6,65536:90:6,65536:54:3,262144:90:6")
    ap.add_argument("--paths", default="3,1,0")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--oracle-max", type=int, default=8192)
    ap.add_argument("--debug", default="0")
    args = ap.parse_args()
    ctx = krr.Context(0)
    for spec in args.sizes.split(","):
        n, d, sigma = spec.split(":")
        n, d, sigma = int(n), int(d), float(sigma)
        rng = np.random.default_rng(n + d)
        x = rng.standard_normal((n, d))
        v = rng.standard_normal(n)
        _lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, sigma))
        ref = None
        if n <= args.oracle_max:
            from oracle import oracle_ffi as oracle
            ref = oracle.kernel_matvec(x, sigma, 1e-3, v)
        outs = {}
        for path in [int(p) for p in args.paths.split(",")]:
            for dbg in [int(x) for x in args.debug.split(",")]:
                ctx.set_option("k1_path", path)
                ctx.set_option("i8_debug", dbg)
                eff = ctx.get_option("k1_path_effective")
                o = matvec(ctx, v)
                if dbg == 0:
                    outs[path] = o
                tot, k1 = C.c_double(), C.c_double()
                _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-3, args.steps, C.byref(tot), C.byref(k1)))
                row = {"n": n, "d": d, "sigma": sigma, "path": path, "eff": eff, "debug": dbg,
                       "k1_ms": k1.value, "gevals": n * n / (k1.value * 1e-3) / 1e9}
                if ref is not None and dbg == 0:
                    row["rel_vs_oracle"] = float(np.linalg.norm(o - ref) / np.linalg.norm(ref))
                if 0 in outs and path != 0 and dbg == 0:
                    row["rel_vs_dmma"] = float(np.linalg.norm(o - outs[0]) / np.linalg.norm(outs[0]))
                print(json.dumps(row), flush=True)
        ctx.set_option("i8_debug", 0)
        if 0 in outs and 3 in outs:
            print(json.dumps({"n": n, "i8x_vs_dmma": float(np.linalg.norm(outs[3] - outs[0]) / np.linalg.norm(outs[0]))}))


if __name__ == "__main__":
    main()
