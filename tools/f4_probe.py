"""SURVEY 8f4 measurements: the polynomial kernel through the fused K1 (DMMA, ipow epilogue)
against the Gaussian K1 at the same shape, the sketch-chain stages (TensorSketch, SRHT,
Gaussian map) and one polynomial train to tolerance.

python tools/f4_probe.py [--n 65536] [--d 90] [--steps 3]
Prints JSON lines; writes gpurun_out/f4_probe.json when that directory exists.
"""
import argparse
import ctypes as C
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

import paper_1611_03220_b200 as krr  # noqa: E402
from paper_1611_03220_b200 import _lib  # noqa: E402


def bench_matvec(ctx, x, kernel, steps, k1_path=-1):
    ctx.set_option("k1_path", k1_path)
    krr._set_data(ctx, x, kernel)
    tot, k1 = C.c_double(), C.c_double()
    _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 0.0, steps, C.byref(tot), C.byref(k1)))
    n = x.shape[0]
    ms = tot.value / steps
    return {"kernel": kernel.family, "degree": kernel.degree if kernel.family == "polynomial" else None,
            "k1_path": int(ctx.get_option("k1_path_effective")), "n": n, "d": x.shape[1],
            "ms_per_matvec": ms, "k1_ms": k1.value, "gevals_per_s": n * n / (ms * 1e-3) / 1e9}


def timed(fn):
    t0 = time.perf_counter()
    out = fn()
    return out, time.perf_counter() - t0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=65536)
    ap.add_argument("--d", type=int, default=90)
    ap.add_argument("--steps", type=int, default=3)
    args = ap.parse_args()
    rows = []
    ctx = krr.Context(0)
    n, d = args.n, args.d
    rng = np.random.default_rng(0)
    x = rng.normal(size=(n, d)) / np.sqrt(d)
    poly = krr.KernelSpec.polynomial(1.0 / d, 1.0, 3)
    for kern, path in [(krr.KernelSpec.gaussian(1.0), 0), (krr.KernelSpec.gaussian(1.0), -1), (poly, -1),
                       (krr.KernelSpec.polynomial(1.0 / d, 1.0, 2), -1), (krr.KernelSpec.polynomial(1.0 / d, 1.0, 6), -1),
                       (poly, 0), (krr.KernelSpec.polynomial(1.0 / d, 1.0, 6), 0)]:
        r = bench_matvec(ctx, x, kern, args.steps, path)
        rows.append(r)
        print(json.dumps(r), flush=True)

    # sketch stages over all n rows (device time inside apply_rows incl. host table upload)
    for spec, kern in [(krr.ChainSpec("TensorSketch", 4096), poly), (krr.ChainSpec("TensorSketch", 4000), poly),
                       (krr.ChainSpec("TensorSketch", 2048, 1024, 512), poly),
                       (krr.ChainSpec("RandomFourier", 4096, 2048, 1024), krr.KernelSpec.gaussian(1.0))]:
        chain = krr.realize_chain(spec, kern, d, 7)
        chain.apply_rows(x[:256], ctx=ctx)  # warm-up
        _, sec = timed(lambda: chain.apply_rows(x, ctx=ctx))
        r = {"chain": [spec.first, spec.s1, spec.s2, spec.s3], "rows": n, "apply_rows_s": sec}
        rows.append(r)
        print(json.dumps(r), flush=True)

    # polynomial train to tolerance (TensorSketch -> SRHT chain)
    y = rng.normal(size=(n, 1))
    cfg = krr.SolverConfig(lambda_=1e-2, tau=1e-6, max_iter=300, chain=krr.ChainSpec("TensorSketch", 4096, 2048),
                           seed=0)
    res, sec = timed(lambda: krr.train(krr.Dataset(x, y), poly, cfg, ctx=ctx))
    st = res.report.per_rhs[0]
    r = {"train": "polynomial q=3 TS(4096)->SRHT(2048)", "n": n, "d": d, "iterations": st.iterations,
         "converged": st.converged, "final_residual": st.final_residual, "wall_s": sec,
         "phase_ms": res.report.phase_ms}
    rows.append(r)
    print(json.dumps(r), flush=True)
    ctx.close()
    out = ROOT / "gpurun_out"
    if out.is_dir():
        (out / "f4_probe.json").write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
