"""GPU probe: FP64 pipe micro-benchmarks + K1 mat-vec throughput at the BASELINE shapes.

python tools/probe.py [--sizes 8192:16,65536:54,...] [--steps 3]
Prints one JSON object (written to gpurun_out/probe.json when that directory exists).
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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8192:16,65536:54,262144:90,1048576:90")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--exp-mode", type=int, default=1)
    args = ap.parse_args()
    out = {}
    ctx = krr.Context(0)
    res = np.zeros(8)
    _lib.check(_lib.LIB.krr_microbench(ctx.handle, _lib.ptr(res)))
    out["microbench"] = dict(zip(["dmma_tflops", "dfma_tflops", "mixed_tflops", "exp_libdevice_gevals",
                                  "exp_table_gevals", "sms", "clock_mhz"], res[:7].tolist()))
    print(json.dumps(out["microbench"]), flush=True)
    rows = []
    for spec in args.sizes.split(","):
        n, d = (int(v) for v in spec.split(":"))
        rng = np.random.default_rng(0)
        x = rng.standard_normal((n, d))
        t0 = time.perf_counter()
        _lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, 6.0))
        t_set = time.perf_counter() - t0
        tot, k1 = C.c_double(), C.c_double()
        _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))  # warm
        _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, args.steps, C.byref(tot), C.byref(k1)))
        ms = tot.value / args.steps
        pairs = n * (n - 1) / 2
        dp = (d + 2 + 3) // 4 * 4
        row = {"n": n, "d": d, "ms_per_matvec": ms, "k1_ms": k1.value,
               "gevals_per_s": n * n / (ms * 1e-3) / 1e9,
               "unique_pairs_per_s": pairs / (k1.value * 1e-3) / 1e9,
               "dot_tflops": pairs * 2 * d / (k1.value * 1e-3) / 1e12,
               "fp64_lane_ops_tflops_equiv": pairs * (2 * dp + 2 * 11) / (k1.value * 1e-3) / 1e12,
               "set_data_s": t_set}
        rows.append(row)
        print(json.dumps(row), flush=True)
    out["matvec"] = rows
    ctx.close()
    od = ROOT / "gpurun_out"
    if od.exists():
        (od / "probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
