"""GPU probe: FP64 pipe micro-benchmarks + K1 mat-vec throughput at the BASELINE shapes.

python tools/probe.py [--sizes 8192:16,65536:54,...] [--steps 3] [--resident -1|0|1]
Prints JSON lines (and writes gpurun_out/probe.json when that directory exists).
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
from paper_1611_03220_b200 import _lib
from paper_1611_03220_b200 import _diag  # noqa: E402

MB_KEYS = ["dmma_tflops", "dfma_tflops", "mixed_tflops", "exp_libdevice_gevals", "exp_table_gevals",
           "sms", "clock_mhz", "split_warps_tflops", "imma_legacy_tops"]


def report(n, d, ms, k1, t_set, res, exp_mode, warps, grouped=0, path=0):
    pairs = n * (n - 1) / 2
    dp = (d + 2 + 3) // 4 * 4
    row = {"n": n, "d": d, "path": ["dmma", "i8", "f32"][path], "resident": res, "warps": warps, "grouped": grouped, "exp_mode": exp_mode, "ms_per_matvec": ms, "k1_ms": k1,
           "gevals_per_s": n * n / (ms * 1e-3) / 1e9,
           "unique_pairs_per_s": pairs / (k1 * 1e-3) / 1e9,
           "dot_tflops": pairs * 2 * d / (k1 * 1e-3) / 1e12,
           "fp64_ops_tflops_equiv": pairs * 2 * (dp + 12) / (k1 * 1e-3) / 1e12,
           "set_data_s": t_set}
    print(json.dumps(row), flush=True)
    return row


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="8192:16,65536:54,262144:90")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--exp-mode", type=int, default=1)
    ap.add_argument("--resident", type=int, default=-1, help="-1: both K1 variants")
    ap.add_argument("--warps", type=int, default=-1, help="-1: both 8 and 16")
    ap.add_argument("--grouped", type=int, default=-1, help="-1: both (resident 8-warp only)")
    ap.add_argument("--path", type=int, default=0, help="K1 path: 0 = FP64 DMMA, 1 = tcgen05 INT8 slices, -1 both")
    ap.add_argument("--no-microbench", action="store_true")
    ap.add_argument("--precision", type=int, default=64, help="64 (fp64) or 32 (fp32 mode)")
    ap.add_argument("--i8-debug", default="0", help="comma list of K1-I8 profiling modes (1 no MMA, 2 no exp)")
    args = ap.parse_args()
    out = {}
    ctx = krr.Context(0)
    if not args.no_microbench:
        res = np.zeros(9)
        _diag.check(_diag.LIB.krr_diag_microbench(0, _lib.ptr(res)))
        out["microbench"] = dict(zip(MB_KEYS, res.tolist()))
        print(json.dumps(out["microbench"]), flush=True)
    rows = []
    for spec in args.sizes.split(","):
        n, d = (int(v) for v in spec.split(":"))
        x = np.random.default_rng(0).standard_normal((n, d))
        t0 = time.perf_counter()
        _lib.check(_lib.LIB.krr_set_data(ctx.handle, _lib.ptr(x), n, d, 6.0))
        t_set = time.perf_counter() - t0
        combos = [(r, w, gp) for w in ([8, 16] if args.warps < 0 else [args.warps])
                  for r in ([1, 0] if args.resident < 0 else [args.resident])
                  for gp in ([1, 0] if args.grouped < 0 and r == 1 and w == 8 else
                             [max(args.grouped, 0) if r == 1 and w == 8 else 0])]
        paths = [0, 1] if args.path < 0 else [args.path]
        combos = [(r, w, gp, pa) for pa in paths for (r, w, gp) in (combos if pa == 0 else [(1, 8, 1)])]
        dbgs = [int(v) for v in args.i8_debug.split(",")]
        combos = [(r, w, gp, pa, dbg) for (r, w, gp, pa) in combos for dbg in (dbgs if pa == 1 else [0])]
        ctx.set_precision(args.precision)
        for res, w, gp, pa, dbg in combos:
            ctx.set_option("k1_path", pa)
            ctx.set_option("i8_debug", dbg)
            ctx.set_option("k1_resident", res)
            ctx.set_option("k1_warps", w)
            ctx.set_option("k1_grouped", gp)
            ctx.set_option("exp_mode", args.exp_mode)
            tot, k1 = C.c_double(), C.c_double()
            _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, 1, C.byref(tot), C.byref(k1)))  # warm
            _lib.check(_lib.LIB.krr_bench_matvec(ctx.handle, 1e-6, args.steps, C.byref(tot), C.byref(k1)))
            if dbg:
                print(json.dumps({"i8_debug": dbg}), flush=True)
            rows.append(report(n, d, tot.value / args.steps, k1.value, t_set, res, args.exp_mode, w, gp,
                               2 if args.precision == 32 else pa))
        ctx.set_option("i8_debug", 0)
    out["matvec"] = rows
    ctx.close()
    od = ROOT / "gpurun_out"
    if od.exists():
        (od / "probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
