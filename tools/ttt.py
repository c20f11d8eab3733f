"""Time-to-tolerance: the full device path (RFF K2 -> Woodbury build -> PCG) on BASELINE
configs, with phase timings, iterations and residual histories.

python tools/ttt.py --configs 2,3 [--max-iter 500] [--oracle-iters 0]
Writes gpurun_out/ttt_<cfg>.json.  With --oracle-iters K > 0 the first K iterations are
also run through the CPU oracle (on-the-fly K, all host threads) for iterate-level parity.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1611_03220_b200 as krr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="2")
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--tau", type=float, default=1e-6)
    ap.add_argument("--oracle-iters", type=int, default=0)
    ap.add_argument("--n", type=int, default=0, help="override n (sub-sampled config)")
    ap.add_argument("--precision", type=int, default=64, help="64 (fp64, default) or 32 (optional fp32 mode)")
    ap.add_argument("--pcg-graph", type=int, default=1, help="1: graph-resident PCG loop (default), 0: host loop")
    args = ap.parse_args()
    od = ROOT / "gpurun_out"
    od.mkdir(exist_ok=True)
    for cfg in [int(c) for c in args.configs.split(",")]:
        n, d, t, sigma, lam, s = krr.CONFIGS[cfg]
        if args.n:
            n = args.n
        t0 = time.perf_counter()
        x, y = krr.generate_config(cfg, n, d, t, 0)
        gen_s = time.perf_counter() - t0
        sc = krr.SolverConfig(tau=args.tau, max_iter=args.max_iter, lambda_=lam,
                              chain=krr.ChainSpec(s1=s), seed=0)
        ctx = krr.Context(0)
        ctx.set_precision(args.precision)
        ctx.set_option("pcg_graph", args.pcg_graph)
        res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), sc, ctx=ctx)
        out = {"config": cfg, "precision": args.precision, "n": n, "d": d, "t": t, "sigma": sigma, "lambda": lam, "s": s,
               "tau": args.tau, "max_iter": args.max_iter, "gen_s": gen_s,
               "phase_ms": res.report.phase_ms, "wall_s": res.report.wall_time_sec,
               "per_rhs": [{"iterations": r.iterations, "converged": r.converged,
                            "final_residual": r.final_residual,
                            "residual_history": r.residual_history} for r in res.report.per_rhs],
               "total_matvecs": res.report.total_matvecs,
               "ms_per_iteration": res.report.phase_ms["solve"] / max(1, res.report.total_matvecs)}
        if args.oracle_iters > 0:
            from oracle import oracle_ffi as oracle
            oracle.set_threads(os.cpu_count() or 1)
            k = args.oracle_iters
            t1 = time.perf_counter()
            ref = oracle.train(x, y[:, :1], sigma, lam, s, 0, args.tau, k, dense_k=False)
            cpu_s = time.perf_counter() - t1
            sc2 = krr.SolverConfig(tau=args.tau, max_iter=k, lambda_=lam, chain=krr.ChainSpec(s1=s), seed=0)
            g = krr.train(krr.Dataset(x, y[:, :1]), krr.KernelSpec.gaussian(sigma), sc2, ctx=ctx)
            hg = np.array(g.report.per_rhs[0].residual_history)
            hr = ref.residual_history[0, :k]
            out["oracle_parity"] = {
                "iterations": k, "cpu_seconds": cpu_s, "cpu_threads": os.cpu_count(),
                "hist_max_rel": float(np.max(np.abs(hg - hr) / hr)),
                "alpha_rel": float(np.linalg.norm(g.model.c - ref.c) / np.linalg.norm(ref.c))}
        ctx.close()
        print(json.dumps({k2: v for k2, v in out.items() if k2 != "per_rhs"}), flush=True)
        print(json.dumps({"iterations": [r["iterations"] for r in out["per_rhs"]],
                          "final_residual": [r["final_residual"] for r in out["per_rhs"]]}), flush=True)
        tag = ("_n" + str(n) if args.n else "") + ("_fp32" if args.precision == 32 else "") + \
            ("_hostloop" if not args.pcg_graph else "")
        (od / f"ttt_{cfg}{tag}.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
