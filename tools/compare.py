"""The reference's `krr bench` three-row comparison (krr.cpp:299-437) on the device, for a
BASELINE config: preconditioned PCG (RFF Woodbury), plain CG (no preconditioner) and the
sketch-and-solve random-features baseline (solver.cpp:175-193).  The last 20 % of the
generated rows are held out as the test set.  Metric: mean squared error of the scores
(and the sign error rate for the +-1 config 2).

python tools/compare.py --configs 1,2 [--max-iter 500] [--tau 1e-6] [--precision 64]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1611_03220_b200 as krr  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2")
    ap.add_argument("--max-iter", type=int, default=500)
    ap.add_argument("--tau", type=float, default=1e-6)
    ap.add_argument("--precision", type=int, default=64)
    args = ap.parse_args()
    out_all = []
    for cfg in [int(c) for c in args.configs.split(",")]:
        n, d, t, sigma, lam, s = krr.CONFIGS[cfg]
        x, y = krr.generate_config(cfg, n, d, t, 0)
        ntr = int(n * 0.8)
        xtr, ytr, xte, yte = x[:ntr], y[:ntr], x[ntr:], y[ntr:]
        kern = krr.KernelSpec.gaussian(sigma)
        chain = krr.ChainSpec(s1=s)

        def metrics(pred_tr, pred_te):
            m = {"train_mse": float(np.mean((pred_tr - ytr) ** 2)), "test_mse": float(np.mean((pred_te - yte) ** 2))}
            if cfg == 2:
                m["train_error"] = float(np.mean(np.sign(pred_tr) != ytr))
                m["test_error"] = float(np.mean(np.sign(pred_te) != yte))
            return m

        rows = []
        ctx = krr.Context(0)
        ctx.set_precision(args.precision)
        # row 1: PCG + RFF Woodbury preconditioner
        t0 = time.perf_counter()
        res = krr.train(krr.Dataset(xtr, ytr), kern,
                        krr.SolverConfig(tau=args.tau, max_iter=args.max_iter, lambda_=lam, chain=chain, seed=0), ctx=ctx)
        wall = time.perf_counter() - t0
        rows.append({"name": "pcg+precond", "iterations": max(r.iterations for r in res.report.per_rhs),
                     "time_sec": wall, **metrics(krr.predict_scores(res.model, xtr, ctx=ctx),
                                                  krr.predict_scores(res.model, xte, ctx=ctx))})
        # row 2: plain CG
        t0 = time.perf_counter()
        c, rep = krr.solve_regularized(xtr, kern, ytr, lam, None, args.tau, args.max_iter, ctx=ctx)
        wall = time.perf_counter() - t0
        m2 = krr.KrrModel(kern, xtr, c, [], lam, 0)
        rows.append({"name": "plain-cg", "iterations": max(r.iterations for r in rep.per_rhs), "time_sec": wall,
                     **metrics(krr.predict_scores(m2, xtr, ctx=ctx), krr.predict_scores(m2, xte, ctx=ctx))})
        # row 3: random-features sketch-and-solve
        t0 = time.perf_counter()
        rf = krr.train_random_features_baseline(krr.Dataset(xtr, ytr), kern, chain, lam, seed=0, ctx=ctx)
        wall = time.perf_counter() - t0
        rows.append({"name": "random-features", "iterations": None, "time_sec": wall,
                     **metrics(krr.baseline_predict_scores(rf, xtr, ctx=ctx), krr.baseline_predict_scores(rf, xte, ctx=ctx))})
        ctx.close()
        rec = {"config": cfg, "n_train": ntr, "n_test": n - ntr, "d": d, "sigma": sigma, "lambda": lam, "s": s,
               "precision": args.precision, "rows": rows}
        out_all.append(rec)
        print(f"config {cfg} (n_train = {ntr}, d = {d}, s = {s}, lambda = {lam}):")
        print(f"  {'method':18s}{'iterations':>12s}{'time (s)':>12s}{'train mse':>14s}{'test mse':>14s}")
        for r in rows:
            it = "-" if r["iterations"] is None else str(r["iterations"])
            print(f"  {r['name']:18s}{it:>12s}{r['time_sec']:12.3f}{r['train_mse']:14.6f}{r['test_mse']:14.6f}")
        print(json.dumps(rec), flush=True)
    od = ROOT / "gpurun_out"
    if od.exists():
        (od / "compare.json").write_text(json.dumps(out_all, indent=1))


if __name__ == "__main__":
    main()
