"""Measured parity margins against the oracle (the numbers behind tests/test_gpu_config_parity.py):
python tools/parity_report.py > profiles/r2_parity_report.json"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import paper_1611_03220_b200 as krr  # noqa: E402
from oracle import oracle_ffi as oracle  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def train(ctx, cfg, max_iter, lam=None, tau=1e-6):
    n, d, t, sigma, l0, s = krr.CONFIGS[cfg]
    x, y = krr.generate_config(cfg, n, d, t, 0)
    sc = krr.SolverConfig(tau=tau, max_iter=max_iter, lambda_=lam or l0, chain=krr.ChainSpec(s1=s), seed=0)
    return x, y, krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), sc, ctx=ctx)


out = {}
ctx = krr.Context(0)
for lam in (3e-2, 1e-2):
    n, d, t, sigma, _, s = krr.CONFIGS[1]
    x, y, res = train(ctx, 1, 500, lam)
    fam = [oracle.train(x, y, sigma, lam, s, 0, 1e-6, 500, order=k) for k in (2, 0, 1)]
    out[f"config1_shape_lambda_{lam}"] = {
        "gpu_iterations": res.report.per_rhs[0].iterations, "oracle_iterations": [f.iterations[0] for f in fam],
        "alpha_rel_vs_oracle": rel(res.model.c, fam[0].c),
        "oracle_order_spread": max(rel(f.c, fam[0].c) for f in fam[1:])}
for cfg in (2, 3):
    fx = dict(np.load(ROOT / "tests" / "golden" / f"config{cfg}_fixture.npz"))
    rows, its, s = fx["rows"], int(fx["iters"]), int(fx["s"])
    hist_err, x_err = [], []
    for k in range(1, its + 1):
        x, y, res = train(ctx, cfg, k)
        hist_err.append(rel(res.report.per_rhs[0].residual_history, fx["residual_history"][:k]))
        x_err.append(rel(res.model.c[rows, 0], fx["x_rows"][k - 1]))
    out[f"config{cfg}"] = {"iterations": its, "residual_history_rel_max": max(hist_err), "iterate_rel_per_k": x_err,
                           "u_first_rel": rel(ctx.read_u(0, 64, rows), fx["u_first"]),
                           "u_last_rel": rel(ctx.read_u(s - 64, 64, rows), fx["u_last"])}
    ctx.precond_drop()
ctx.close()
for cfg in (4, 5):
    fx = dict(np.load(ROOT / "tests" / "golden" / f"config{cfg}_fixture.npz"))
    rows = fx["rows"]
    n, d, t, sigma, lam, s = krr.CONFIGS[cfg]
    c = krr.Context(0)
    x, y, res = train(c, cfg, 1)
    u0 = rel(c.read_u(0, 64, rows), fx["u_first"])
    c.precond_drop()
    chain = krr.realize_chain(krr.ChainSpec(s1=s), krr.KernelSpec.gaussian(sigma), d, 0)
    z = chain.rff.apply_rows(x[rows], ctx=c)
    ky = krr.GaussianOperator(x, krr.KernelSpec.gaussian(sigma), lam, ctx=c).matmat(y)
    out[f"config{cfg}"] = {"u_first_rel": u0, "z_rows_max_abs": float(np.max(np.abs(z[:, :64] - fx["z_rows"]))),
                           "ky_rows_rel": rel(ky[rows[:fx["ky_rows"].shape[0]]], fx["ky_rows"])}
    c.close()
print(json.dumps(out, indent=1))
