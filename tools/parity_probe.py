"""Parity diagnostics: GPU vs oracle (two summation orders) residual histories and alpha.

python tools/parity_probe.py  -> prints JSON lines; writes gpurun_out/parity_probe.json
"""
import json
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import paper_1611_03220_b200 as krr  # noqa: E402
from oracle import oracle_ffi as oracle  # noqa: E402


def relerr(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def hist_div(h, g):
    m = min(len(h), len(g))
    h, g = np.asarray(h[:m]), np.asarray(g[:m])
    d = np.abs(h - g) / np.maximum(np.abs(h), 1e-300)
    first = int(np.argmax(d > 1e-8)) + 1 if np.any(d > 1e-8) else None
    return {"max_rel_first20": float(d[:20].max()) if m else 0.0, "first_it_above_1e-8": first}


def case(name, x, y, sigma, lam, s, tau, max_iter):
    out = {"case": name, "n": x.shape[0], "d": x.shape[1], "sigma": sigma, "lam": lam, "s": s,
           "tau": tau, "max_iter": max_iter}
    if s:
        a = oracle.train(x, y, sigma, lam, s, 0, tau, max_iter, order=0, dense_k=x.shape[0] <= 8192)
        b = oracle.train(x, y, sigma, lam, s, 0, tau, max_iter, order=1, dense_k=x.shape[0] <= 8192)
        cfg = krr.SolverConfig(tau=tau, max_iter=max_iter, lambda_=lam, chain=krr.ChainSpec(s1=s), seed=0)
        res = krr.train(krr.Dataset(x, y), krr.KernelSpec.gaussian(sigma), cfg)
        c, rep = res.model.c, res.report
    else:
        a = oracle.solve_gaussian(x, sigma, lam, None, 1.0, y, tau, max_iter, order=0)
        b = oracle.solve_gaussian(x, sigma, lam, None, 1.0, y, tau, max_iter, order=1)
        c, rep = krr.solve_regularized(x, krr.KernelSpec.gaussian(sigma), y, lam, None, tau, max_iter)
    ha = a.residual_history[0, : a.iterations[0]]
    hb = b.residual_history[0, : b.iterations[0]]
    hg = rep.per_rhs[0].residual_history
    out.update({
        "iters": {"oracle0": a.iterations[0], "oracle1": b.iterations[0], "gpu": rep.per_rhs[0].iterations},
        "converged": {"oracle0": a.converged[0], "gpu": rep.per_rhs[0].converged},
        "final_res": {"oracle0": a.final_residual[0], "gpu": rep.per_rhs[0].final_residual},
        "alpha_rel": {"floor_o0_o1": relerr(b.c, a.c), "gpu_o0": relerr(c, a.c), "gpu_o1": relerr(c, b.c)},
        "hist": {"o0_o1": hist_div(ha, hb), "gpu_o0": hist_div(ha, hg)},
        "phase_ms": getattr(rep, "phase_ms", {}),
    })
    print(json.dumps(out), flush=True)
    return out


def main():
    rows = []
    x = oracle.random_matrix(800, 5, 21)
    y = oracle.random_matrix(800, 1, 22)
    rows.append(case("plain_cg_800", x, y, 1.5, 1e-1, 0, 1e-8, 500))
    for (n, d, sig, lam, s) in [(2000, 3, 2.0, 1e-2, 256), (4000, 8, 4.0, 1e-2, 512),
                                (4000, 16, 6.0, 1e-2, 1024), (3000, 54, 3.0, 1e-4, 512)]:
        x = oracle.random_matrix(n, d, 11)
        y = oracle.random_matrix(n, 1, 12)
        rows.append(case(f"train_{n}_{d}", x, y, sig, lam, s, 1e-8 if lam >= 1e-2 else 1e-6, 500))
    x, y = krr.generate_config(1, 8192, 16, 1, 0)
    rows.append(case("C1_first60", x, y, 4.0, 1e-3, 1024, 1e-6, 60))
    od = ROOT / "gpurun_out"
    if od.exists():
        (od / "parity_probe.json").write_text(json.dumps(rows, indent=1))


if __name__ == "__main__":
    main()
