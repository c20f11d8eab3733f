#!/usr/bin/env python
"""Oracle fixtures at the BASELINE configs: what the reference algorithm
(oracle/krr_oracle.cpp, Eigen-like summation order, all host threads) produces on the
BASELINE generators, for the -m gpu parity tests in tests/test_gpu_config_parity.py.

  python tests/golden/make_config_fixtures.py 2 3 4 5      # -> tests/golden/config{c}_fixture.npz

C2 / C3 (full iterate-level pins): the whole train path on the CPU — RFF features
(sketches.cpp:37-41), build_preconditioner (precond.cpp:20-40: Z^T Z + lambda I, LLT with the
jitter retry, U = L^-1 Z^T), then pcg_solve (solver.cpp:22-67) with K on the fly for ITERS
iterations; stored: the residual history, the iterate x_k at sampled rows after every
iteration, alpha's norm, and blocks of U (its first and last 64 rows at the sampled columns:
the last rows depend on every entry of Z^T Z, the whole Cholesky factor and the TRSM).

C4 / C5 (n = 1M / 524288: a CPU Z^T Z alone is ~1e14 flop): the leading-block pin — U's first
64 rows depend only on Z's first 64 feature columns (U = L^-1 Z^T with L lower triangular), so
Z[:, :64] is formed for all n rows, G00 = Z0^T Z0 + lambda I (64 x 64), L00 = chol(G00), and
U[:64, rows] = L00^-1 Z0[rows]^T at the sampled columns; plus Z rows, and sampled rows of
(K + lambda I) y (the first PCG mat-vec's input is y's preconditioned image; y itself is pinned).
"""
from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parents[1]
sys.path.insert(0, str(ROOT))

from oracle import oracle_ffi as oracle  # noqa: E402

# cfg: (n, d, t, sigma, lambda, s) -- BASELINE.json configs[1..4]
CONFIGS = {2: (65536, 54, 1, 3.0, 1e-4, 2048), 3: (262144, 90, 1, 6.0, 1e-5, 4096),
           4: (1048576, 90, 1, 6.0, 1e-6, 8192), 5: (524288, 440, 16, 20.0, 1e-5, 16384)}
ITERS = {2: 10, 3: 3}
NSAMPLE = 256
BLOCK = 64


def sample_rows(n: int) -> np.ndarray:
    r = np.random.default_rng(20261020).choice(n, size=NSAMPLE - 2, replace=False)
    return np.unique(np.concatenate([[0, n - 1], r])).astype(np.int64)


def full_fixture(cfg: int) -> dict:
    n, d, t, sigma, lam, s = CONFIGS[cfg]
    its = ITERS[cfg]
    oracle.set_threads(oracle.num_threads())
    t0 = time.perf_counter()
    x, y = oracle.generate_config(cfg, n, d, t, 0)
    rows = sample_rows(n)
    w, b = oracle.rff_realize(0, d, s, sigma)
    z = oracle.rff_apply_rows(x, w, b)
    z_rows = z[rows, :BLOCK].copy()
    u, jit = oracle.build_preconditioner(z, lam)
    del z
    t_build = time.perf_counter() - t0
    u_first = u[:BLOCK][:, rows].copy()
    u_last = u[s - BLOCK:][:, rows].copy()
    xs = []

    def observer(it, xk):
        xs.append(np.asarray(xk)[rows].copy())

    res = oracle.pcg_solve(lambda v: oracle.kernel_matvec(x, sigma, lam, v),
                           lambda v: oracle.precond_apply(u, lam, v), y[:, 0], 1e-6, its, observer=observer)
    t_all = time.perf_counter() - t0
    return dict(cfg=cfg, n=n, d=d, s=s, sigma=sigma, lam=lam, iters=its, rows=rows, z_rows=z_rows,
                u_first=u_first, u_last=u_last, jitter=int(jit),
                residual_history=np.asarray(res.residual_history, dtype=np.float64),
                x_rows=np.asarray(xs), alpha_norm=float(np.linalg.norm(res.solution)),
                alpha_rows=np.asarray(res.solution)[rows].copy(), iterations=res.iterations,
                seconds_build=t_build, seconds_total=t_all, threads=oracle.num_threads())


def block_fixture(cfg: int) -> dict:
    n, d, t, sigma, lam, s = CONFIGS[cfg]
    oracle.set_threads(oracle.num_threads())
    t0 = time.perf_counter()
    x, y = oracle.generate_config(cfg, n, d, t, 0)
    rows = sample_rows(n)
    w, b = oracle.rff_realize(0, d, s, sigma)
    # apply_rows on the first BLOCK features: the oracle scales by sqrt(2 / rows(w)); rescale to s
    z0 = oracle.rff_apply_rows(x, w[:BLOCK], b[:BLOCK]) * np.sqrt(BLOCK / s)
    g00 = z0.T @ z0 + lam * np.eye(BLOCK)
    l00 = oracle.cholesky(g00)
    u_first = oracle.triangular_solve(l00, np.ascontiguousarray(z0[rows].T))
    ky = np.concatenate([oracle.kernel_matvec(x, sigma, lam, y, rows=(int(r), int(r) + 1)) for r in rows[:32]])
    return dict(cfg=cfg, n=n, d=d, s=s, sigma=sigma, lam=lam, rows=rows, z_rows=z0[rows].copy(),
                u_first=u_first, ky_rows=ky, seconds_total=time.perf_counter() - t0, threads=oracle.num_threads())


def main(argv):
    for a in argv or ["2", "3", "4", "5"]:
        cfg = int(a)
        fx = full_fixture(cfg) if cfg in ITERS else block_fixture(cfg)
        out = HERE / f"config{cfg}_fixture.npz"
        np.savez_compressed(out, **{k: np.asarray(v) for k, v in fx.items()})
        print(f"config {cfg}: {out.name} ({out.stat().st_size / 1024:.0f} KiB, {fx['seconds_total']:.0f} s)",
              flush=True)


if __name__ == "__main__":
    main(sys.argv[1:])
