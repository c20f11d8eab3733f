import sys, numpy as np
sys.path.insert(0,'.')
import paper_1611_03220_b200 as krr
from oracle import oracle_ffi as oracle
ctx = krr.Context(0)
n, d = 256, 4
x = oracle.random_matrix(n, d, 2)
ctx.set_option("k1_path", 1)
op = krr.GaussianOperator(x, krr.KernelSpec.gaussian(2.0), 0.0, ctx=ctx)
kk = np.column_stack([op(np.eye(n)[:, j]) for j in range(0, 8)])
want = oracle.gram_matrix(x, 2.0)[:, :8]
err = kk - want
print("max err", np.abs(err).max())
i, j = np.unravel_index(np.argmax(np.abs(err)), err.shape)
print("worst", i, j, kk[i, j], want[i, j])
d2 = ((x[:, None, :] - x[None, :8, :]) ** 2).sum(-1)
lk = -np.log(np.maximum(kk, 1e-300)) * 8.0   # recovered d2 (scale = 1/8)
print("d2 true vs recovered (first rows of col 1):")
for r in range(8, 16):
    print(r, d2[r, 1], lk[r, 1], np.dot(x[r], x[1]), (d2[r,1]-lk[r,1])/2)
bad = np.abs(err) > 1e-10
for j in range(8):
    rows = np.nonzero(bad[:, j])[0]
    print("col", j, "bad rows", rows[:40], len(rows))
# pair-level exact check via full matmat (DMMA K1T not involved: single columns)
