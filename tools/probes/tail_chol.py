import sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2206_14148_b200 as tb
from oracle import sgpr as osgpr
from paper_2206_14148_b200 import synthetic
seed = 70
rng = np.random.default_rng(5000 + seed)
N = int(rng.integers(500, 20_000)); d = int(rng.choice([2, 3, 5, 8, 11, 16])); M = int(rng.integers(8, min(600, N // 2)))
kind = "rbf"; dtype = np.float32 if rng.random() < 0.7 else np.float64
var = float(rng.uniform(0.5, 2.0)); ls = [float(v) for v in rng.uniform(0.8, 2.5, d)]; noise = float(rng.uniform(0.01, 0.2))
X, y, Z, Xs = synthetic.sgpr_data(N, d, M, seed=seed, n_test=64, dtype=dtype)
K = osgpr.kuu(Z, kind, var, ls, 1e-6)
w = np.linalg.eigvalsh(K); print("Kuu eig min %.3e max %.3e" % (w[0], w[-1]))
for nz in (noise, 1e3, 1e8):
    try:
        m = tb.SGPR(X, y, Z, kind, var, ls, nz, engine="i8", tail="packed"); e = m.elbo(); print("noise", nz, "ok", e)
    except Exception as ex:
        print("noise", nz, "ERR", repr(ex)[:120])
for jit in (1e-6, 1e-5, 1e-4):
    try:
        m = tb.SGPR(X, y, Z, kind, var, ls, noise, engine="i8", tail="packed", jitter=jit); e = m.elbo(); print("jitter", jit, "ok")
    except Exception as ex:
        print("jitter", jit, "ERR", repr(ex)[:120])
# numpy cholesky of Kuu and A with the oracle stats
S, v, yy = osgpr.sufficient_stats(X, y, Z, kind, var, ls)
A = K + S / noise
for nm, Mx in (("Kuu", K), ("A", A)):
    try:
        np.linalg.cholesky(Mx); print(nm, "numpy chol ok, cond %.3e" % np.linalg.cond(Mx))
    except Exception as ex:
        print(nm, "numpy chol FAIL", ex)
