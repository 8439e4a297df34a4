import sys
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import paper_2206_14148_b200 as tb
from oracle import sgpr as osgpr
from paper_2206_14148_b200 import synthetic
from conftest import rel_err
for seed in [int(v) for v in sys.argv[1].split(",")]:
    rng = np.random.default_rng(5000 + seed)
    N = int(rng.integers(500, 20_000)); d = int(rng.choice([2, 3, 5, 8, 11, 16])); M = int(rng.integers(8, min(600, N // 2)))
    kind = ["rbf", "matern32"][seed % 2]
    dtype = np.float32 if rng.random() < 0.7 else np.float64
    var = float(rng.uniform(0.5, 2.0)); ls = [float(v) for v in rng.uniform(0.8, 2.5, d)]; noise = float(rng.uniform(0.01, 0.2))
    engine = "auto" if rng.random() < 0.7 else "f64"
    X, y, Z, Xs = synthetic.sgpr_data(N, d, M, seed=seed, n_test=64, dtype=dtype)
    limit = None
    if rng.random() < 0.5:
        inputs = (N * d + N + M * d) * np.dtype(dtype).itemsize
        full = tb.sgpr.plan(N, M, d, kernel=kind).peak_bytes
        limit = inputs + int((full - inputs) * rng.uniform(0.5, 1.0)) + 2**20
    ref, w = osgpr.elbo(X, y, Z, kind, var, ls, noise)
    mu_ref = osgpr.predict_mean(Xs, Z, w, kind, var, ls)
    m = tb.SGPR(X, y, Z, kind, var, ls, noise, memory_limit=limit, engine=engine); e = m.elbo(); mu = m.predict_mean(Xs)
    st = None
    print(seed, "engine", engine, "->", m.engine, "limit", limit, "cond_lb", m.cond_kuu_lb, "tail", m.tail,
          "fits", m._dense_tail_fits(), "elbo rel %.1e mean %.1e" % (abs(e - ref) / abs(ref), rel_err(mu, mu_ref)))
