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
    ref, w = osgpr.elbo(X, y, Z, kind, var, ls, noise)
    mu_ref = osgpr.predict_mean(Xs, Z, w, kind, var, ls)
    K = osgpr.kuu(Z, kind, var, ls, 1e-6)
    S, v, yy = osgpr.sufficient_stats(X, y, Z, kind, var, ls)
    for eng in ("auto", "f64"):
        m = tb.SGPR(X, y, Z, kind, var, ls, noise, engine=eng); e = m.elbo(); mu = m.predict_mean(Xs)
        print(seed, N, d, M, kind, "cond(Kuu) %.2e cond(A) %.2e" % (np.linalg.cond(K), np.linalg.cond(K + S / noise)),
              eng, "->", m.engine, "cond_lb", None if m.cond_kuu_lb is None else "%.2e" % m.cond_kuu_lb,
              "elbo rel %.1e mean %.1e" % (abs(e - ref) / abs(ref), rel_err(mu, mu_ref)))
