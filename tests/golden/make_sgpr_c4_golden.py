"""Generate the C4-shape SGPR golden (tests/golden/sgpr_c4_shape.npz).

The reference has no SGPR code, so this fixture
comes from the fp64 oracle (oracle/sgpr.py, the GPflow 2.3.1 restatement
pinned against scikit-learn's exact GP in tests/test_oracle.py), evaluated at
the benchmarked configuration's shape with N reduced so numpy finishes in a
few minutes: d = 11, M = 1e4 (M_pad = 79 tiles of 128), RBF, variance 1,
lengthscale 1, noise 0.01 — BASELINE.json configs[3] / bench.py SG_*.
Z is drawn independently of X from the same N(0, I) (as bench.py does).

Stored:
* elbo / mean          — unquantised fp64 statistics (the north-star gate, 1e-4)
* elbo_q / mean_q      — statistics of the 24-bit fixed-point Kuf that the i8
                         engine computes exactly (oracle.sgpr.sufficient_stats_fixed24
                         semantics), so the GPU engine + packed tail can be held
                         far tighter than 1e-4
* v_q, diag_q, rows_q  — v, diag(Sigma) and 8 full rows of Sigma under that
                         quantisation (rows in the first, a middle and the last,
                         ragged tile), and Sigma_q @ r for a seeded r (checksum)
* x_sha                — sha256 of the generated inputs (generator drift check)

Sigma_q is formed exactly: Q = a 2^12 + b (a, b < 2^12), so a a^T, b b^T and
(a+b)(a+b)^T are integer sums below 2^53 and exact in fp64 GEMMs.

    python tests/golden/make_sgpr_c4_golden.py        (about 2-4 minutes, 8 cores)
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import sgpr as osgpr  # noqa: E402
from oracle.mvm import kernel_matrix  # noqa: E402
from paper_2206_14148_b200 import synthetic  # noqa: E402

N, D, M, N_TEST, SEED = 30_000, 11, 10_000, 300, 2024
VAR, LS, NOISE = 1.0, 1.0, 0.01
ROWS = np.array([0, 1, 127, 128, 5000, 9983, 9998, 9999])


def kuf_chunks(X, Z, step=2048):
    for s in range(0, X.shape[0], step):
        yield s, kernel_matrix(Z, X[s:s + step], "rbf", VAR, LS)


def main():
    t0 = time.time()
    X, y, Z, Xs = synthetic.sgpr_data(N, D, M, seed=SEED, n_test=N_TEST, dtype=np.float32,
                                      z="normal")
    h = hashlib.sha256()
    for a in (X, y, Z, Xs):
        h.update(np.ascontiguousarray(a).tobytes())
    y64 = y.astype(np.float64)
    S = np.zeros((M, M))
    v = np.zeros(M)
    Sa = np.zeros((M, M))
    Sb = np.zeros((M, M))
    Sab = np.zeros((M, M))
    vq = np.zeros(M)
    for s, K in kuf_chunks(X, Z):
        ys = y64[s:s + K.shape[1]]
        S += K @ K.T
        v += K @ ys
        Q = np.minimum(np.rint(K * (2.0 ** 24 / VAR)), 2.0 ** 24 - 1)
        a = np.floor(Q / 4096.0)
        b = Q - a * 4096.0
        c = a + b
        Sa += a @ a.T
        Sb += b @ b.T
        Sab += c @ c.T
        vq += Q @ ys
        print(f"chunk {s}: {time.time() - t0:.0f}s", flush=True)
    cross = Sab - Sa - Sb                      # a b^T + b a^T, exact integers
    Sq = (Sa * 2.0 ** 24 + cross * 2.0 ** 12 + Sb) * (VAR * VAR * 2.0 ** -48)
    vq *= VAR * 2.0 ** -24
    del Sa, Sb, Sab, cross
    yy = float(y64 @ y64)
    Kuu = osgpr.kuu(Z, "rbf", VAR, LS)
    elbo, w = osgpr.elbo_from_stats(S, v, yy, N, Kuu, NOISE, VAR)
    elbo_q, w_q = osgpr.elbo_from_stats(Sq, vq, yy, N, Kuu, NOISE, VAR)
    mean = osgpr.predict_mean(Xs, Z, w, "rbf", VAR, LS)
    mean_q = osgpr.predict_mean(Xs, Z, w_q, "rbf", VAR, LS)
    r = np.random.default_rng(7).standard_normal(M)
    out = dict(N=N, d=D, M=M, seed=SEED, variance=VAR, lengthscale=LS, noise=NOISE,
               x_sha=h.hexdigest(), elbo=elbo, elbo_q=elbo_q, mean=mean, mean_q=mean_q,
               v_q=vq, yy=yy, diag_q=np.diag(Sq).copy(), rows=ROWS, rows_q=Sq[ROWS].copy(),
               check_q=Sq @ r, cond_kuu=float(np.linalg.cond(Kuu)))
    np.savez_compressed(os.path.join(HERE, "sgpr_c4_shape.npz"), **out)
    print(f"elbo {elbo:.10e}  elbo_q {elbo_q:.10e}  rel {(elbo_q - elbo) / abs(elbo):.2e}  "
          f"mean dq {np.abs(mean_q - mean).max() / np.abs(mean).max():.2e}  "
          f"cond {out['cond_kuu']:.3e}  {time.time() - t0:.0f}s")


if __name__ == "__main__":
    main()
