"""Seeded synthetic inputs for the benchmark configurations.

``uniform_inputs`` reproduces the reference's ``random_inputs``
(/root/reference/pkg/src/tensorbudget/frontend.py:128-138): one
``default_rng(seed)``, parameters drawn in graph-parameter order
(database x first, then queries q, frontend.py:108-109) from U[low, high).
The Gaussian generators follow SURVEY.md §8(d) for configs C1-C5.
"""

from __future__ import annotations

import numpy as np


def uniform_inputs(shapes, seed: int, dtype=np.float64, low=-1.0, high=1.0):
    rng = np.random.default_rng(seed)
    return [rng.uniform(low, high, size=s).astype(dtype) for s in shapes]


def gaussian_knn(n: int, m: int, d: int, seed: int = 0, dtype=np.float32):
    """x ~ N(0,1)[n,d], q ~ N(0,1)[m,d] drawn from one stream (x first)."""
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((n, d), dtype=np.float32 if dtype == np.float32 else np.float64)
    q = rng.standard_normal((m, d), dtype=np.float32 if dtype == np.float32 else np.float64)
    return x.astype(dtype, copy=False), q.astype(dtype, copy=False)


def quantized_knn(n: int, m: int, d: int, seed: int = 0, dtype=np.float32):
    """Tie-stress variant: values round(U[0,1)*255)/255 (quantised pixels)."""
    rng = np.random.default_rng(seed)
    x = (np.round(rng.uniform(0, 1, (n, d)) * 255) / 255).astype(dtype)
    q = (np.round(rng.uniform(0, 1, (m, d)) * 255) / 255).astype(dtype)
    return x, q


def sgpr_data(N: int, d: int, M: int, seed: int = 0, n_test: int = 0,
              noise: float = 0.1, dtype=np.float32, z: str = "subset"):
    """X ~ N(0, I_d), y = sin(sum X) + noise*eps, Z = a random subset of X
    (z="subset") or independent N(0, I_d) draws (z="normal", as bench.py's
    C4 does), X* ~ N(0, I_d)."""
    rng = np.random.default_rng(seed)
    X = rng.standard_normal((N, d)).astype(dtype)
    y = (np.sin(X.astype(np.float64).sum(axis=1))
         + noise * rng.standard_normal(N)).astype(dtype)
    if z == "normal":
        Z = rng.standard_normal((M, d)).astype(dtype)
    else:
        Z = X[rng.choice(N, size=M, replace=False)].copy()
    Xs = rng.standard_normal((n_test, d)).astype(dtype)
    return X, y, Z, Xs
