"""Kernel matrix / kernel-MVM oracle (TEST INFRASTRUCTURE ONLY).

* ``se_mvm_reference`` follows the reference's ``build_kernel_mvm`` graph op
  for op (/root/reference/pkg/src/tensorbudget/frontend.py:34-54):
  ``K[i,j] = variance * exp(square(x_i - y_j) * (-0.5 / lengthscale**2))`` and
  ``out = K @ v`` — the ordering of the scale, exp and variance multiply is the
  reference's.  Pinned by reference golden vectors (tests/golden).
* ``kernel_matrix`` generalises it to d-dimensional inputs with per-dimension
  lengthscales (the RBF / Matérn-3/2 kernels GPflow 2.3.1 evaluates for the
  paper's SGPR runs): r^2 = ||(x - z) / l||^2,
  RBF = s^2 exp(-r^2/2), Matérn-3/2 = s^2 (1 + sqrt3 r) exp(-sqrt3 r) with
  r = sqrt(max(r^2, 1e-36)).  Evaluated in fp64 from direct differences.
"""

from __future__ import annotations

import numpy as np

KERNELS = ("rbf", "matern32")


def se_mvm_reference(x, y, v, variance: float = 1.0, lengthscale: float = 1.0,
                     chunk: int = 1024) -> np.ndarray:
    x = np.asarray(x)
    y = np.asarray(y)
    v = np.asarray(v)
    dt = x.dtype.type
    scale = dt(-0.5 / lengthscale ** 2)
    var = dt(variance)
    out = np.empty(x.shape[0], x.dtype)
    for s in range(0, x.shape[0], chunk):
        sq = np.square(x[s:s + chunk, None] - y[None, :])
        kern = var * np.exp(sq * scale)
        out[s:s + chunk] = kern @ v
    return out


def scaled_sqdist(X, Z, lengthscales) -> np.ndarray:
    X = np.asarray(X, np.float64)
    Z = np.asarray(Z, np.float64)
    ls = np.broadcast_to(np.asarray(lengthscales, np.float64), (X.shape[1],))
    Xs = X / ls
    Zs = Z / ls
    diff = Xs[:, None, :] - Zs[None, :, :]
    return np.sum(diff * diff, axis=-1)


def kernel_matrix(X, Z, kind: str = "rbf", variance: float = 1.0,
                  lengthscales=1.0) -> np.ndarray:
    if kind not in KERNELS:
        raise ValueError(f"kernel must be one of {KERNELS}")
    r2 = scaled_sqdist(X, Z, lengthscales)
    if kind == "rbf":
        return variance * np.exp(-0.5 * r2)
    r = np.sqrt(np.maximum(r2, 1e-36))
    s3 = np.sqrt(3.0) * r
    return variance * (1.0 + s3) * np.exp(-s3)


def kernel_mvm(X, Z, w, kind="rbf", variance=1.0, lengthscales=1.0,
               chunk: int = 2048) -> np.ndarray:
    """out[i] = sum_j k(X_i, Z_j) w_j in fp64, chunked over X rows."""
    X = np.asarray(X, np.float64)
    out = np.empty(X.shape[0], np.float64)
    for s in range(0, X.shape[0], chunk):
        out[s:s + chunk] = kernel_matrix(X[s:s + chunk], Z, kind, variance,
                                         lengthscales) @ np.asarray(w, np.float64)
    return out
