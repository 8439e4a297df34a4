"""fp64 SGPR (Titsias ELBO + predictive mean) oracle — TEST INFRASTRUCTURE ONLY.

PARITY PARTIALLY PINNED.  The reference package has no SGPR code
(/root/reference/SPEC.md:13,453); the paper ran GPflow 2.3.1 ``SGPR``
(PAPER.md:277), which is neither vendored nor installed here.  This module
restates GPflow 2.3.1 ``SGPR.elbo`` / ``SGPR.predict_f`` (zero mean function,
one output, jitter 1e-6) in numpy fp64:

    Kuu = k(Z,Z) + jitter I,  L = chol(Kuu)
    Sigma = Kuf Kuf^T,  v = Kuf y                   (sufficient statistics)
    AAT = L^-1 Sigma L^-T / s2,  B = I + AAT,  LB = chol(B)
    c = LB^-1 L^-1 v / s2
    ELBO = -N/2 log 2pi - sum log diag LB - N/2 log s2 - yy/(2 s2)
           + c^T c / 2 - tr(Kff)/(2 s2) + tr(AAT)/2
    mean(X*) = K(X*, Z) w,   w = L^-T LB^-T c

Pinned pieces: the SE kernel formula (reference frontend.py:22-54, via
oracle.mvm goldens) and triangular-solve semantics (reference
interpreter.py:475-490).  Everything else is held by the self-checks in
tests/test_oracle.py: Sigma-first == GPflow's A-first order to ~1e-12,
ELBO == exact GP log marginal likelihood at Z = X, ELBO <= log ML, and
invariance to permuting N.
"""

from __future__ import annotations

import math

import numpy as np

from .mvm import kernel_matrix

LOG2PI = math.log(2.0 * math.pi)


def _tri_solve(L, B, lower=True, trans=False):
    from scipy.linalg import solve_triangular
    return solve_triangular(L, B, lower=lower, trans=1 if trans else 0)


def sufficient_stats(X, y, Z, kind="rbf", variance=1.0, lengthscales=1.0,
                     chunk: int = 8192):
    """Sigma = Kuf Kuf^T, v = Kuf y, yy = y^T y, accumulated over N chunks in
    ascending order (the contracted-dim running add of the reference's
    splitter, split.py:322-324)."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64).reshape(-1)
    M = Z.shape[0]
    Sigma = np.zeros((M, M))
    v = np.zeros(M)
    for s in range(0, X.shape[0], chunk):
        Kuf = kernel_matrix(Z, X[s:s + chunk], kind, variance, lengthscales)
        Sigma += Kuf @ Kuf.T
        v += Kuf @ y[s:s + chunk]
    return Sigma, v, float(y @ y)


def sufficient_stats_fixed24(X, y, Z, kind="rbf", variance=1.0, lengthscales=1.0,
                             chunk: int = 8192):
    """Statistics of the B200 fixed-point engine (TB_SGPR_ENGINE_I8), restated
    exactly: Q = min(rint(Kuf / variance * 2^24), 2^24 - 1) once, then
    Sigma = variance^2 2^-48 Q Q^T and v = variance 2^-24 Q y with no rounding
    inside the integer Gram (digit planes a2 2^16 + a1 2^8 + a0, each level
    sum < 2^53, so float64 matmuls of the digit planes are exact)."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64).reshape(-1)
    M = Z.shape[0]
    Sigma = np.zeros((M, M))
    v = np.zeros(M)
    for s in range(0, X.shape[0], chunk):
        K = kernel_matrix(Z, X[s:s + chunk], kind, variance, lengthscales)
        Q = np.minimum(np.rint(K * (2.0 ** 24 / variance)), 2.0 ** 24 - 1)
        a2 = np.floor(Q / 65536.0)
        a1 = np.floor((Q - a2 * 65536.0) / 256.0)
        a0 = Q - a2 * 65536.0 - a1 * 256.0
        L4 = a2 @ a2.T
        L3 = a2 @ a1.T + a1 @ a2.T
        L2 = a2 @ a0.T + a1 @ a1.T + a0 @ a2.T
        L1 = a1 @ a0.T + a0 @ a1.T
        L0 = a0 @ a0.T
        P = (((L4 * 256.0 + L3) * 256.0 + L2) * 256.0 + L1) * 256.0 + L0
        Sigma += P * (variance * variance * 2.0 ** -48)
        v += (Q @ y[s:s + chunk]) * (variance * 2.0 ** -24)
    return Sigma, v, float(y @ y)


def kuu(Z, kind="rbf", variance=1.0, lengthscales=1.0, jitter=1e-6):
    K = kernel_matrix(Z, Z, kind, variance, lengthscales)
    return K + jitter * np.eye(Z.shape[0])


def elbo_from_stats(Sigma, v, yy, N, Kuu, noise_variance, variance):
    """ELBO (and the pieces the predictive mean needs) from the statistics."""
    L = np.linalg.cholesky(Kuu)
    tmp = _tri_solve(L, Sigma)                       # L^-1 Sigma
    AAT = _tri_solve(L, tmp.T).T / noise_variance    # L^-1 Sigma L^-T / s2
    AAT = 0.5 * (AAT + AAT.T)
    B = np.eye(Kuu.shape[0]) + AAT
    LB = np.linalg.cholesky(B)
    c = _tri_solve(LB, _tri_solve(L, v)) / noise_variance
    trKff = N * variance                             # stationary kernels
    bound = (-0.5 * N * LOG2PI - np.sum(np.log(np.diag(LB)))
             - 0.5 * N * math.log(noise_variance) - 0.5 * yy / noise_variance
             + 0.5 * float(c @ c) - 0.5 * trKff / noise_variance
             + 0.5 * float(np.trace(AAT)))
    w = _tri_solve(L, _tri_solve(LB, c, trans=True), trans=True)
    return float(bound), w


def elbo(X, y, Z, kind="rbf", variance=1.0, lengthscales=1.0,
         noise_variance=0.01, jitter=1e-6):
    """Sigma-first fp64 ELBO; returns (elbo, w)."""
    Sigma, v, yy = sufficient_stats(X, y, Z, kind, variance, lengthscales)
    K = kuu(Z, kind, variance, lengthscales, jitter)
    return elbo_from_stats(Sigma, v, yy, X.shape[0], K, noise_variance, variance)


def elbo_afirst(X, y, Z, kind="rbf", variance=1.0, lengthscales=1.0,
                noise_variance=0.01, jitter=1e-6):
    """GPflow's own operation order (A = L^-1 Kuf / sigma first)."""
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64).reshape(-1)
    N = X.shape[0]
    L = np.linalg.cholesky(kuu(Z, kind, variance, lengthscales, jitter))
    sigma = math.sqrt(noise_variance)
    A = _tri_solve(L, kernel_matrix(Z, X, kind, variance, lengthscales)) / sigma
    AAT = A @ A.T
    LB = np.linalg.cholesky(np.eye(Z.shape[0]) + AAT)
    c = _tri_solve(LB, A @ y) / sigma
    bound = (-0.5 * N * LOG2PI - np.sum(np.log(np.diag(LB)))
             - 0.5 * N * math.log(noise_variance)
             - 0.5 * float(y @ y) / noise_variance + 0.5 * float(c @ c)
             - 0.5 * N * variance / noise_variance + 0.5 * float(np.trace(AAT)))
    return float(bound)


def predict_mean(Xnew, Z, w, kind="rbf", variance=1.0, lengthscales=1.0):
    return kernel_matrix(Xnew, Z, kind, variance, lengthscales) @ w


def exact_log_marginal(X, y, kind="rbf", variance=1.0, lengthscales=1.0,
                       noise_variance=0.01):
    X = np.asarray(X, np.float64)
    y = np.asarray(y, np.float64).reshape(-1)
    K = kernel_matrix(X, X, kind, variance, lengthscales)
    K += noise_variance * np.eye(X.shape[0])
    L = np.linalg.cholesky(K)
    a = _tri_solve(L, y)
    return float(-0.5 * a @ a - np.sum(np.log(np.diag(L)))
                 - 0.5 * X.shape[0] * LOG2PI)


def elbo_grads_fd(X, y, Z, kind="rbf", variance=1.0, lengthscales=1.0,
                  noise_variance=0.01, jitter=1e-6, rel_step=1e-5):
    """Central finite differences of the fp64 ELBO (``elbo`` above) w.r.t.
    the kernel variance, each lengthscale (ARD), the noise variance and every
    inducing-point coordinate: the oracle for the GPU gradient (GPflow's
    training loss is -ELBO).  O(h^2) truncation, h = rel_step * |param|."""
    Z = np.asarray(Z, np.float64)
    ls = np.broadcast_to(np.asarray(lengthscales, np.float64), (Z.shape[1],)).copy()

    def f(var, lsv, noise, Zv):
        return elbo(X, y, Zv, kind, var, lsv, noise, jitter)[0]

    def cd(fn, x0):
        h = rel_step * max(abs(x0), 1e-3)
        return (fn(x0 + h) - fn(x0 - h)) / (2 * h)

    g = {"variance": cd(lambda t: f(t, ls, noise_variance, Z), variance),
         "noise_variance": cd(lambda t: f(variance, ls, t, Z), noise_variance)}
    gl = np.empty_like(ls)
    for t in range(ls.size):
        def fl(val, t=t):
            l2 = ls.copy()
            l2[t] = val
            return f(variance, l2, noise_variance, Z)
        gl[t] = cd(fl, ls[t])
    g["lengthscales"] = gl
    gz = np.empty_like(Z)
    for i in range(Z.shape[0]):
        for t in range(Z.shape[1]):
            def fz(val, i=i, t=t):
                Z2 = Z.copy()
                Z2[i, t] = val
                return f(variance, ls, noise_variance, Z2)
            gz[i, t] = cd(fz, Z[i, t])
    g["Z"] = gz
    return g
