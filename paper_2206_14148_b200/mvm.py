"""Kernel matrix-vector products on B200 (paper §5.1; SGPR predictive mean).

``se_kernel_mvm`` is the reference's ``build_kernel_mvm`` workload
(/root/reference/pkg/src/tensorbudget/frontend.py:34-54): out = K v with
K[i,j] = variance * exp(-(x_i - y_j)^2 / (2 l^2)) over 1-D inputs.  The
reference must split the n x n matrix into row chunks under its threshold
(8 TB at n = 1e6); here K is never formed — the fused
kernel streams Z tiles through shared memory and accumulates in fp64.
``kernel_mvm`` is the d-dimensional RBF / Matérn-3/2 generalisation used by
``sgpr_predict_mean``.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .errors import EvaluationError


def _torch():
    import torch
    return torch


def _as_lengthscales(lengthscales, dim):
    ls = np.ascontiguousarray(np.broadcast_to(np.asarray(lengthscales, np.float64), (dim,)))
    if np.any(ls <= 0):
        raise ValueError("lengthscales must be strictly positive")
    return ls


def kernel_mvm(X, Z, w, kind: str = "rbf", variance: float = 1.0, lengthscales=1.0,
               stream=None):
    """out[i] = sum_j k(X_i, Z_j) w_j (fp64 accumulation).

    X[n, dim], Z[M, dim] share a dtype (f32/f64); w[M] is used in fp64.
    numpy in -> numpy out; CUDA tensors in -> CUDA fp64 tensor out.
    """
    torch = _torch()
    if kind not in _lib.KERNELS:
        raise ValueError(f"kernel must be one of {tuple(_lib.KERNELS)}")
    if variance <= 0:
        raise ValueError("variance must be strictly positive")
    host = isinstance(X, np.ndarray)
    if host:
        dev = torch.device("cuda")
        Xt = torch.from_numpy(np.ascontiguousarray(X)).to(dev)
        Zt = torch.from_numpy(np.ascontiguousarray(Z)).to(dev)
        wt = torch.from_numpy(np.ascontiguousarray(np.asarray(w, np.float64))).to(dev)
    else:
        Xt, Zt = X.contiguous(), Z.contiguous()
        wt = w.to(torch.float64).contiguous()
        dev = Xt.device
    if Xt.ndim != 2 or Zt.ndim != 2 or Xt.shape[1] != Zt.shape[1]:
        raise EvaluationError("X[n,dim] and Z[M,dim] must share the feature dim")
    if Xt.dtype != Zt.dtype or Xt.dtype not in (torch.float32, torch.float64):
        raise EvaluationError("X and Z must share an f32/f64 dtype")
    if wt.numel() != Zt.shape[0]:
        raise EvaluationError("w must have one entry per row of Z")
    n, dim = int(Xt.shape[0]), int(Xt.shape[1])
    M = int(Zt.shape[0])
    ls = _as_lengthscales(lengthscales, dim)
    out = torch.empty(n, dtype=torch.float64, device=dev)
    st = stream if stream is not None else torch.cuda.current_stream(dev)
    rc = _lib.load().tb_kernel_mvm(
        Xt.data_ptr(), Zt.data_ptr(), wt.data_ptr(), n, M, dim, _lib.KERNELS[kind],
        _lib.TB_F32 if Xt.dtype == torch.float32 else _lib.TB_F64, float(variance),
        ls.ctypes.data_as(ctypes.c_void_p), out.data_ptr(), st.cuda_stream)
    _lib.check(rc, "kernel_mvm")
    return out.cpu().numpy() if host else out


def se_kernel_mvm(x, y, v, variance: float = 1.0, lengthscale: float = 1.0):
    """The reference's SE kernel MVM over 1-D inputs (frontend.py:34-54)."""
    x2 = x.reshape(-1, 1)
    y2 = y.reshape(-1, 1)
    return kernel_mvm(x2, y2, v, "rbf", variance, lengthscale)
