"""Sparse GP regression (Titsias ELBO + predictive mean) on B200.

The paper's §5.3 workload (GPflow 2.3.1 ``SGPR`` with
eXLA splitting).  The reference package has no SGPR code;
this module follows GPflow 2.3.1 ``SGPR.elbo`` / ``SGPR.predict_f`` (zero
mean function, one output, ``default_jitter() = 1e-6``) in the Sigma-first
order: the N-streaming sufficient statistics Sigma = Kuf Kuf^T, v = Kuf y,
yy = y^T y come from the CUDA library (``tb_sgpr_stats_run``, fused Kuf tile
generation + exact fp64 Gram, never materialising the M x N matrix beyond one
planner-sized chunk), the O(M^3) tail runs in fp64 on cuSOLVER via
torch.linalg, and the predictive mean is the fused kernel MVM K(X*, Z) w.

Multi-GPU: each rank passes its own rows of (X, y); the statistics are
summed with one NCCL ``all_reduce`` before the (redundant, per-rank) tail.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BudgetExceeded, EvaluationError
from .mvm import _as_lengthscales
from .sizes import as_limit

LOG2PI = math.log(2.0 * math.pi)


def _alloc_bytes(b: int) -> int:
    """What the caching allocator charges for one b-byte buffer (512-B
    granules up to 1 MiB, 2 MiB above; tb_common.cuh alloc_bytes)."""
    return -(-b // 512) * 512 if b <= (1 << 20) else -(-b // (2 << 20)) * (2 << 20)


def _torch():
    import torch
    return torch


def _dev_tensor(a, device):
    torch = _torch()
    if isinstance(a, np.ndarray):
        return torch.from_numpy(np.ascontiguousarray(a)).to(device)
    return a.to(device).contiguous()


# cond(Kuu) lower bound (max/min of the packed tail's diag(L)^2) above which
# engine "auto" recomputes the statistics in fp64 when the dense tail fits
# the limit: the fixed-point statistics move the predictive mean by ~cond(Kuu)
# x 2e-12 (5e-4 seen at cond 2.8e8), and the diag bound under-reads cond(Kuu)
# by up to ~250x on smooth kernels (fuzz: 8.6e5 for 2.1e8)
COND_FP64 = 1e5


def plan(N: int, M: int, dim: int, *, kernel: str = "rbf", dtype=np.float32,
         memory_limit=None, resident_bytes: int | None = None,
         engine: str = "auto") -> _lib.SgprPlan:
    """Planner only (CPU): chunk of training points so that resident inputs +
    Sigma/v + workspace fit ``memory_limit``.  ``engine``: "i8" (exact Gram of
    the 24-bit fixed-point Kuf on the INT8 tensor cores; default), "f64"
    (fp64 DMMA) or "f64_simt" (fp64 CUDA cores)."""
    if kernel not in _lib.KERNELS:
        raise ValueError(f"kernel must be one of {tuple(_lib.KERNELS)}")
    if engine not in _lib.SGPR_ENGINES:
        raise ValueError(f"engine must be one of {tuple(_lib.SGPR_ENGINES)}")
    es = np.dtype(dtype).itemsize
    if resident_bytes is None:
        resident_bytes = (N * dim + N + M * dim) * es
    p = _lib.SgprPlan()
    rc = _lib.load().tb_sgpr_plan_create(N, M, dim, _lib.KERNELS[kernel],
                                         _lib.TB_F32 if np.dtype(dtype) == np.float32 else _lib.TB_F64,
                                         _lib.SGPR_ENGINES[engine], as_limit(memory_limit),
                                         resident_bytes, ctypes.byref(p))
    _lib.check(rc, f"sgpr_N{N}_M{M}_d{dim}", live=resident_bytes)
    return p


def kernel_matrix(A, B, kind="rbf", variance=1.0, lengthscales=1.0, stream=None):
    """fp64 K(A, B) on the device (same kernel code as the statistics)."""
    torch = _torch()
    dim = int(A.shape[1])
    ls = _as_lengthscales(lengthscales, dim)
    out = torch.empty((int(A.shape[0]), int(B.shape[0])), dtype=torch.float64, device=A.device)
    st = stream if stream is not None else torch.cuda.current_stream(A.device)
    rc = _lib.load().tb_kernel_matrix(
        A.data_ptr(), B.data_ptr(), int(A.shape[0]), int(B.shape[0]), dim, _lib.KERNELS[kind],
        _lib.TB_F32 if A.dtype == torch.float32 else _lib.TB_F64, float(variance),
        ls.ctypes.data_as(ctypes.c_void_p), out.data_ptr(), st.cuda_stream)
    _lib.check(rc, "kernel_matrix")
    return out


@dataclass
class SgprStats:
    Sigma: object    # torch fp64, in plan.sigma_layout (full [M, M] or packed lower tiles)
    v: object        # torch fp64 [M]
    yy: float
    N: int
    plan: _lib.SgprPlan

    def full_sigma(self, stream=None):
        """Sigma as the full symmetric [M, M] fp64 matrix (tail input)."""
        torch = _torch()
        if self.plan.sigma_layout == _lib.TB_SIGMA_FULL:
            return self.Sigma
        M = self.v.numel()
        out = torch.empty((M, M), dtype=torch.float64, device=self.Sigma.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.Sigma.device)
        rc = _lib.load().tb_sgpr_sigma_unpack(ctypes.byref(self.plan), self.Sigma.data_ptr(),
                                              out.data_ptr(), st.cuda_stream)
        _lib.check(rc, "sgpr_sigma_unpack")
        return out


class SGPR:
    """GPflow-2.3.1-compatible SGPR on B200 (zero mean, single output).

    X[N, dim], y[N] (or [N, 1]), Z[M, dim]: numpy arrays or CUDA tensors (f32
    or f64, shared dtype).  ``memory_limit`` bounds the statistics pass
    (inputs + Sigma + v + workspace).  With ``group`` set, X/y are this
    rank's shard and the statistics are all-reduced over the group.
    """

    def __init__(self, X, y, Z, kernel: str = "rbf", variance: float = 1.0,
                 lengthscales=1.0, noise_variance: float = 0.01, jitter: float = 1e-6,
                 memory_limit=None, group=None, device=None, engine: str = "auto",
                 tail: str = "packed"):
        torch = _torch()
        if kernel not in _lib.KERNELS:
            raise ValueError(f"kernel must be one of {tuple(_lib.KERNELS)}")
        if variance <= 0 or noise_variance <= 0 or jitter < 0:
            raise ValueError("variance and noise_variance must be positive, jitter >= 0")
        self.device = torch.device(device or "cuda")
        self.X = _dev_tensor(X, self.device)
        self.y = _dev_tensor(y, self.device).reshape(-1)
        self.Z = _dev_tensor(Z, self.device)
        if self.X.ndim != 2 or self.Z.ndim != 2 or self.X.shape[1] != self.Z.shape[1]:
            raise EvaluationError("X[N,dim] and Z[M,dim] must share the feature dim")
        if self.y.numel() != self.X.shape[0]:
            raise EvaluationError("y must have one entry per row of X")
        if not (self.X.dtype == self.Z.dtype == self.y.dtype) or \
                self.X.dtype not in (torch.float32, torch.float64):
            raise EvaluationError("X, y, Z must share an f32/f64 dtype")
        self.kernel = kernel
        self.variance = float(variance)
        self.dim = int(self.X.shape[1])
        self.lengthscales = _as_lengthscales(lengthscales, self.dim)
        self.noise_variance = float(noise_variance)
        self.jitter = float(jitter)
        self.memory_limit = memory_limit
        self.group = group
        if engine not in _lib.SGPR_ENGINES:
            raise ValueError(f"engine must be one of {tuple(_lib.SGPR_ENGINES)}")
        self.engine = engine
        if tail not in ("packed", "dense"):
            raise ValueError("tail must be 'packed' or 'dense'")
        self.tail = tail          # packed: in place on the fixed-point engine's tiles
        self._stats = None
        self._w = None
        self.cond_kuu_lb = None   # set by the packed tail: max/min diag(L)^2

    # -- hot path -----------------------------------------------------------
    def statistics(self, stream=None) -> SgprStats:
        torch = _torch()
        N, dim = int(self.X.shape[0]), self.dim
        M = int(self.Z.shape[0])
        es = self.X.element_size()
        p = plan(N, M, dim, kernel=self.kernel,
                 dtype=np.float32 if self.X.dtype == torch.float32 else np.float64,
                 memory_limit=self.memory_limit,
                 resident_bytes=(N * dim + N + M * dim) * es, engine=self.engine)
        Sigma = torch.empty(int(p.sigma_bytes) // 8, dtype=torch.float64, device=self.device)
        if p.sigma_layout == _lib.TB_SIGMA_FULL:
            Sigma = Sigma.view(M, M)
        v = torch.empty(M, dtype=torch.float64, device=self.device)
        yy = torch.empty(1, dtype=torch.float64, device=self.device)
        ws = torch.empty(max(int(p.workspace_bytes), 1), dtype=torch.uint8, device=self.device)
        st = stream if stream is not None else torch.cuda.current_stream(self.device)
        rc = _lib.load().tb_sgpr_stats_run(
            ctypes.byref(p), self.X.data_ptr(), self.y.data_ptr(), self.Z.data_ptr(),
            self.variance, self.lengthscales.ctypes.data_as(ctypes.c_void_p),
            Sigma.data_ptr(), v.data_ptr(), yy.data_ptr(), 0, ws.data_ptr(), ws.numel(),
            st.cuda_stream)
        _lib.check(rc, "sgpr_stats")
        del ws
        n_total, yy_total = N, float(yy.item())
        if self.group is not None:
            from .distributed import allreduce_statistics
            Sigma, v, yy_total, n_total = allreduce_statistics(Sigma, v, yy, N, self.group)
        self._stats = SgprStats(Sigma, v, yy_total, n_total, p)
        return self._stats

    # -- O(M^3) tail --------------------------------------------------------
    def _tail(self):
        s = self._stats if self._stats is not None and self._stats.Sigma is not None \
            else self.statistics()
        if s.plan.sigma_layout == _lib.TB_SIGMA_TILES and self.tail == "packed":
            try:
                bound = self._tail_packed(s)
                # well conditioned (the usual case): done.  Otherwise the 2^-25
                # rounding of Kuf, amplified by cond(A), can move the
                # predictive weights past 1e-4: engine "auto" redoes the
                # statistics in fp64 when the dense tail fits the limit
                if not (self.engine == "auto" and self.cond_kuu_lb > COND_FP64
                        and self._dense_tail_fits()):
                    return bound
                self._refit_ill_conditioned()
                s = self.statistics()
            except EvaluationError as ex:
                # The packed tail factors A = Kuu + Sigma/s2 itself, whose
                # condition number is about cond(Kuu) cond(B); the dense tail
                # factors GPflow's B = I + L^-1 Sigma L^-T / s2 (>= I).  With
                # cond(A) ~ 1e14 (long lengthscales, dense inducing points)
                # the blocked packed factorisation can meet a negative pivot
                # where LAPACK-style cuSOLVER on B does not: recompute the
                # statistics (the packed tail consumed them) and take the
                # dense tail when it fits the limit, else re-raise.
                if "not positive definite" not in str(ex) or not self._dense_tail_fits():
                    raise
                self._refit_ill_conditioned()
                s = self.statistics()
        return self._tail_dense(s)

    def _dense_grad_fits(self, chunk_n: int) -> bool:
        """Whether the dense gradient path fits memory_limit."""
        if self.memory_limit is None:
            return True
        from .sizes import as_limit
        M = int(self.Z.shape[0])
        resident = (self.X.numel() + self.y.numel() + self.Z.numel()) * self.X.element_size()
        return grad_memory_bytes(M, self.dim, chunk_n) + resident <= as_limit(self.memory_limit)

    def _refit_ill_conditioned(self):
        """After the packed factorisation failed: drop the consumed
        statistics and, for engine "auto", recompute them in fp64 (at cond(A)
        ~ 1e14 the 24-bit fixed-point rounding of Kuf, exact as it is, moves
        the ELBO by ~1e-4); an explicitly chosen engine is kept."""
        self._stats = None
        if self.engine == "auto":
            self.engine = "f64"

    def _dense_tail_fits(self) -> bool:
        """Whether the dense tail (full Sigma + ~5 M x M fp64 work matrices
        beside the packed statistics and the inputs) fits memory_limit."""
        if self.memory_limit is None:
            return True
        from .sizes import as_limit
        limit = as_limit(self.memory_limit)
        M = int(self.Z.shape[0])
        engine = "f64" if self.engine == "auto" else self.engine     # as _refit_ill_conditioned
        inputs = sum(int(t.numel()) * t.element_size() for t in (self.X, self.y, self.Z))
        try:
            stats = int(plan(int(self.X.shape[0]), M, self.dim, kernel=self.kernel,
                             memory_limit=self.memory_limit, resident_bytes=inputs,
                             engine=engine).sigma_bytes)
        except BudgetExceeded:
            return False
        return inputs + stats + 6 * 8 * M * M + (8 << 20) <= limit

    def _tail_packed(self, s):
        """In place on the packed tiles (tb_sgpr_tail_run): the evaluation
        never holds more than the packed Sigma + one packed factor, so the
        whole ELBO stays inside memory_limit.  Consumes the statistics."""
        torch = _torch()
        lib = _lib.load()
        p = s.plan
        M = s.v.numel()
        ws = torch.empty(max(int(lib.tb_sgpr_tail_workspace(ctypes.byref(p))), 1),
                         dtype=torch.uint8, device=self.device)
        w = torch.empty(M, dtype=torch.float64, device=self.device)
        out = torch.empty(6, dtype=torch.float64, device=self.device)
        st = torch.cuda.current_stream(self.device)
        rc = lib.tb_sgpr_tail_run(ctypes.byref(p), self.Z.data_ptr(), self.variance,
                                  self.lengthscales.ctypes.data_as(ctypes.c_void_p), self.jitter,
                                  self.noise_variance, s.Sigma.data_ptr(), s.v.data_ptr(),
                                  w.data_ptr(), out.data_ptr(), ws.data_ptr(), ws.numel(),
                                  st.cuda_stream)
        s.Sigma = None                     # overwritten by the in-place factorisation
        _lib.check(rc, "sgpr_tail")
        del ws
        logdet_l, logdet_p, uu, xx, dmin, dmax = (float(t) for t in out.tolist())
        # max/min of diag(L)^2 bounds cond(Kuu) from below
        self.cond_kuu_lb = dmax / dmin if dmin > 0 else math.inf
        s2, N = self.noise_variance, s.N
        bound = (-0.5 * N * LOG2PI - (logdet_p - logdet_l) - 0.5 * N * math.log(s2)
                 - 0.5 * s.yy / s2 + 0.5 * uu / (s2 * s2) - 0.5 * N * self.variance / s2
                 + 0.5 * (xx - int(p.M_pad)))
        self._w = w
        return bound

    def _tail_dense(self, s):
        """cuSOLVER / cuBLAS through torch.linalg on full fp64 matrices."""
        torch = _torch()
        M = s.v.numel()
        s2 = self.noise_variance
        Kuu = kernel_matrix(self.Z, self.Z, self.kernel, self.variance, self.lengthscales)
        Kuu.diagonal().add_(self.jitter)
        L = torch.linalg.cholesky(Kuu)
        del Kuu
        Sigma = s.full_sigma()
        tmp = torch.linalg.solve_triangular(L, Sigma, upper=False)            # L^-1 Sigma
        del Sigma
        AAT = torch.linalg.solve_triangular(L, tmp.mT, upper=False).mT          # L^-1 Sigma L^-T
        del tmp
        AAT = 0.5 * (AAT + AAT.mT) / s2
        trAAT = float(AAT.diagonal().sum().item())
        AAT.diagonal().add_(1.0)
        LB = torch.linalg.cholesky(AAT)
        del AAT
        Lv = torch.linalg.solve_triangular(L, s.v.reshape(M, 1), upper=False)
        c = torch.linalg.solve_triangular(LB, Lv, upper=False) / s2
        N = s.N
        bound = (-0.5 * N * LOG2PI - float(torch.log(LB.diagonal()).sum().item())
                 - 0.5 * N * math.log(s2) - 0.5 * s.yy / s2 + 0.5 * float((c * c).sum().item())
                 - 0.5 * N * self.variance / s2 + 0.5 * trAAT)
        t = torch.linalg.solve_triangular(LB.mT, c, upper=True)
        w = torch.linalg.solve_triangular(L.mT, t, upper=True).reshape(M)
        self._w = w
        return bound

    def elbo(self) -> float:
        return self._tail()

    # -- gradient (GPflow 2.3.1 SGPR training loss; paper §5.3 Table 2) -------
    def grad_peak_bytes(self) -> int:
        """Device bytes of elbo_and_grads on the packed path (inputs included):
        the larger of the statistics pass's plan and the gradient tail (the
        packed statistics + two column panels of vectors + its workspace)."""
        torch = _torch()
        N, M = int(self.X.shape[0]), int(self.Z.shape[0])
        es = self.X.element_size()
        p = plan(N, M, self.dim, kernel=self.kernel,
                 dtype=np.float32 if self.X.dtype == torch.float32 else np.float64,
                 memory_limit=self.memory_limit,
                 resident_bytes=(N * self.dim + N + M * self.dim) * es, engine=self.engine)
        if p.sigma_layout != _lib.TB_SIGMA_TILES:
            return -1
        lib = _lib.load()
        ab = _alloc_bytes
        resident = sum(ab(t.numel() * t.element_size()) for t in (self.X, self.y, self.Z))
        tail = (resident + ab(int(p.sigma_bytes)) + ab(M * 8) + ab(8)
                + ab(int(lib.tb_sgpr_grad_workspace(ctypes.byref(p))))
                + ab(8 * 8) + ab(2 * (1 + self.dim) * 8) + ab(2 * M * self.dim * 8))
        return max(int(p.peak_bytes), tail)

    def elbo_and_grads(self, chunk_n: int = 4096):
        """ELBO and its gradient w.r.t. kernel variance, lengthscales (ARD),
        likelihood noise variance and the inducing points Z (the quantities
        GPflow trains; values are w.r.t. the constrained parameters).

        With the packed statistics (engine "i8", the default) and tail
        "packed", the gradient runs inside memory_limit through
        ``tb_sgpr_grad_run`` (``_elbo_and_grads_packed``); otherwise the dense
        path below (fp64 engines, or tail="dense").

        The O(M^3) tail is differentiated analytically on dense fp64
        matrices (cuSOLVER Cholesky / inverse, cuBLAS; at most ~4 M x M live):
        with A = Kuu + Sigma / s2 and w = A^-1 v / s2, G = dELBO/dSigma =
        (Kuu^-1 - A^-1 - w w^T) / (2 s2), g = dELBO/dv = w / s2,
        dELBO/dKuu = s2 G - Kuu^-1 Sigma Kuu^-1 / (2 s2), plus the explicit
        noise and variance terms; dELBO/dKuu is contracted with the kernel
        derivatives by ``tb_sgpr_kuf_grad`` over Z x Z.  The data then enter only through
        W = 2 G Kuf + g y^T, streamed over N in chunks: W by one fp64 GEMM
        (cuBLAS) and the reduction against the kernel derivatives by the
        fused kernel ``tb_sgpr_kuf_grad``.  Multi-GPU: the chunk sums are
        all-reduced like the statistics.  Returns (elbo, dict of gradients)."""
        torch = _torch()
        M, dim = int(self.Z.shape[0]), self.dim
        if self.tail == "packed" and dim <= 16 and self.grad_peak_bytes() >= 0:
            try:
                res = self._elbo_and_grads_packed()
                # as in _tail: engine "auto" redoes an ill-conditioned problem
                # from fp64 statistics when the dense path fits the limit
                if not (self.engine == "auto" and self.cond_kuu_lb > COND_FP64
                        and self._dense_grad_fits(chunk_n)):
                    return res
                self._refit_ill_conditioned()
            except EvaluationError as ex:
                # as in _tail: a negative pivot of the packed factorisation
                # of A on a very ill-conditioned problem -> the dense path
                # below (GPflow's formulation), if it fits; the packed path
                # consumed the statistics, which are recomputed
                if "not positive definite" not in str(ex):
                    raise
                self._refit_ill_conditioned()
        if self.memory_limit is not None:
            limit = as_limit(self.memory_limit)
            resident = (self.X.numel() + self.y.numel() + self.Z.numel()) * self.X.element_size()
            need = grad_memory_bytes(M, dim, chunk_n) + resident
            if need > limit:
                raise BudgetExceeded(
                    "sgpr_elbo_and_grads", need, resident,
                    message=f"sgpr_elbo_and_grads: the dense fp64 gradient tail needs "
                            f"~{need / 1e9:.2f} GB at M={M} (N-independent), over "
                            f"memory_limit={limit}; the ELBO alone (elbo()) stays in budget")
        s = self._stats if self._stats is not None and self._stats.Sigma is not None \
            else self.statistics()
        f64 = torch.float64
        dev = self.device
        N, s2, var = float(s.N), self.noise_variance, self.variance
        lib = _lib.load()
        st = torch.cuda.current_stream(dev)
        dt = _lib.TB_F32 if self.X.dtype == torch.float32 else _lib.TB_F64
        lsp = self.lengthscales.ctypes.data_as(ctypes.c_void_p)
        # --- the O(M^3) tail, differentiated analytically (A = Kuu + Sigma/s2,
        # w = A^-1 v / s2), dense fp64, in place
        Sig = s.full_sigma()
        v = s.v
        Kuu = kernel_matrix(self.Z, self.Z, self.kernel, var, self.lengthscales)
        Kuu.diagonal().add_(self.jitter)
        L = torch.linalg.cholesky(Kuu)
        Kuu.add_(Sig, alpha=1.0 / s2)                          # A, in place
        P = torch.linalg.cholesky(Kuu)
        del Kuu
        logdet_k = 2.0 * float(torch.log(L.diagonal()).sum())
        logdet_a = 2.0 * float(torch.log(P.diagonal()).sum())
        Kinv = torch.cholesky_inverse(L)
        del L
        Ainv = torch.cholesky_inverse(P)
        del P
        w = Ainv @ v / s2
        vw = float(v @ w)                                      # v^T A^-1 v / s2
        tr_ks = float((Kinv * Sig).sum())                      # tr(Kuu^-1 Sigma)
        tr_as = float((Ainv * Sig).sum())                      # tr(A^-1 Sigma)
        wsw = float(w @ (Sig @ w))
        elbo = (-0.5 * N * LOG2PI - 0.5 * (logdet_a - logdet_k) - 0.5 * N * math.log(s2)
                - 0.5 * s.yy / s2 + 0.5 * vw / s2 - 0.5 * N * var / s2 + 0.5 * tr_ks / s2)
        d_s2 = (0.5 * tr_as / s2**2 + 0.5 * wsw / s2**2 - vw / s2**2 - 0.5 * N / s2
                + 0.5 * s.yy / s2**2 + 0.5 * N * var / s2**2 - 0.5 * tr_ks / s2**2)
        T = Kinv @ Sig
        del Sig
        H = T @ Kinv                                           # Kuu^-1 Sigma Kuu^-1
        del T
        Gm = Kinv.sub_(Ainv).addr_(w, w, alpha=-1.0)           # Kuu^-1 - A^-1 - w w^T
        del Ainv
        # dELBO/dKuu = Gm / 2 - Kuu^-1 Sigma Kuu^-1 / (2 s2)
        H.mul_(-0.5 / s2).add_(Gm, alpha=0.5)
        g = w / s2                                             # dELBO/dv
        G2 = Gm.div_(s2)                                       # 2 G, G = dELBO/dSigma
        # --- Kuu side: sum_ij H_ij dk(z_i, z_j) (both arguments for Z)
        grad_hyp_k = torch.zeros(1 + dim, dtype=f64, device=dev)
        grad_z_k = torch.zeros((M, dim), dtype=f64, device=dev)
        K0 = kernel_matrix(self.Z, self.Z, self.kernel, var, self.lengthscales)
        H.mul_(2.0)
        wsk = torch.empty(max(int(lib.tb_sgpr_kuf_grad_workspace(M, M, dim)), 1),
                          dtype=torch.uint8, device=dev)
        rc = lib.tb_sgpr_kuf_grad(self.Z.data_ptr(), self.Z.data_ptr(), H.data_ptr(),
                                  K0.data_ptr(), M, M, dim, _lib.KERNELS[self.kernel], dt, var,
                                  lsp, grad_hyp_k.data_ptr(), grad_z_k.data_ptr(), wsk.data_ptr(),
                                  wsk.numel(), st.cuda_stream)
        _lib.check(rc, "sgpr_kuf_grad(Kuu)")
        del H, K0, wsk
        grad_hyp_k.mul_(0.5)                                   # W = 2H doubled the hyp sums
        # --- data side, streamed over N: W = 2 G Kuf + g y^T
        grad_hyp = torch.zeros(1 + dim, dtype=f64, device=dev)
        grad_z = torch.zeros((M, dim), dtype=f64, device=dev)
        ws = torch.empty(max(int(lib.tb_sgpr_kuf_grad_workspace(chunk_n, M, dim)), 1),
                         dtype=torch.uint8, device=dev)
        for n0 in range(0, int(self.X.shape[0]), chunk_n):
            Xc = self.X[n0:n0 + chunk_n].contiguous()
            yc = self.y[n0:n0 + chunk_n].to(f64)
            K = kernel_matrix(self.Z, Xc, self.kernel, var, self.lengthscales)
            W = torch.addr(G2 @ K, g, yc)                   # 2 G K + g y^T
            rc = lib.tb_sgpr_kuf_grad(
                Xc.data_ptr(), self.Z.data_ptr(), W.data_ptr(), K.data_ptr(), int(Xc.shape[0]),
                M, dim, _lib.KERNELS[self.kernel], dt, var, lsp, grad_hyp.data_ptr(),
                grad_z.data_ptr(), ws.data_ptr(), ws.numel(), st.cuda_stream)
            _lib.check(rc, "sgpr_kuf_grad")
        if self.group is not None:
            import torch.distributed as dist
            dist.all_reduce(grad_hyp, group=self.group)
            dist.all_reduce(grad_z, group=self.group)
        grad_hyp += grad_hyp_k
        grad_z += grad_z_k
        grads = {"variance": -0.5 * N / s2 + float(grad_hyp[0]),
                 "lengthscales": grad_hyp[1:].cpu().numpy(),
                 "noise_variance": d_s2,
                 "Z": grad_z.cpu().numpy()}
        return float(elbo), grads

    def _elbo_and_grads_packed(self):
        """tb_sgpr_grad_run: only the packed factors L = chol(Kuu) and
        P = chol(Kuu + Sigma/s2) stay resident; 2 dELBO/dKuu and
        2 dELBO/dSigma are produced and consumed one 128-column panel at a
        time (DESIGN.md §4 "Gradient").  Consumes the statistics."""
        torch = _torch()
        M, dim = int(self.Z.shape[0]), self.dim
        if self.memory_limit is not None:
            limit = as_limit(self.memory_limit)
            need = self.grad_peak_bytes()
            if need > limit:
                resident = (self.X.numel() + self.y.numel() + self.Z.numel()) * \
                    self.X.element_size()
                raise BudgetExceeded(
                    "sgpr_elbo_and_grads", need, resident,
                    message=f"sgpr_elbo_and_grads: needs {need} bytes on the device "
                            f"(memory_limit={limit})")
        s = self._stats if self._stats is not None and self._stats.Sigma is not None \
            else self.statistics()
        p = s.plan
        f64 = torch.float64
        dev = self.device
        lib = _lib.load()
        st = torch.cuda.current_stream(dev)
        wsb = int(lib.tb_sgpr_grad_workspace(ctypes.byref(p)))
        ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
        out8 = torch.zeros(8, dtype=f64, device=dev)
        gh = torch.zeros(2 * (1 + dim), dtype=f64, device=dev)
        gz = torch.zeros(2 * M * dim, dtype=f64, device=dev)
        rc = lib.tb_sgpr_grad_run(ctypes.byref(p), self.X.data_ptr(), self.y.data_ptr(),
                                  self.Z.data_ptr(), self.variance,
                                  self.lengthscales.ctypes.data_as(ctypes.c_void_p), self.jitter,
                                  self.noise_variance, s.Sigma.data_ptr(), s.v.data_ptr(),
                                  out8.data_ptr(), gh.data_ptr(), gz.data_ptr(), ws.data_ptr(),
                                  ws.numel(), st.cuda_stream)
        s.Sigma = None                         # overwritten by the factor P
        self._w = None
        _lib.check(rc, "sgpr_grad_run")
        del ws
        if self.group is not None:             # data-side sums over the ranks' rows
            import torch.distributed as dist
            dist.all_reduce(gh[:1 + dim], group=self.group)
            dist.all_reduce(gz[:M * dim], group=self.group)
        sl, sp, uu, tr_ka, tr_ak, wkw, dmin, dmax = (float(t) for t in out8.tolist())
        self.cond_kuu_lb = dmax / dmin if dmin > 0 else math.inf
        N, s2, var, yy = float(s.N), self.noise_variance, self.variance, s.yy
        logdet_k, logdet_a = 2.0 * sl, 2.0 * sp
        vw = uu / s2                                 # v^T A^-1 v / s2
        tr_ks = s2 * (tr_ka - M)                     # tr(Kuu^-1 Sigma)
        tr_as = s2 * (M - tr_ak)                     # tr(A^-1 Sigma)
        wsw = vw - s2 * wkw                          # w^T Sigma w
        elbo = (-0.5 * N * LOG2PI - 0.5 * (logdet_a - logdet_k) - 0.5 * N * math.log(s2)
                - 0.5 * yy / s2 + 0.5 * vw / s2 - 0.5 * N * var / s2 + 0.5 * tr_ks / s2)
        d_s2 = (0.5 * tr_as / s2**2 + 0.5 * wsw / s2**2 - vw / s2**2 - 0.5 * N / s2
                + 0.5 * yy / s2**2 + 0.5 * N * var / s2**2 - 0.5 * tr_ks / s2**2)
        hyp = gh[:1 + dim] + 0.5 * gh[1 + dim:]
        gzs = (gz[:M * dim] + gz[M * dim:]).reshape(M, dim)
        grads = {"variance": -0.5 * N / s2 + float(hyp[0]),
                 "lengthscales": hyp[1:].cpu().numpy(),
                 "noise_variance": d_s2,
                 "Z": gzs.cpu().numpy()}
        return float(elbo), grads

    def predict_mean(self, Xnew):
        """mu(X*) = K(X*, Z) L^-T LB^-T c (GPflow predict_f mean)."""
        from .mvm import kernel_mvm
        if self._w is None:
            self._tail()
        host = isinstance(Xnew, np.ndarray)
        Xt = _dev_tensor(Xnew, self.device).to(self.Z.dtype)
        mu = kernel_mvm(Xt, self.Z, self._w, self.kernel, self.variance, self.lengthscales)
        return mu.cpu().numpy() if host else mu


def grad_memory_bytes(M: int, dim: int, chunk_n: int = 4096) -> int:
    """Device bytes SGPR.elbo_and_grads needs beyond its inputs (planner-style
    estimate, checked against torch's peak by tests/test_sgpr_gpu.py).  The
    O(M^3) tail is differentiated analytically on dense fp64 matrices: at
    most ~5 live M x M matrices (Sigma, the two inverses, Kuu^-1 Sigma and
    its product) besides the packed statistics and cuSOLVER workspace
    (measured peak 6.4 M^2 fp64 words; budgeted 7).
    The N-streaming pass then holds G (twice) plus three M x chunk_n fp64
    panels (K, G K, W) and the reduction partials.  Independent of N."""
    mm = 8 * M * M
    tail = 7 * mm + 8 * (-(-M // 128)) * (M * dim + (1 + dim) * (-(-M // 32)))
    stream = 2 * mm + 3 * 8 * M * chunk_n + 8 * (-(-chunk_n // 128)) * (M * dim + (1 + dim) * (-(-M // 32)))
    return int(max(tail, stream)) + (1 << 20)


def _torch_kernel(A, B, kind, variance, ls):
    """Differentiable fp64 k(A, B) (same formulas as the CUDA kernels;
    r^2 by the expansion to stay O(|A| |B|) in memory)."""
    torch = _torch()
    a, b = A / ls, B / ls
    r2 = ((a * a).sum(1)[:, None] + (b * b).sum(1)[None, :] - 2.0 * (a @ b.mT)).clamp_min(0.0)
    if kind == "rbf":
        return variance * torch.exp(-0.5 * r2)
    r = r2.clamp_min(1e-36).sqrt()
    return variance * (1.0 + math.sqrt(3.0) * r) * torch.exp(-math.sqrt(3.0) * r)


def _elbo_torch(Sigma, v, yy, N, Kuu, s2, variance):
    """Differentiable copy of the tail (SGPR._tail / oracle.sgpr.elbo_from_stats)."""
    torch = _torch()
    M = v.numel()
    L = torch.linalg.cholesky(Kuu)
    tmp = torch.linalg.solve_triangular(L, Sigma, upper=False)
    AAT = torch.linalg.solve_triangular(L, tmp.mT, upper=False).mT / s2
    AAT = 0.5 * (AAT + AAT.mT)
    B = AAT + torch.eye(M, dtype=AAT.dtype, device=AAT.device)
    LB = torch.linalg.cholesky(B)
    Lv = torch.linalg.solve_triangular(L, v.reshape(M, 1), upper=False)
    c = torch.linalg.solve_triangular(LB, Lv, upper=False) / s2
    return (-0.5 * N * LOG2PI - torch.log(LB.diagonal()).sum() - 0.5 * N * torch.log(s2)
            - 0.5 * yy / s2 + 0.5 * (c * c).sum() - 0.5 * N * variance / s2
            + 0.5 * AAT.diagonal().sum())


def sgpr_elbo(X, y, Z, kernel="rbf", variance=1.0, lengthscales=1.0,
              noise_variance=0.01, *, jitter=1e-6, memory_limit=None, group=None,
              engine="auto") -> float:
    """Titsias collapsed ELBO of GPflow 2.3.1 SGPR, on the B200 path."""
    return SGPR(X, y, Z, kernel, variance, lengthscales, noise_variance, jitter,
                memory_limit, group, engine=engine).elbo()


def sgpr_predict_mean(Xnew, X, y, Z, kernel="rbf", variance=1.0, lengthscales=1.0,
                      noise_variance=0.01, *, jitter=1e-6, memory_limit=None, group=None,
                      engine="auto"):
    m = SGPR(X, y, Z, kernel, variance, lengthscales, noise_variance, jitter,
             memory_limit, group, engine=engine)
    return m.predict_mean(Xnew)
