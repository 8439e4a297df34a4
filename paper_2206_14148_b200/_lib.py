"""ctypes binding of the C-ABI library ``libtb_pairwise.so`` (include/tb_pairwise.h).

The library is built in-tree (``__graft_entry__.build()`` /
``make -C paper_2206_14148_b200/csrc``).  There is no CPU fallback: if the
library is missing, or a compute entry point is called without a B200,
the call fails loudly.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .errors import (BudgetExceeded, EvaluationError, KernelUnavailable,
                     UnsplittableCandidate)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtb_pairwise.so")

TB_OK, TB_ERR_ARG, TB_ERR_BUDGET, TB_ERR_UNSPLITTABLE = 0, 1, 2, 3
TB_ERR_CUDA, TB_ERR_UNSUPPORTED, TB_ERR_NO_DEVICE = 4, 5, 6
TB_F32, TB_F64 = 0, 1
METRICS = {"l2": 0, "l1": 1, "cosine": 2}
ENGINES = {"auto": 0, "tc3": 1, "simt": 2, "tc1": 3}
KERNELS = {"rbf": 0, "matern32": 1}
SGPR_ENGINES = {"auto": 0, "i8": 1, "f64": 2, "f64_simt": 3}
TB_SIGMA_FULL, TB_SIGMA_TILES = 0, 1

_i64 = ctypes.c_int64
_i32 = ctypes.c_int32
_vp = ctypes.c_void_p


class KnnPlan(ctypes.Structure):
    _fields_ = [
        ("n", _i64), ("m", _i64), ("d", _i64), ("k", _i64),
        ("metric", _i32), ("dtype", _i32), ("out_dtype", _i32), ("engine", _i32),
        ("memory_limit", _i64), ("resident_bytes", _i64),
        ("cand", _i32), ("slices", _i32),
        ("chunk_rows", _i64), ("n_chunks", _i64), ("d_pad", _i64), ("m_pad", _i64),
        ("workspace_bytes", _i64), ("output_bytes", _i64), ("peak_bytes", _i64),
        ("off", _i64 * 16),
    ]


class SgprPlan(ctypes.Structure):
    _fields_ = [
        ("N", _i64), ("M", _i64), ("dim", _i64),
        ("kernel", _i32), ("dtype", _i32),
        ("memory_limit", _i64), ("resident_bytes", _i64),
        ("engine", _i32), ("sigma_layout", _i32), ("M_pad", _i64), ("sigma_bytes", _i64),
        ("chunk_n", _i64), ("workspace_bytes", _i64), ("output_bytes", _i64),
        ("peak_bytes", _i64), ("off", _i64 * 8),
    ]


_SIGS = {
    "tb_knn_plan_create": (ctypes.c_int, [_i64, _i64, _i64, _i64, _i32, _i32, _i32, _i32,
                                          _i64, _i64, ctypes.POINTER(KnnPlan)]),
    "tb_knn_plan_create_ex": (ctypes.c_int, [_i64, _i64, _i64, _i64, _i32, _i32, _i32, _i32,
                                             _i64, _i64, _i64, ctypes.POINTER(KnnPlan)]),
    "tb_knn_run_host": (ctypes.c_int, [ctypes.POINTER(KnnPlan), _vp, _vp, _i64, _vp, _vp,
                                       _vp, _vp, _vp, _vp, _vp, _i64, _vp]),
    "tb_knn_run": (ctypes.c_int, [ctypes.POINTER(KnnPlan), _vp, _vp, _i64, _vp, _vp,
                                  _vp, _i64, _vp]),
    "tb_knn_run_ex": (ctypes.c_int, [ctypes.POINTER(KnnPlan), _vp, _vp, _i64, _vp, _vp,
                                     _vp, _i64, _vp, ctypes.POINTER(_vp), _i32]),
    "tb_topk_merge": (ctypes.c_int, [_vp, _vp, _i32, _i64, _i64, _i32, _vp, _vp, _vp]),
    "tb_knn_fallback_count": (ctypes.c_int, [ctypes.POINTER(KnnPlan), _vp, _vp,
                                             ctypes.POINTER(_i64)]),
    "tb_knn_check": (ctypes.c_int, [ctypes.POINTER(KnnPlan), _vp, _vp]),
    "tb_sgpr_plan_create": (ctypes.c_int, [_i64, _i64, _i64, _i32, _i32, _i32, _i64, _i64,
                                           ctypes.POINTER(SgprPlan)]),
    "tb_sgpr_stats_run": (ctypes.c_int, [ctypes.POINTER(SgprPlan), _vp, _vp, _vp,
                                         ctypes.c_double, _vp, _vp, _vp, _vp, _i32,
                                         _vp, _i64, _vp]),
    "tb_sgpr_sigma_unpack": (ctypes.c_int, [ctypes.POINTER(SgprPlan), _vp, _vp, _vp]),
    "tb_sgpr_tail_workspace": (_i64, [ctypes.POINTER(SgprPlan)]),
    "tb_sgpr_tail_run": (ctypes.c_int, [ctypes.POINTER(SgprPlan), _vp, ctypes.c_double, _vp,
                                        ctypes.c_double, ctypes.c_double, _vp, _vp, _vp, _vp,
                                        _vp, _i64, _vp]),
    "tb_sgpr_grad_workspace": (_i64, [ctypes.POINTER(SgprPlan)]),
    "tb_sgpr_grad_run": (ctypes.c_int, [ctypes.POINTER(SgprPlan), _vp, _vp, _vp, ctypes.c_double,
                                        _vp, ctypes.c_double, ctypes.c_double, _vp, _vp, _vp,
                                        _vp, _vp, _vp, _i64, _vp]),
    "tb_sgpr_kuf_grad_workspace": (_i64, [_i64, _i64, _i64]),
    "tb_sgpr_kuf_grad": (ctypes.c_int, [_vp, _vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32,
                                        ctypes.c_double, _vp, _vp, _vp, _vp, _i64, _vp]),
    "tb_kernel_mvm": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _i32, _i32,
                                     ctypes.c_double, _vp, _vp, _vp]),
    "tb_kernel_matrix": (ctypes.c_int, [_vp, _vp, _i64, _i64, _i64, _i32, _i32,
                                        ctypes.c_double, _vp, _vp, _vp]),
    "tb_last_error": (ctypes.c_char_p, []),
    "tb_capabilities": (ctypes.c_int32, []),
}

EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load():
    """Load (once) and return the ctypes library; raises if it is missing."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(LIB_PATH):
            raise KernelUnavailable(
                f"{LIB_PATH} is missing: build it with "
                "`python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback)")
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def last_error() -> str:
    return load().tb_last_error().decode("utf-8", "replace")


def check(rc: int, what: str, *, requested: int = 0, live: int = 0, trace=None):
    """Map a status code to the reference's exception vocabulary."""
    if rc == TB_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == TB_ERR_BUDGET:
        raise BudgetExceeded(what, requested, live, trace, message=msg)
    if rc == TB_ERR_ARG:
        raise EvaluationError(msg)
    if rc == TB_ERR_UNSPLITTABLE:
        raise UnsplittableCandidate(msg)
    if rc in (TB_ERR_UNSUPPORTED, TB_ERR_NO_DEVICE):
        raise KernelUnavailable(msg)
    raise RuntimeError(msg)
