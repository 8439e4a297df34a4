"""B200-native memory-safe pairwise-kernel hot path (arXiv 2206.14148).

Drop-in for the reference package ``tensorbudget``'s kNN / kernel-MVM path,
plus the paper's SGPR workload: fused sm_100a kernels behind a C-ABI library
(``libtb_pairwise.so``, include/tb_pairwise.h), a runtime tile planner that
honours ``memory_limit`` before any allocation, and NCCL sharding over N.

Importing this package does not touch the GPU; the first compute call loads
the library and fails loudly if it (or a B200) is missing.
"""

from .errors import (BudgetExceeded, EvaluationError, KernelUnavailable,
                     UnsplittableCandidate)
from .graph import (DType, Graph, KernelSpec, MemoryEvent, MemoryTrace,
                    PassConfig, TensorValue, build_kernel_mvm, build_knn,
                    estimate_peak_memory, evaluate, random_inputs, run_pipeline)
from .mvm import kernel_mvm, se_kernel_mvm
from .neighbors import KnnOperator, knn
from .sgpr import SGPR, sgpr_elbo, sgpr_predict_mean
from .sizes import format_size, parse_size

__all__ = [
    "BudgetExceeded", "DType", "EvaluationError", "Graph", "KernelSpec",
    "KernelUnavailable", "KnnOperator", "MemoryEvent", "MemoryTrace",
    "PassConfig", "TensorValue", "UnsplittableCandidate", "build_kernel_mvm",
    "build_knn", "estimate_peak_memory", "evaluate", "format_size", "knn",
    "parse_size", "random_inputs", "run_pipeline", "SGPR", "sgpr_elbo",
    "sgpr_predict_mean", "kernel_mvm", "se_kernel_mvm",
]
