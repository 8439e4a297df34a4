"""CPU oracle for the pairwise-kernel hot path — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline /
reference arm may import this package, and only as the checker (or as the
timed CPU reference arm).  The product path (``paper_2206_14148_b200``) never
imports it and has no CPU fallback.

Contents
--------
knn   : restatement of the reference's kNN path (tensorbudget
        ``build_knn`` -> ``match_replace`` Euclidean rewrite -> split ->
        ``evaluate`` TopK) plus a fast fp64 exact checker and the tie-aware
        comparator the parity tests use.  PINNED against golden vectors
        produced by the reference itself (tests/golden/make_golden.py).
mvm   : the SE kernel matrix-vector product of ``build_kernel_mvm``.  PINNED
        against reference golden vectors.
sgpr  : fp64 Titsias/GPflow-2.3.1 SGPR ELBO and predictive mean.  The
        reference has no SGPR code, so this restatement is
        only PARTIALLY PINNED: its SE-kernel formula is pinned by the
        reference's kernel-MVM goldens and its triangular solves by the
        reference TriangularSolve semantics; the rest rests on self-checks
        (Sigma-first == A-first, exact-GP equality at Z=X, ELBO <= log ML).
"""

from . import knn, mvm, sgpr  # noqa: F401
