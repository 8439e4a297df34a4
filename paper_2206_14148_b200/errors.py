"""Exception vocabulary of the reference, kept so callers' except clauses work.

BudgetExceeded      interpreter.py:44-54 (RuntimeError, fields instruction,
                    requested, live, trace)
EvaluationError     interpreter.py:40-41 (arity / shape / dtype mismatches)
UnsplittableCandidate  split.py:31-32 (one tile cannot fit the split size)
KernelUnavailable   new: the CUDA library or a B200 is missing (there is
                    deliberately no CPU fallback)
"""

from __future__ import annotations


class EvaluationError(Exception):
    pass


class BudgetExceeded(RuntimeError):
    """An allocation would push live bytes over the configured budget."""

    def __init__(self, instruction: str, requested: int, live: int, trace=None,
                 message: str | None = None):
        self.instruction = instruction
        self.requested = requested
        self.live = live
        self.trace = trace
        super().__init__(message or (
            f"{instruction}: allocating {requested} bytes would exceed the budget "
            f"(live={live})"))


class UnsplittableCandidate(Exception):
    pass


class KernelUnavailable(RuntimeError):
    pass
