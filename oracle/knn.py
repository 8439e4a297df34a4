"""kNN oracle (TEST INFRASTRUCTURE ONLY — see oracle/__init__.py).

Restates the reference's brute-force kNN path on the CPU in numpy:

* ``reference_port``  — the reference's own algorithm, step for step: the
  graph ``build_knn`` emits (/root/reference/pkg/src/tensorbudget/frontend.py:98-114)
  after the Euclidean rewrite (match_replace.py:139-159: ``add(add(bcast |q|^2,
  bcast |x|^2), mul(-2, dot(q, x)))``, no clamp for a TopK consumer), split
  along the query axis as split.py:221-222/285-301 plans it, with the TopK of
  interpreter.py:371-390 (full *stable* argsort, first k, ties -> lower index,
  indices returned in the operand float dtype).  This is what the CPU
  baseline times.
* ``exact``           — the parity checker: the same fp64 arithmetic, but
  selecting with ``argpartition`` and then stable-sorting every candidate
  tied with the k-th value, which yields exactly the stable-argsort answer
  at a fraction of the cost (SURVEY.md §8(c) "kNN cost").
* ``compare``         — the tie-aware parity gate of the north star: indices
  identical except at distance ties within 1e-5 relative; distances within
  1e-4 by the reference's ``rel_err`` (tests/conftest.py:7-12,
  cli.py:202-208).

Pinned by tests/test_oracle.py against fixtures produced by the reference
itself (tests/golden/make_golden.py).
"""

from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------------------
# the reference algorithm


def reference_split_rows(n: int, m: int, d: int, dtype, split_bytes: int | None) -> int:
    """Query rows per loop trip the reference's plan_split would choose for
    the [m, n] distance producer (split.py:285-301): floor(split / bytes-per-
    index) clamped to [1, m]; None means no split (one trip)."""
    if split_bytes is None:
        return m
    per_index = n * np.dtype(dtype).itemsize
    return max(1, min(m, split_bytes // per_index))


def reference_port(x: np.ndarray, q: np.ndarray, k: int,
                   split_bytes: int | None = None) -> tuple[np.ndarray, np.ndarray]:
    """(values[m,k], indices[m,k]) with indices in the operand float dtype,
    computed the way the reference's pipelined graph evaluates it."""
    x = np.ascontiguousarray(x)
    q = np.ascontiguousarray(q)
    n, d = x.shape
    m = q.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k={k} must satisfy 1 <= k <= n={n}")
    dt = x.dtype
    xn = np.sum(np.square(x), axis=1)               # hoisted loop invariant
    rows = reference_split_rows(n, m, d, dt, split_bytes)
    vals = np.empty((m, k), dt)
    idx = np.empty((m, k), dt)
    for s in range(0, m, rows):
        qc = q[s:s + rows]
        qn = np.sum(np.square(qc), axis=1)
        cross = np.einsum("ad,bd->ab", qc, x, optimize=True)
        dist = (qn[:, None] + xn[None, :]) + (dt.type(-2.0) * cross)
        order = np.argsort(dist, axis=1, kind="stable")[:, :k]
        vals[s:s + rows] = np.take_along_axis(dist, order, axis=1)
        idx[s:s + rows] = order.astype(dt)
    return vals, idx


# ---------------------------------------------------------------------------
# fast exact checker


def _dist_block(qc, x64, xn, metric):
    """fp64 [rows(qc), n] distances in the reference graph's formulas:
    l2 expanded (match_replace.py:149-155), l1 = sum |q - x|
    (frontend.py:57-63), cosine = 1 - q.x / (|q| |x|) (frontend.py:66-73)."""
    if metric == "l2":
        qn = np.sum(np.square(qc), axis=1)
        return (qn[:, None] + xn[None, :]) + (-2.0 * (qc @ x64.T))
    if metric == "l1":
        step = max(1, int(2e7 // max(1, x64.shape[0] * x64.shape[1])))
        return np.concatenate([np.sum(np.abs(qc[a:a + step, None, :] - x64[None, :, :]), axis=2)
                               for a in range(0, qc.shape[0], step)])
    if metric == "cosine":
        qn = np.sqrt(np.sum(np.square(qc), axis=1))
        return 1.0 - (qc @ x64.T) / (qn[:, None] * xn[None, :])
    raise ValueError(f"unknown metric {metric!r}")


def exact(x: np.ndarray, q: np.ndarray, k: int, chunk: int = 256, metric: str = "l2",
          ) -> tuple[np.ndarray, np.ndarray]:
    """fp64 distances of the reference graph for ``metric``, stable-argsort
    semantics.  Returns (dist f64[m,k], idx int64[m,k])."""
    x64 = np.asarray(x, dtype=np.float64)
    q64 = np.asarray(q, dtype=np.float64)
    n = x64.shape[0]
    m = q64.shape[0]
    if not 1 <= k <= n:
        raise ValueError(f"k={k} must satisfy 1 <= k <= n={n}")
    if metric == "cosine":
        xn = np.sqrt(np.sum(np.square(x64), axis=1))
    else:
        xn = np.sum(np.square(x64), axis=1)
    out_d = np.empty((m, k), np.float64)
    out_i = np.empty((m, k), np.int64)
    for s in range(0, m, chunk):
        qc = q64[s:s + chunk]
        dist = _dist_block(qc, x64, xn, metric)
        if k < n:
            part = np.argpartition(dist, k - 1, axis=1)[:, :k]
            kth = np.max(np.take_along_axis(dist, part, axis=1), axis=1)
        else:
            kth = np.max(dist, axis=1)
        for r in range(dist.shape[0]):
            cand = np.nonzero(dist[r] <= kth[r])[0]        # ascending index
            order = cand[np.argsort(dist[r, cand], kind="stable")][:k]
            out_i[s + r] = order
            out_d[s + r] = dist[r, order]
    return out_d, out_i


def direct_dist(x: np.ndarray, q: np.ndarray, rows: np.ndarray,
                idx: np.ndarray, metric: str = "l2") -> np.ndarray:
    """Exact fp64 distance for the given (query row, data index) pairs:
    sum((q - x)^2), sum |q - x|, or 1 - cos."""
    x64 = np.asarray(x, dtype=np.float64)
    q64 = np.asarray(q, dtype=np.float64)
    a, b = q64[rows], x64[idx]
    if metric == "l1":
        return np.sum(np.abs(a - b), axis=-1)
    if metric == "cosine":
        return 1.0 - np.sum(a * b, axis=-1) / (np.sqrt(np.sum(a * a, axis=-1)) *
                                                np.sqrt(np.sum(b * b, axis=-1)))
    diff = a - b
    return np.sum(diff * diff, axis=-1)


# ---------------------------------------------------------------------------
# parity gate


def rel_err(a, b) -> float:
    """Max absolute deviation over the reference's max magnitude
    (tests/conftest.py:7-12 of the reference)."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    if a.size == 0:
        return 0.0
    scale = max(float(np.max(np.abs(b))), 1e-300)
    return float(np.max(np.abs(a - b))) / scale


def compare(got_dist, got_idx, ref_dist, ref_idx, x, q,
            tie_rtol: float = 1e-5, dist_rtol: float = 1e-4, metric: str = "l2") -> dict:
    """Tie-aware kNN parity report.

    A position whose index differs from the reference counts as a tie (and
    passes) when the exact fp64 distance of the returned neighbour equals the
    reference's distance at that position within ``tie_rtol`` relative.
    Returned indices must be unique per query and in range.
    """
    got_idx = np.asarray(got_idx).astype(np.int64)
    ref_idx = np.asarray(ref_idx).astype(np.int64)
    got_dist = np.asarray(got_dist, dtype=np.float64)
    ref_dist = np.asarray(ref_dist, dtype=np.float64)
    n = np.asarray(x).shape[0]
    m, k = ref_idx.shape
    report = {"queries": m, "k": k, "identical": 0, "tie_swaps": 0,
              "mismatches": 0, "bad_index": 0, "dist_rel_err": 0.0,
              "first_bad": None}
    if got_idx.shape != ref_idx.shape:
        report["mismatches"] = m
        report["first_bad"] = ("shape", got_idx.shape, ref_idx.shape)
        return report
    for r in range(m):
        gi, ri = got_idx[r], ref_idx[r]
        if np.any(gi < 0) or np.any(gi >= n) or len(set(gi.tolist())) != k:
            report["bad_index"] += 1
            report["first_bad"] = report["first_bad"] or ("index", r, gi.tolist())
            continue
        if np.array_equal(gi, ri):
            report["identical"] += 1
            continue
        diff = np.nonzero(gi != ri)[0]
        dg = direct_dist(x, q, np.full(diff.shape, r), gi[diff], metric)
        scale = np.maximum(np.abs(ref_dist[r, diff]), 1e-30)
        if np.all(np.abs(dg - ref_dist[r, diff]) <= tie_rtol * scale + 1e-12):
            report["tie_swaps"] += 1
        else:
            report["mismatches"] += 1
            report["first_bad"] = report["first_bad"] or (
                "neighbour", r, gi.tolist(), ri.tolist())
    if metric == "cosine":
        # cosine distances live in [0, 2]; exactly parallel rows have distance
        # 0 computed as a few ulps of either sign, so the error is measured
        # against the metric's scale, not against an all-~0 reference
        report["dist_rel_err"] = float(np.max(np.abs(got_dist - ref_dist), initial=0.0)
                                       / max(float(np.max(np.abs(ref_dist), initial=0.0)), 1.0))
    else:
        # the reference's expanded form ||q||^2 + ||x||^2 - 2 q.x leaves a few
        # ulps of that sum where the true distance is 0 (duplicates); the
        # error is measured against max(max |ref|, 1e-6 of the norms' scale)
        x64 = np.asarray(x, dtype=np.float64)
        q64 = np.asarray(q, dtype=np.float64)
        sq = (float(np.max(np.einsum("ij,ij->i", x64, x64), initial=0.0))
              + float(np.max(np.einsum("ij,ij->i", q64, q64), initial=0.0)))
        floor = 1e-6 * sq if metric == "l2" else 0.0
        den = max(float(np.max(np.abs(ref_dist), initial=0.0)), floor)
        diff = float(np.max(np.abs(got_dist - ref_dist), initial=0.0))
        report["dist_rel_err"] = diff / den if den > 0 else (0.0 if diff == 0 else np.inf)
    report["ok"] = (report["mismatches"] == 0 and report["bad_index"] == 0
                    and report["dist_rel_err"] <= dist_rtol)
    return report
