"""Exactness fuzz of the kNN path on the B200: randomly drawn shapes,
metrics, dtypes, engines, k, data distributions and memory limits (which
force several database chunks), every answer checked against the fp64
oracle (indices identical except at exact-distance ties, distances to
1e-12 relative in fp64 output)."""

import os

import numpy as np
import pytest

import paper_2206_14148_b200 as tb
from oracle import knn as oknn

pytestmark = pytest.mark.gpu


def _data(rng, kind, n, m, d):
    if kind == "gauss":
        a = rng.standard_normal((n + m, d))
    elif kind == "offset":
        a = rng.standard_normal((n + m, d)) + 50.0
    elif kind == "quantized":
        a = np.round(rng.random((n + m, d)) * 7) / 7          # many exact ties
    elif kind == "clustered":
        a = (rng.standard_normal((20, d)) * 5)[rng.integers(0, 20, n + m)]
        a = a + 0.05 * rng.standard_normal((n + m, d))
    else:                                                      # duplicates
        base = rng.standard_normal((max(1, n // 4), d))
        a = base[rng.integers(0, len(base), n + m)]
    return a[:n], a[n:]


@pytest.mark.parametrize("seed", range(int(os.environ.get("TB_FUZZ_SEEDS", "24"))))
def test_knn_random_cases_exact(seed):
    rng = np.random.default_rng(1000 + seed)
    metric = ["l2", "cosine", "l1"][seed % 3]
    kind = ["gauss", "offset", "quantized", "clustered", "duplicates"][seed % 5]
    n = int(rng.integers(1, 30_000))
    m = int(rng.integers(1, 300))
    d = int(rng.choice([1, 3, 8, 31, 64, 96, 128, 130, 300]))
    k = int(rng.integers(1, min(64, n) + 1))
    dtype = np.float32 if seed % 2 else np.float64
    engine = "simt" if metric == "l1" else str(rng.choice(["auto", "tc1", "tc3", "simt"]))
    if metric == "cosine" and engine == "simt":
        engine = "tc1"
    x, q = (a.astype(dtype) for a in _data(rng, kind, n, m, d))
    if metric == "cosine":                      # zero rows are rejected by design
        x[np.all(x == 0, axis=1)] = 1.0
        q[np.all(q == 0, axis=1)] = 1.0
    inputs = (n + m) * d * np.dtype(dtype).itemsize
    limit = None
    if rng.random() < 0.5:                      # squeeze the workspace: several chunks
        try:
            full = tb.neighbors.plan(n, m, d, k, metric=metric, dtype=dtype,
                                     engine=engine).peak_bytes
        except tb.KernelUnavailable:
            full = None
        if full is not None:
            limit = inputs + max(int((full - inputs) * rng.uniform(0.3, 0.9)), 4 * 2**20)
    try:
        res = tb.knn(x, q, k, metric=metric, engine=engine, memory_limit=limit,
                     out_dtype=np.float64, return_result=True)
    except (tb.BudgetExceeded, tb.KernelUnavailable):
        return
    ref_d, ref_i = oknn.exact(x, q, k, metric=metric)
    rep = oknn.compare(res.dist, res.idx, ref_d, ref_i, x, q, metric=metric)
    assert rep["ok"], (seed, metric, kind, n, m, d, k, engine, limit, rep)
