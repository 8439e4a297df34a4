"""Generate golden fixtures by running the REFERENCE implementation.

Run in the build container (where /root/reference exists):

    python tests/golden/make_golden.py

It imports the reference package read-only from /root/reference/pkg/src and
evaluates its own graphs (``build_knn`` / ``build_kernel_mvm`` ->
``run_pipeline`` -> ``evaluate``), so the fixtures are the reference's
answers, not ours.  Large inputs are regenerated from their seed by the
tests (``paper_2206_14148_b200.synthetic``); a sha256 of the inputs is stored
so drift in the generator is detected.  f32 inputs are evaluated by the
reference in f64 (the north star's "fp64 reference").
"""

from __future__ import annotations

import hashlib
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

import tensorbudget as tb  # noqa: E402  (the reference)

from paper_2206_14148_b200 import synthetic  # noqa: E402


def sha(*arrays) -> str:
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def ref_knn(x, q, k, threshold=None, metric="l2"):
    x = np.asarray(x, np.float64)
    q = np.asarray(q, np.float64)
    g = tb.build_knn(x.shape[0], q.shape[0], x.shape[1], k, metric, tb.DType.F64)
    if threshold is not None:
        g = tb.run_pipeline(g, tb.PassConfig(tensor_size_threshold=threshold))
    t0 = time.perf_counter()
    (vals, idx), trace = tb.evaluate(g, [x, q])
    dt = time.perf_counter() - t0
    return vals.array, idx.array.astype(np.int64), trace.peak_live_bytes, dt


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {name}: " + ", ".join(
        f"{k}{list(np.shape(v))}" for k, v in arrays.items()))


def main():
    # SPEC.md:438 line example: points {0,1,2}, query 0.6, k=2
    x = np.array([[0.0], [1.0], [2.0]])
    q = np.array([[0.6]])
    d, i, _, _ = ref_knn(x, q, 2)
    save("knn_spec_line.npz", x=x, q=q, k=2, dist=d, idx=i)

    # exact ties: lower index must win (interpreter.py:379-381)
    x = np.array([[0.0, 0.0], [2.0, 0.0], [-2.0, 0.0], [3.0, 0.0],
                  [0.0, 2.0], [0.0, 0.0], [1.0, 1.0]])
    q = np.array([[0.0, 0.0], [1.0, 0.0]])
    d, i, _, _ = ref_knn(x, q, 5)
    save("knn_ties.npz", x=x, q=q, k=5, dist=d, idx=i)

    # C1 with the reference's own random_inputs (U[-1,1], seed 0), pipelined
    n, m, dd, k = 10_000, 1_000, 16, 10
    x, q = synthetic.uniform_inputs([(n, dd), (m, dd)], seed=0)
    d, i, peak, dt = ref_knn(x, q, k, threshold=2 * 10**6)
    save("knn_c1_uniform.npz", n=n, m=m, d=dd, k=k, seed=0, sha=sha(x, q),
         dist=d, idx=i, peak=peak, seconds=dt)

    # C1 Gaussian (BASELINE.json configs[0]), seed 1
    x, q = synthetic.gaussian_knn(n, m, dd, seed=1, dtype=np.float64)
    d, i, peak, dt = ref_knn(x, q, k, threshold=10 * 10**6)
    save("knn_c1_gauss.npz", n=n, m=m, d=dd, k=k, seed=1, sha=sha(x, q),
         dist=d, idx=i, peak=peak, seconds=dt)

    # C2-shaped database (1e6 x 128, f32 N(0,1)), 48-query subset, evaluated
    # by the reference in f64.  Queries are independent, so a subset pins
    # the full config.
    n, m, dd, k = 1_000_000, 10_000, 128, 10
    x, q = synthetic.gaussian_knn(n, m, dd, seed=2, dtype=np.float32)
    sub = np.arange(0, m, m // 48)[:48]
    d, i, peak, dt = ref_knn(x, q[sub], k, threshold=600 * 10**6)
    save("knn_c2_subset.npz", n=n, m=m, d=dd, k=k, seed=2, sha=sha(x[:4096], q),
         rows=sub, dist=d, idx=i, peak=peak, seconds=dt)
    del x, q

    # tie stress: quantised pixels in 4-d
    n, m, dd, k = 20_000, 64, 4, 10
    x, q = synthetic.quantized_knn(n, m, dd, seed=3)
    d, i, _, _ = ref_knn(x, q, k)
    save("knn_quantized.npz", n=n, m=m, d=dd, k=k, seed=3, sha=sha(x, q),
         dist=d, idx=i)

    # SE kernel MVM (frontend.py:34-54), f64, naive and pipelined graphs
    n = 700
    spec = tb.KernelSpec(variance=1.7, lengthscale=0.45)
    g = tb.build_kernel_mvm(n, spec)
    ins = tb.random_inputs(g, seed=5)
    out, _ = tb.evaluate(g, ins)
    gp = tb.run_pipeline(g, tb.PassConfig(tensor_size_threshold=100_000))
    outp, tr = tb.evaluate(gp, ins)
    save("mvm_se.npz", x=ins[0], y=ins[1], v=ins[2], variance=1.7,
         lengthscale=0.45, out=out.array, out_pipelined=outp.array,
         peak_pipelined=tr.peak_live_bytes)

    # TriangularSolve semantics (interpreter.py:475-490)
    rng = np.random.default_rng(11)
    a = np.tril(rng.uniform(0.5, 2.0, (12, 12)))
    b = rng.uniform(-1, 1, (12, 3))
    gb = tb.GraphBuilder("trsm")
    pa, pb = gb.param(a.shape, tb.DType.F64), gb.param(b.shape, tb.DType.F64)
    gt = gb.build(gb.triangular_solve(pa, pb, True))
    out, _ = tb.evaluate(gt, [a, b])
    save("trsm_lower.npz", a=a, b=b, out=out.array)

    # budget KAT: naive [100,100,100] f64 distance requests exactly 8e6 bytes
    g = tb.build_pairwise_distance(100, 100, 100)
    try:
        tb.evaluate(g, tb.random_inputs(g, seed=0), budget=10**6)
        requested = -1
    except tb.BudgetExceeded as exc:
        requested = exc.requested
    est = tb.estimate_peak_memory(tb.build_knn(10_000, 1_000, 16, 10))
    save("budget.npz", naive_requested=requested, knn_c1_naive_peak=est)


def metrics():
    """L1 and cosine kNN (frontend.py:57-73 naive forms, TopK of
    interpreter.py:371-390) on the reference, naive and query-split."""
    out = {}
    # reference random_inputs style U[-1, 1]
    x, q = synthetic.uniform_inputs([(3000, 16), (100, 16)], seed=4)
    for metric in ("l1", "cosine"):
        d, i, _, _ = ref_knn(x, q, 10, metric=metric)
        dp, ip, _, _ = ref_knn(x, q, 10, threshold=2 * 10**6, metric=metric)
        assert np.array_equal(i, ip)
        out[f"{metric}_uniform_dist"], out[f"{metric}_uniform_idx"] = d, i
    out["uniform_x"], out["uniform_q"] = x, q
    # ties: small integer lattice (L1) and scaled copies of directions (cosine)
    rng = np.random.default_rng(6)
    x = rng.integers(0, 4, (2000, 3)).astype(np.float64)
    q = rng.integers(0, 4, (50, 3)).astype(np.float64)
    d, i, _, _ = ref_knn(x, q, 10, metric="l1")
    out["l1_ties_x"], out["l1_ties_q"], out["l1_ties_dist"], out["l1_ties_idx"] = x, q, d, i
    base = rng.integers(1, 4, (400, 3)).astype(np.float64)
    x = np.concatenate([base, 2.0 * base, 3.0 * base])[rng.permutation(1200)]
    q = rng.integers(1, 4, (40, 3)).astype(np.float64)
    d, i, _, _ = ref_knn(x, q, 10, metric="cosine")
    out["cos_ties_x"], out["cos_ties_q"], out["cos_ties_dist"], out["cos_ties_idx"] = x, q, d, i
    save("knn_metrics.npz", **out)


if __name__ == "__main__":
    if sys.argv[1:] == ["metrics"]:
        metrics()
    else:
        main()
        metrics()
