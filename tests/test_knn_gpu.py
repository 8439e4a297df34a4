"""kNN parity on the B200: the CUDA path (through the C-ABI) against the
reference's golden answers and the fp64 oracle.  Gate (north star): indices
identical except at distance ties within 1e-5 relative; distances within
1e-4 (the reference's rel_err)."""

import os

import numpy as np
import pytest

from conftest import golden, rel_err
from oracle import knn as oknn
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200 import neighbors, synthetic

pytestmark = pytest.mark.gpu

ENGINES = ["simt", "tc3", "tc1"]


def _torch():
    import torch
    return torch


def engines_available():
    from paper_2206_14148_b200 import _lib
    out = []
    for e in ENGINES:
        try:
            neighbors.plan(300, 10, 8, 3, engine=e)
            x = np.random.default_rng(0).standard_normal((300, 8)).astype(np.float32)
            neighbors.knn(x, x[:10], 3, engine=e)
            out.append(e)
        except tb.KernelUnavailable:
            pass
    return out


@pytest.fixture(scope="module")
def engines():
    e = engines_available()
    assert "simt" in e
    return e


def check(dist, idx, ref_d, ref_i, x, q):
    rep = oknn.compare(dist, idx, ref_d, ref_i, x, q)
    assert rep["ok"], rep
    return rep


@pytest.mark.parametrize("name", ["knn_spec_line.npz", "knn_ties.npz"])
def test_small_kats(name, engines):
    g = golden(name)
    for e in engines:
        d, i = tb.knn(g["x"], g["q"], int(g["k"]), engine=e)
        assert np.array_equal(i, g["idx"]), e
        assert rel_err(d, g["dist"]) < 1e-12, e


@pytest.mark.parametrize("name", ["knn_c1_uniform.npz", "knn_c1_gauss.npz"])
def test_c1_f64(name, engines):
    g = golden(name)
    n, m, d, k = (int(g[s]) for s in "nmdk")
    if "uniform" in name:
        x, q = synthetic.uniform_inputs([(n, d), (m, d)], seed=int(g["seed"]))
    else:
        x, q = synthetic.gaussian_knn(n, m, d, seed=int(g["seed"]), dtype=np.float64)
    for e in engines:
        dist, idx = tb.knn(x, q, k, engine=e)
        rep = check(dist, idx, g["dist"], g["idx"], x, q)
        assert rep["identical"] >= m - 2, (e, rep)
        assert rel_err(dist, g["dist"]) < 1e-12, e   # fp64 re-rank


def test_graph_evaluate_c1(engines):
    g = golden("knn_c1_uniform.npz")
    graph = tb.build_knn(int(g["n"]), int(g["m"]), int(g["d"]), int(g["k"]))
    graph = tb.run_pipeline(graph, tb.PassConfig(tensor_size_threshold=2 * 10**6))
    ins = tb.random_inputs(graph, seed=int(g["seed"]))
    (vals, idx), trace = tb.evaluate(graph, ins, budget=50 * 10**6)
    assert idx.array.dtype == np.float64        # reference: indices in float dtype
    assert np.array_equal(idx.array.astype(np.int64), g["idx"])
    assert rel_err(vals.array, g["dist"]) < 1e-12
    assert trace.peak_live_bytes <= 50 * 10**6


def test_c2_full_shape_subset_against_reference(engines):
    torch = _torch()
    g = golden("knn_c2_subset.npz")
    n, m, d, k = (int(g[s]) for s in "nmdk")
    x, q = synthetic.gaussian_knn(n, m, d, seed=int(g["seed"]), dtype=np.float32)
    xt = torch.from_numpy(x).cuda()
    qt = torch.from_numpy(q).cuda()
    rows = g["rows"]
    extra = np.random.default_rng(9).choice(m, 64, replace=False)
    ref_d2, ref_i2 = oknn.exact(x, q[extra], k)
    for e in engines:
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        op = neighbors.KnnOperator(n, m, d, k, engine=e, memory_limit="1GB")
        dist, idx = op.run(xt, qt)
        torch.cuda.synchronize()
        peak = torch.cuda.max_memory_allocated() - base + (n + m) * d * 4
        assert peak <= 10**9, (e, peak)
        dist, idx = dist.cpu().numpy(), idx.cpu().numpy()
        check(dist[rows], idx[rows], g["dist"], g["idx"], x, q[rows])
        check(dist[extra], idx[extra], ref_d2, ref_i2, x, q[extra])
        if e != "tc1":    # single-pass bf16 certifies only with a wide K'
            assert op.fallback_count() <= m // 100, e


def test_quantized_ties(engines):
    g = golden("knn_quantized.npz")
    n, m, d, k = (int(g[s]) for s in "nmdk")
    x, q = synthetic.quantized_knn(n, m, d, seed=int(g["seed"]))
    for e in engines:
        dist, idx = tb.knn(x, q, k, engine=e)
        check(dist, idx, g["dist"], g["idx"], x, q)


@pytest.mark.parametrize("n,m,d,k", [
    (1, 1, 1, 1), (3, 2, 1, 3), (17, 5, 3, 17), (300, 129, 130, 7),
    (1000, 257, 64, 50), (4097, 3, 16, 10), (20000, 1, 200, 1)])
def test_edge_shapes(n, m, d, k, engines):
    rng = np.random.default_rng(n + m + d + k)
    x = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((m, d)).astype(np.float32)
    ref_d, ref_i = oknn.exact(x, q, k)
    for e in engines + ["auto"]:
        dist, idx = tb.knn(x, q, k, engine=e)
        check(dist, idx, ref_d, ref_i, x, q)


@pytest.mark.parametrize("engine", ["tc3", "tc1"])
@pytest.mark.parametrize("n,m,d", [(60000, 300, 784), (20000, 130, 300), (5000, 64, 1000)])
def test_streamed_query_tc_engine_large_d(n, m, d, engine):
    """d > 128: the tcgen05 engine streams query k-blocks through the ring
    (C3 is MNIST-shaped, d = 784), bf16x3 and fp16 single pass.  Exact vs
    the fp64 oracle; no fallback."""
    x, q = synthetic.gaussian_knn(n, m, d, seed=d)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(n, m, d, 10, engine=engine)
    import torch
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() == 0
    xq, qq = synthetic.quantized_knn(n // 4, m, d, seed=1)      # tie stress
    rd, ri = oknn.exact(xq, qq, 10)
    dist, idx = tb.knn(xq, qq, 10, engine=engine)
    check(dist, idx, rd, ri, xq, qq)


@pytest.mark.parametrize("n,m,d", [(70000, 300, 128), (30000, 1000, 64), (9000, 129, 17)])
def test_cta_pair_tc_kernel(n, m, d, monkeypatch):
    """The opt-in CTA-pair kernel (TB_TC_PAIR=1: cta_group::2, odd query-tile
    counts leave the last pair half empty) gives the same exact answers."""
    monkeypatch.setenv("TB_TC_PAIR", "1")
    x, q = synthetic.gaussian_knn(n, m, d, seed=n + d)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(n, m, d, 10, engine="tc3")
    import torch
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() == 0


@pytest.mark.parametrize("n,m,d", [(70000, 300, 128), (9000, 129, 17), (20000, 130, 300)])
def test_single_cta_tc1_kernel(n, m, d, monkeypatch):
    """tc1 defaults to multicast clusters of 2 CTAs; TB_TC_MC=0 selects the
    1-CTA kernel, which must give the same exact answers."""
    monkeypatch.setenv("TB_TC_MC", "0")
    x, q = synthetic.gaussian_knn(n, m, d, seed=n + 3 * d)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(n, m, d, 10, engine="tc1")
    import torch
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() == 0


@pytest.mark.parametrize("engine", ["tc1", "tc3"])
@pytest.mark.parametrize("seed_tiles", ["1", "16", "400"])
def test_seed_launch_length_is_exact(engine, seed_tiles, monkeypatch):
    """The seed launch only primes the shared thresholds: any length
    (TB_TC_SEED, including one longer than the database) gives the same exact
    answers and a consistent candidate-list count."""
    monkeypatch.setenv("TB_TC_SEED", seed_tiles)
    n, m, d = 70000, 300, 128
    x, q = synthetic.gaussian_knn(n, m, d, seed=11)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(n, m, d, 10, engine=engine)
    import torch
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() == 0


@pytest.mark.parametrize("offset,tail", [(100.0, False), (0.5, False), (0.0, True)])
def test_fp16_engine_offset_and_heavy_tail_data(offset, tail):
    """tc1 centres l2 data with a large common offset on the sample mean
    (distances are translation invariant), and the norm-split certification
    keeps heavy-tailed outliers from widening every query's bound: exact,
    and (almost) no query needs the brute-force fallback."""
    import torch
    rng = np.random.default_rng(7)
    a = rng.standard_cauchy((30300, 48)).clip(-1e4, 1e4) if tail else \
        rng.standard_normal((30300, 48)) + offset
    x, q = a[:30000].astype(np.float32), a[30000:].astype(np.float32)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(30000, 300, 48, 10, engine="tc1")
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() <= 3


@pytest.mark.parametrize("scale", [1e5, 1e3, 1e-4, 3e-9])
def test_fp16_engine_scaling_is_exact(scale):
    """Engine tc1 (fp16 single pass) scales operands by powers of two into
    fp16 range: large data (redo pass with t < 1), tiny data (t > 1) and data
    that fits as is must all give the exact answer without fallbacks."""
    import torch
    x, q = synthetic.gaussian_knn(40000, 300, 96, seed=int(-np.log10(scale) * 10) % 97)
    x, q = x * np.float32(scale), q * np.float32(scale)
    ref_d, ref_i = oknn.exact(x, q, 10)
    op = neighbors.KnnOperator(40000, 300, 96, 10, engine="tc1")
    dist, idx = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    check(dist.cpu().numpy(), idx.cpu().numpy(), ref_d, ref_i, x, q)
    assert op.fallback_count() == 0


def test_duplicates_resolve_to_lower_index(engines):
    rng = np.random.default_rng(4)
    base = rng.standard_normal((50, 12)).astype(np.float32)
    x = np.concatenate([base, base, base])          # every point three times
    q = base[:20] + 1e-3
    ref_d, ref_i = oknn.exact(x, q, 9)
    for e in engines:
        dist, idx = tb.knn(x, q, 9, engine=e)
        check(dist, idx, ref_d, ref_i, x, q)


def test_memory_limit_forces_chunks_same_answer(engines):
    rng = np.random.default_rng(5)
    n, m, d, k = 200_000, 300, 96, 10
    x = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((m, d)).astype(np.float32)
    ref_d, ref_i = oknn.exact(x, q, k)
    for e in engines:
        resident = (n + m) * d * 4
        p = neighbors.plan(n, m, d, k, engine=e, memory_limit=resident + 30 * 10**6)
        assert p.peak_bytes <= resident + 30 * 10**6
        dist, idx = tb.knn(x, q, k, engine=e, memory_limit=resident + 30 * 10**6)
        check(dist, idx, ref_d, ref_i, x, q)


def test_budget_exceeded_raises_before_work():
    x = np.zeros((10_000, 16))
    with pytest.raises(tb.BudgetExceeded):
        tb.knn(x, x[:100], 5, memory_limit="1MB")


def test_index_base_and_f64_out(engines):
    rng = np.random.default_rng(6)
    x = rng.standard_normal((5000, 32)).astype(np.float32)
    q = rng.standard_normal((40, 32)).astype(np.float32)
    ref_d, ref_i = oknn.exact(x, q, 5)
    for e in engines:
        dist, idx = tb.knn(x, q, 5, engine=e, index_base=1_000_000, out_dtype=np.float64)
        assert dist.dtype == np.float64
        check(dist, idx - 1_000_000, ref_d, ref_i, x, q)
        assert rel_err(dist, ref_d) < 1e-12


def test_fallback_path_is_exact(engines, monkeypatch):
    monkeypatch.setenv("TB_FORCE_FALLBACK", "1")
    rng = np.random.default_rng(7)
    x = rng.standard_normal((3000, 20))
    q = rng.standard_normal((37, 20))
    ref_d, ref_i = oknn.exact(x, q, 6)
    res = tb.knn(x, q, 6, engine="simt", return_result=True)
    assert res.fallback_queries == 37
    check(res.dist, res.idx, ref_d, ref_i, x, q)
    assert rel_err(res.dist, ref_d) < 1e-12


@pytest.mark.parametrize("metric", ["l2", "cosine", "l1"])
@pytest.mark.parametrize("d", [20, 128, 300])
def test_fallback_stages_exact(metric, d, monkeypatch):
    """Both fallback stages, every query forced through them: the bounded
    hit-buffer scan (most queries) and, for queries with more rows tied at
    the k-th distance than the hit buffer holds (90 exact duplicates of the
    nearest row), the exhaustive kernels; ties -> lower index throughout."""
    monkeypatch.setenv("TB_FORCE_FALLBACK", "1")
    rng = np.random.default_rng(d)
    x = rng.standard_normal((6000, d)).astype(np.float32)
    q = rng.standard_normal((41, d)).astype(np.float32)
    dup = rng.choice(6000, 90, replace=False)
    x[dup] = q[3] + 0.01                      # query 3: 90 rows tied at its k nearest
    engine = "simt" if metric == "l1" else "tc1"
    ref_d, ref_i = oknn.exact(x, q, 10, metric=metric)
    res = tb.knn(x, q, 10, metric=metric, engine=engine, return_result=True)
    assert res.fallback_queries == 41
    assert np.array_equal(res.idx[3], np.sort(dup)[:10])
    mcheck(res.dist, res.idx, ref_d, ref_i, x, q, metric)


def test_input_buffers_untouched(engines):
    torch = _torch()
    rng = np.random.default_rng(8)
    x = torch.from_numpy(rng.standard_normal((4000, 40)).astype(np.float32)).cuda()
    q = torch.from_numpy(rng.standard_normal((70, 40)).astype(np.float32)).cuda()
    x0, q0 = x.clone(), q.clone()
    for e in engines:
        tb.knn(x, q, 4, engine=e)
    assert torch.equal(x, x0) and torch.equal(q, q0)


def test_deterministic_repeats(engines):
    rng = np.random.default_rng(10)
    x = rng.standard_normal((30000, 64)).astype(np.float32)
    q = rng.standard_normal((500, 64)).astype(np.float32)
    for e in engines:
        a = tb.knn(x, q, 10, engine=e)
        b = tb.knn(x, q, 10, engine=e)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])


def test_topk_merge_abi():
    torch = _torch()
    from paper_2206_14148_b200 import distributed
    rng = np.random.default_rng(11)
    x = rng.standard_normal((9000, 24))
    q = rng.standard_normal((33, 24))
    ref_d, ref_i = oknn.exact(x, q, 8)
    parts = np.array_split(np.arange(9000), 3)
    dl, il = [], []
    for p in parts:
        d, i = oknn.exact(x[p], q, 8)
        dl.append(d)
        il.append(i + p[0])
    od, oi = distributed.merge_topk(torch.from_numpy(np.stack(dl)).cuda(),
                                    torch.from_numpy(np.stack(il)).cuda())
    assert np.array_equal(oi.cpu().numpy(), ref_i)
    assert rel_err(od.cpu().numpy(), ref_d) < 1e-12


def test_topk_merge_keeps_int64_global_indices():
    """Shards far into an 8-GPU database: global indices past 2^31 survive
    the merge unchanged and exact-score ties still resolve to the lower
    global index (reference TopK tie rule, interpreter.py:379-381)."""
    torch = _torch()
    from paper_2206_14148_b200 import distributed
    m, k, L = 7, 5, 3
    base = np.array([3_000_000_000, 2_147_483_000, 5_000_000_123], np.int64)
    rng = np.random.default_rng(12)
    d = np.sort(rng.integers(0, 6, size=(L, m, k)).astype(np.float64), axis=2)   # many ties
    i = np.empty((L, m, k), np.int64)
    for l in range(L):
        i[l] = base[l] + np.sort(rng.choice(1000, size=(m, k), replace=True), axis=1) * 3 + \
            np.arange(k)
    od, oi = distributed.merge_topk(torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda())
    dd = d.transpose(1, 0, 2).reshape(m, L * k)
    ii = i.transpose(1, 0, 2).reshape(m, L * k)
    for r in range(m):
        order = np.lexsort((ii[r], dd[r]))[:k]
        assert np.array_equal(oi.cpu().numpy()[r], ii[r, order])
        assert np.array_equal(od.cpu().numpy()[r], dd[r, order])


def test_misaligned_views_are_rejected_or_copied():
    """Row kernels read x, q with 16-byte vector loads: the operator rejects
    a view that does not start on a 16-byte boundary (instead of faulting
    the context) and the functional knn() copies it."""
    torch = _torch()
    rng = np.random.default_rng(13)
    x = rng.standard_normal((2000, 32)).astype(np.float32)
    q = rng.standard_normal((40, 32)).astype(np.float32)
    buf = torch.empty(2000 * 32 + 1, dtype=torch.float32, device="cuda")
    xv = buf[1:].view(2000, 32)
    xv.copy_(torch.from_numpy(x))
    qd = torch.from_numpy(q).cuda()
    op = neighbors.KnnOperator(2000, 40, 32, 5)
    with pytest.raises(tb.EvaluationError):
        op.run(xv, qd)
    d, i = tb.knn(xv, qd, 5)
    ref_d, ref_i = oknn.exact(x, q, 5)
    check(d.cpu().numpy(), i.cpu().numpy(), ref_d, ref_i, x, q)


@pytest.mark.parametrize("chunk", [0, 2048, 777])
def test_run_host_pipelined_matches_device_run(chunk):
    """tb_knn_run_host (host buffers, per-chunk H2D overlapped with compute)
    returns exactly what the device-resident call returns, and the oracle's
    answer, for 1 and several database chunks (ragged last chunk)."""
    import torch
    x, q = synthetic.gaussian_knn(9000, 300, 64, seed=21)
    op = neighbors.KnnOperator(9000, 300, 64, 10, max_chunk_rows=chunk)
    if chunk:
        assert op.plan.n_chunks > 1
    xh = torch.from_numpy(x).pin_memory()
    qh = torch.from_numpy(q).pin_memory()
    dh, ih = op.run_host(xh, qh)
    torch.cuda.synchronize()
    dd, idd = op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())
    assert np.array_equal(dh.numpy(), dd.cpu().numpy())
    assert np.array_equal(ih.numpy(), idd.cpu().numpy())
    ref_d, ref_i = oknn.exact(x, q, 10)
    assert oknn.compare(dh.numpy(), ih.numpy(), ref_d, ref_i, x, q)["ok"]


# ---------------------------------------------------------------- metrics --
# L1 (CUDA-core engine: no tensor-core form) and cosine (tensor cores over
# unit-normalised rows), the reference's other two metrics
# (frontend.py:19,57-73), exact against the reference's own answers.

def mcheck(dist, idx, ref_d, ref_i, x, q, metric):
    rep = oknn.compare(dist, idx, ref_d, ref_i, x, q, metric=metric)
    assert rep["ok"], rep
    return rep


@pytest.mark.parametrize("metric,case", [("l1", "uniform"), ("cosine", "uniform"),
                                         ("l1", "l1_ties"), ("cosine", "cos_ties")])
def test_metric_reference_goldens(metric, case):
    g = golden("knn_metrics.npz")
    if case == "uniform":
        x, q = g["uniform_x"], g["uniform_q"]
        rd, ri = g[f"{metric}_uniform_dist"], g[f"{metric}_uniform_idx"]
    else:
        x, q, rd, ri = g[f"{case}_x"], g[f"{case}_q"], g[f"{case}_dist"], g[f"{case}_idx"]
    for dt in (np.float64, np.float32):
        dist, idx = tb.knn(x.astype(dt), q.astype(dt), 10, metric=metric)
        if dt == np.float64:
            assert np.array_equal(idx, ri)          # ties resolve exactly as the reference
            assert rel_err(dist, rd) < 1e-12
        else:
            rd32, ri32 = oknn.exact(x.astype(dt), q.astype(dt), 10, metric=metric)
            mcheck(dist, idx, rd32, ri32, x.astype(dt), q.astype(dt), metric)


@pytest.mark.parametrize("metric,n,m,d", [("l1", 30000, 200, 64), ("cosine", 30000, 200, 64),
                                          ("cosine", 20000, 130, 300), ("l1", 6000, 70, 300)])
def test_metric_random_vs_oracle(metric, n, m, d):
    x, q = synthetic.gaussian_knn(n, m, d, seed=n + d)
    ref_d, ref_i = oknn.exact(x, q, 10, metric=metric)
    res = tb.knn(x, q, 10, metric=metric, return_result=True)
    mcheck(res.dist, res.idx, ref_d, ref_i, x, q, metric)
    assert res.fallback_queries == 0


@pytest.mark.parametrize("metric", ["l1", "cosine"])
def test_metric_fallback_and_chunking_exact(metric, monkeypatch):
    x, q = synthetic.gaussian_knn(9000, 90, 24, seed=5)
    ref_d, ref_i = oknn.exact(x, q, 7, metric=metric)
    resident = (9000 + 90) * 24 * 4
    d1, i1 = tb.knn(x, q, 7, metric=metric, memory_limit=resident + 3_000_000)
    mcheck(d1, i1, ref_d, ref_i, x, q, metric)
    monkeypatch.setenv("TB_FORCE_FALLBACK", "1")
    res = tb.knn(x, q, 7, metric=metric, return_result=True)
    assert res.fallback_queries == 90
    mcheck(res.dist, res.idx, ref_d, ref_i, x, q, metric)


def test_metric_engine_rules_and_zero_rows():
    x, q = synthetic.gaussian_knn(500, 5, 8, seed=1)
    with pytest.raises(tb.KernelUnavailable):
        tb.knn(x, q, 3, metric="l1", engine="tc3")
    with pytest.raises(tb.KernelUnavailable):
        tb.knn(x, q, 3, metric="cosine", engine="simt")
    # zero rows are flagged by the prep kernels (database or query side,
    # both tensor-core engines, device and host entry points)
    import torch
    for engine in ("tc1", "tc3"):
        for side in ("x", "q"):
            xz, qz = x.copy(), q.copy()
            (xz if side == "x" else qz)[3] = 0.0
            with pytest.raises(ValueError, match="zero rows"):
                tb.knn(xz, qz, 3, metric="cosine", engine=engine)
            op = neighbors.KnnOperator(500, 5, 8, 3, metric="cosine", engine=engine)
            with pytest.raises(ValueError, match="zero rows"):
                op.run_host(torch.from_numpy(xz), torch.from_numpy(qz))
            op.run(torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda())   # flag cleared
    x[7] = 0.0
    with pytest.raises(ValueError, match="zero rows"):
        tb.knn(x, q, 3, metric="cosine")
    graph = tb.build_knn(500, 5, 8, 3, metric="l1")
    x, q = x.astype(np.float64), q.astype(np.float64)
    (vals, idx), _ = tb.evaluate(graph, [x, q])
    rd, ri = oknn.exact(x, q, 3, metric="l1")
    assert np.array_equal(np.asarray(idx.array).astype(np.int64), ri)


def test_sharded_knn_with_real_kernels_and_cuda_merge():
    """The multi-GPU recipe with the real kernels: 3 uneven database shards
    (index_base = shard start, exact f64 lists) merged by tb_topk_merge equal
    the single-call answer and the oracle (ties -> lower global index)."""
    import torch
    from paper_2206_14148_b200 import distributed
    x, q = synthetic.quantized_knn(20001, 150, 8, seed=4)      # many exact ties
    ref_d, ref_i = oknn.exact(x, q, 10)
    xt, qt = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    dls, ils = [], []
    for r in range(3):
        a, b = distributed.shard_range(20001, r, 3)
        op = neighbors.KnnOperator(b - a, 150, 8, 10, out_dtype=np.float64)
        d, i = op.run(xt[a:b].contiguous(), qt, index_base=a)
        dls.append(d)
        ils.append(i)
    od, oi = distributed.merge_topk(torch.stack(dls), torch.stack(ils))
    check(od.cpu().numpy(), oi.cpu().numpy(), ref_d, ref_i, x, q)
    d1, i1 = tb.knn(x, q, 10, out_dtype=np.float64)
    assert np.array_equal(oi.cpu().numpy(), i1)


def test_nccl_process_group_world1():
    """The NCCL code path (SGPR all_reduce of packed Sigma/v/yy, knn_sharded)
    in a real NCCL process group of size 1 on this B200."""
    import socket
    import torch
    import torch.distributed as dist
    from paper_2206_14148_b200 import distributed
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    dist.init_process_group("nccl", init_method=f"tcp://127.0.0.1:{port}", rank=0,
                            world_size=1, device_id=torch.device("cuda", 0))
    try:
        X, y, Z, _ = synthetic.sgpr_data(6000, 3, 200, seed=3, dtype=np.float32)
        e_group = tb.SGPR(X, y, Z, "rbf", 1.0, 0.8, 0.05, group=dist.group.WORLD).elbo()
        e_local = tb.SGPR(X, y, Z, "rbf", 1.0, 0.8, 0.05).elbo()
        assert e_group == e_local
        x, q = synthetic.gaussian_knn(9000, 64, 16, seed=2)
        xt, qt = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
        d, i = distributed.knn_sharded(xt, qt, 5, index_base=0, group=dist.group.WORLD)
        ref_d, ref_i = oknn.exact(x, q, 5)
        check(d.cpu().numpy(), i.cpu().numpy(), ref_d, ref_i, x, q)
        # host buffers in and out (bench e2e at N > 1): shard 1 of 2, offset
        xs = torch.from_numpy(x[4000:]).pin_memory()
        op = neighbors.KnnOperator(5000, 64, 16, 5, out_dtype=np.float64, max_chunk_rows=1200)
        dh, ih = distributed.knn_sharded_host(xs, torch.from_numpy(q).pin_memory(), 5,
                                              index_base=4000, operator=op,
                                              group=dist.group.WORLD)
        sd, si = oknn.exact(x[4000:], q, 5)
        check(dh.numpy(), ih.numpy() - 4000, sd, si, x[4000:], q)
    finally:
        dist.destroy_process_group()


def _near_margin_case(d, seed, n_bg=40000, m=48, planted=40):
    """Background N(0, 1) rows plus, for every query, `planted` rows at
    controlled squared distances r0 + j * delta (j = 0..planted-1) below the
    query's nearest background distance, with delta swept over six decades
    (1e-6 .. 10 of r0): the k-th and K'-th candidate scores are then placed
    from far inside to far outside the engine's error bound E, and with
    small delta many candidates fall inside one rounding interval."""
    rng = np.random.default_rng(seed)
    xb = rng.standard_normal((n_bg, d)).astype(np.float32)
    q = rng.standard_normal((m, d)).astype(np.float32)
    bg_d, _ = oknn.exact(xb, q, 1)
    rows = []
    for r in range(m):
        r0 = 0.25 * float(bg_d[r, 0])
        delta = r0 * 10.0 ** (-6 + (r % 7))
        delta = min(delta, 0.5 * (float(bg_d[r, 0]) - r0) / planted)
        u = rng.standard_normal((planted, d))
        u /= np.linalg.norm(u, axis=1, keepdims=True)
        rad = np.sqrt(r0 + delta * np.arange(planted))
        rows.append(q[r].astype(np.float64) + rad[:, None] * u)
    x = np.concatenate([xb, np.concatenate(rows).astype(np.float32)])
    perm = rng.permutation(x.shape[0])           # planted rows spread over all tiles
    return x[perm], q


@pytest.mark.parametrize("engine", ["tc1", "tc3"])
@pytest.mark.parametrize("d", [16, 128, 784])
def test_certification_near_margin_is_exact(engine, d):
    """Adversarial certification (capi.cu error model): candidates placed at
    controlled gaps around the bound E.  Every returned answer - certified
    by T* - E > exact k-th or recomputed by the exact fallback - must equal
    the fp64 oracle exactly (indices, ties to the lower index), and the
    near-tie queries must actually take the fallback (the bound is live)."""
    x, q = _near_margin_case(d, seed=100 + d, n_bg=40000 if d < 784 else 12000)
    k = 10
    ref_d, ref_i = oknn.exact(x, q, k)
    res = tb.knn(x, q, k, engine=engine, return_result=True)
    assert np.array_equal(res.idx, ref_i), np.nonzero((res.idx != ref_i).any(axis=1))
    assert rel_err(res.dist, ref_d) < 1e-6
    assert res.fallback_queries > 0            # the 1e-6 r0 spacings cannot be certified
    assert res.fallback_queries < q.shape[0]   # the wide ones are


@pytest.mark.parametrize("engine", ["tc1", "tc3"])
def test_certification_scaled_duplicates(engine):
    """Groups of rows at exactly equal distance (mirror images q +- v and
    exact duplicates) straddling the k-th position: certification must hand
    back the lower indices of the tie group, on both engines."""
    rng = np.random.default_rng(21)
    d, m = 64, 32
    xb = rng.standard_normal((30000, d)).astype(np.float32)
    q = np.round(rng.standard_normal((m, d)) * 8).astype(np.float32) / 8
    rows = []
    for r in range(m):
        v = np.round(rng.standard_normal((6, d)) * 4) / 64      # exact in f32
        rows += [q[r] + v, q[r] - v, q[r] + v]                  # 18 rows, 6 distances x 3
    x = np.concatenate([xb, np.concatenate(rows).astype(np.float32)])
    perm = rng.permutation(x.shape[0])
    x = x[perm]
    ref_d, ref_i = oknn.exact(x, q, 10)
    d_, i_ = tb.knn(x, q, 10, engine=engine)
    assert np.array_equal(i_, ref_i)
    assert np.array_equal(d_.astype(np.float64), ref_d.astype(np.float32).astype(np.float64)) or \
        rel_err(d_, ref_d) < 1e-7
