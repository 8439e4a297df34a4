"""CPU-only checks of the C-ABI library: it loads, exports every symbol
include/tb_pairwise.h declares, and its planner honours memory_limit
(no compute calls — there is no GPU here)."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200 import _lib, neighbors as tknn
from paper_2206_14148_b200.sizes import format_size, parse_size


def header_symbols():
    text = open(os.path.join(ROOT, "include", "tb_pairwise.h")).read()
    return sorted(set(re.findall(r"TB_API\s+[\w\s\*]+?\b(tb_\w+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    declared = header_symbols()
    assert len(declared) >= 9
    for name in declared:
        assert hasattr(lib, name), name
    assert set(declared) == set(_lib.EXPORTED)


def test_struct_layouts_match_c():
    assert ctypes.sizeof(_lib.KnnPlan) == 256
    assert ctypes.sizeof(_lib.SgprPlan) == 168


def test_capabilities_and_error_string():
    lib = _lib.load()
    caps = lib.tb_capabilities()
    assert caps >> 16 >= 1
    assert isinstance(_lib.last_error(), str)


# ---------------------------------------------------------------- sizes

@pytest.mark.parametrize("text,value", [
    ("1GB", 10**9), ("100MB", 10**8), ("64MiB", 64 * 2**20), ("2KB", 2000),
    ("1.5GB", 1_500_000_000), ("512", 512), ("1GiB", 2**30), (" 3 KiB", 3072)])
def test_parse_size_reference_semantics(text, value):
    assert parse_size(text) == value


@pytest.mark.parametrize("bad", ["", "GB", "1.5B", "abc", "-1GB"])
def test_parse_size_rejects(bad):
    with pytest.raises(ValueError):
        parse_size(bad)


def test_format_size():
    assert format_size(10**9) == "1GB"
    assert format_size(2**20) == "1MiB"
    assert format_size(1234) == "1234B"


# ---------------------------------------------------------------- planner

C2 = dict(n=1_000_000, m=10_000, d=128, k=10)


@pytest.mark.parametrize("engine", ["simt", "tc3"])
def test_c2_plan_fits_one_gb(engine):
    p = tknn.plan(**C2, dtype=np.float32, memory_limit="1GB", engine=engine)
    assert p.peak_bytes <= 10**9
    assert p.resident_bytes == (C2["n"] + C2["m"]) * C2["d"] * 4
    # peak = resident + buffers as a caching allocator charges them
    # (512-B granules up to 1 MiB, 2 MiB above): never below the exact sum
    exact = p.resident_bytes + p.workspace_bytes + p.output_bytes
    assert exact <= p.peak_bytes <= exact + 3 * (2 << 20)
    assert p.n_chunks * p.chunk_rows >= C2["n"]
    assert p.cand >= C2["k"]


def test_plan_chunks_when_limit_tightens():
    loose = tknn.plan(**C2, dtype=np.float32, engine="tc3")
    tight = tknn.plan(**C2, dtype=np.float32, engine="tc3", memory_limit="700MB")
    assert tight.peak_bytes <= 700 * 10**6
    assert tight.n_chunks >= loose.n_chunks
    assert tight.chunk_rows <= loose.chunk_rows


def test_plan_budget_exceeded_before_allocation():
    with pytest.raises(tb.BudgetExceeded) as info:
        tknn.plan(**C2, dtype=np.float32, memory_limit="500MB")
    assert "budget" in str(info.value)
    assert info.value.live == (C2["n"] + C2["m"]) * C2["d"] * 4


def test_plan_monotone_in_limit():
    peaks = []
    for lim in ("600MB", "800MB", "1GB", "4GB", None):
        p = tknn.plan(**C2, dtype=np.float32, memory_limit=lim, engine="tc3")
        if lim:
            assert p.peak_bytes <= parse_size(lim)
        peaks.append(p.peak_bytes)
    assert peaks == sorted(peaks)


@pytest.mark.parametrize("k,n", [(0, 10), (11, 10), (-1, 5)])
def test_plan_rejects_bad_k_like_build_knn(k, n):
    with pytest.raises(ValueError, match="must satisfy"):
        tknn.plan(n, 4, 3, k)


def test_plan_rejects_unknown_metric():
    with pytest.raises(ValueError, match="metric"):
        tknn.plan(10, 4, 3, 2, metric="cheb")


def test_plan_small_shapes():
    for n, m, d, k in [(1, 1, 1, 1), (3, 1, 1, 2), (16, 6, 3, 4), (5000, 0, 7, 5)]:
        p = tknn.plan(n, m, d, k, dtype=np.float64)
        assert p.workspace_bytes > 0
        assert p.n_chunks == 1


def test_plan_f64_out():
    p = tknn.plan(1000, 10, 8, 3, dtype=np.float32, out_dtype=np.float64)
    assert p.output_bytes == 10 * 3 * (8 + 8)


# ------------------------------------------------------------ graph surface

def test_build_knn_validation_mirrors_reference():
    with pytest.raises(ValueError, match="must satisfy"):
        tb.build_knn(5, 2, 3, 6)
    with pytest.raises(ValueError, match="metric"):
        tb.build_knn(5, 2, 3, 2, metric="hamming")
    g = tb.build_knn(16, 6, 3, 4)
    assert g.name == "knn_l2_n16_m6_d3_k4"
    assert [p.dims for p in g.parameters] == [(16, 3), (6, 3)]


def test_passconfig_invariants():
    c = tb.PassConfig(tensor_size_threshold=1000)
    assert c.tensor_split_size == 1000
    with pytest.raises(ValueError):
        tb.PassConfig(tensor_size_threshold=100, tensor_split_size=200)
    with pytest.raises(ValueError):
        tb.PassConfig(tensor_size_threshold=0)


def test_evaluate_rejects_bad_inputs_before_device_work():
    g = tb.build_knn(16, 6, 3, 4)
    with pytest.raises(tb.EvaluationError):
        tb.evaluate(g, [np.zeros((16, 3))])
    with pytest.raises(tb.EvaluationError):
        tb.evaluate(g, [np.zeros((16, 3)), np.zeros((6, 4))])
    with pytest.raises(tb.EvaluationError):
        tb.evaluate(g, [np.zeros((16, 3), np.float32), np.zeros((6, 3), np.float32)])


def test_random_inputs_match_reference_generator():
    g = golden("knn_c1_uniform.npz")
    graph = tb.build_knn(int(g["n"]), int(g["m"]), int(g["d"]), int(g["k"]))
    ins = tb.random_inputs(graph, seed=int(g["seed"]))
    import hashlib
    h = hashlib.sha256()
    for a in ins:
        h.update(a.tobytes())
    assert h.hexdigest() == str(g["sha"])


def test_estimate_peak_memory_is_planner_peak():
    g = tb.build_knn(10_000, 1_000, 16, 10)
    est = tb.estimate_peak_memory(g)
    assert est >= (10_000 + 1_000) * 16 * 8
    # far below the reference's naive-graph peak (it materialises [m,n,d])
    assert est < int(golden("budget.npz")["knn_c1_naive_peak"])


def test_sgpr_planner_engines_and_c4_budget():
    """C4 (N=2e6, d=11, M=1e4, f32, 1 GB): the fixed-point engine keeps Sigma
    as packed lower tiles (414 MB), so two 7808-point chunk buffers fit (Kuf
    generation of chunk c+1 overlaps the Gram of chunk c); the fp64 engine
    keeps the full 800 MB Sigma and gets a much smaller chunk."""
    from paper_2206_14148_b200 import sgpr
    N, M, d = 2_000_000, 10_000, 11
    resident = (N * d + N + M * d) * 4
    p = sgpr.plan(N, M, d, kernel="rbf", memory_limit="1GB", resident_bytes=resident)
    assert p.engine == _lib.SGPR_ENGINES["i8"] and p.sigma_layout == _lib.TB_SIGMA_TILES
    assert p.M_pad == 10_112
    assert p.sigma_bytes == (79 * 80 // 2) * 128 * 128 * 8
    assert p.off[4] == 2 and p.chunk_n == 7808 and p.peak_bytes <= 1_000_000_000
    assert p.off[6] <= p.peak_bytes              # the packed O(M^3) tail fits too
    with pytest.raises(tb.BudgetExceeded, match="tail"):
        sgpr.plan(N, M, d, kernel="rbf", memory_limit="900MB", resident_bytes=resident)
    tight = sgpr.plan(200_000, 2000, d, kernel="rbf", memory_limit="60MB")
    assert tight.chunk_n < 10_880 and tight.peak_bytes <= 60_000_000
    small = sgpr.plan(5000, 300, 4, kernel="rbf")
    assert small.off[4] == 1 and small.chunk_n == 5120          # one chunk: no overlap
    f = sgpr.plan(N, M, d, kernel="rbf", memory_limit="1GB", resident_bytes=resident,
                  engine="f64")
    assert f.sigma_layout == _lib.TB_SIGMA_FULL and f.sigma_bytes == M * M * 8
    assert f.chunk_n < p.chunk_n and f.peak_bytes <= 1_000_000_000
    with pytest.raises(ValueError):
        sgpr.plan(N, M, d, engine="tf32")
    with pytest.raises(tb.BudgetExceeded):
        sgpr.plan(N, M, d, memory_limit="500MB", resident_bytes=resident)


def test_fixed24_oracle_is_a_small_perturbation():
    """oracle.sgpr.sufficient_stats_fixed24 (the i8 engine's exact numerics)
    vs the unquantised fp64 statistics: same ELBO to ~1e-8 on a small case."""
    import numpy as np
    from oracle import sgpr as osgpr
    from paper_2206_14148_b200 import synthetic
    X, y, Z, _ = synthetic.sgpr_data(3000, 3, 120, seed=3, dtype=np.float64)
    S, v, yy = osgpr.sufficient_stats(X, y, Z, "matern32", 1.0, 0.6)
    Sq, vq, yyq = osgpr.sufficient_stats_fixed24(X, y, Z, "matern32", 1.0, 0.6)
    assert np.abs(Sq - S).max() <= 1e-7 * np.abs(S).max()
    K = osgpr.kuu(Z, "matern32", 1.0, 0.6)
    e, _ = osgpr.elbo_from_stats(S, v, yy, 3000, K, 0.01, 1.0)
    eq, _ = osgpr.elbo_from_stats(Sq, vq, yyq, 3000, K, 0.01, 1.0)
    assert abs(eq - e) <= 1e-8 * abs(e)
