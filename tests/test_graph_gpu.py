"""graph.evaluate on the B200 path: the device allocation trace, the
poison_freed option and PassConfig.tensor_split_size (reference surface:
interpreter.py:57-76,149-167,522-551; pipeline.py:18-41)."""

import numpy as np
import pytest

from conftest import rel_err
from oracle import knn as oknn
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200 import graph as G

pytestmark = pytest.mark.gpu


def test_trace_records_every_device_buffer():
    g = tb.build_knn(30000, 200, 32, 10, "l2", tb.DType.F32)
    x, q = tb.random_inputs(g, 3)
    (vals, idx), trace = tb.evaluate(g, [x, q], budget="64MB")
    ref_d, ref_i = oknn.exact(x, q, 10)
    assert oknn.compare(vals.array, idx.array.astype(np.int64), ref_d, ref_i, x, q)["ok"]
    kinds = [(e.instruction.split("/")[-1], e.event) for e in trace.events]
    for name in ("param0", "param1", "workspace", "values", "indices"):
        assert (name, "alloc") in kinds and (name, "free") in kinds
    assert trace.events[-1].live_after == 0                 # everything released
    allocs = sum(e.bytes for e in trace.events if e.event == "alloc")
    assert x.nbytes + q.nbytes <= trace.peak_live_bytes <= 64 * 10**6
    assert trace.peak_live_bytes >= allocs - 4 * 2**20        # measured, not planned
    assert trace.to_csv().splitlines()[0] == "instruction,event,bytes,live_after"


def test_poison_freed_keeps_results_and_trace():
    g = tb.build_knn(5000, 40, 16, 5, "l2", tb.DType.F64)
    x, q = tb.random_inputs(g, 4)
    (v1, i1), t1 = tb.evaluate(g, [x, q])
    (v2, i2), t2 = tb.evaluate(g, [x, q], poison_freed=True)
    assert np.array_equal(i1.array, i2.array) and np.array_equal(v1.array, v2.array)
    assert [(e.instruction, e.event, e.bytes) for e in t1.events] == \
        [(e.instruction, e.event, e.bytes) for e in t2.events]
    g2 = tb.build_kernel_mvm(3000, tb.KernelSpec(1.2, 0.3))
    xs = tb.random_inputs(g2, 5)
    o1, _ = tb.evaluate(g2, xs)
    o2, t3 = tb.evaluate(g2, xs, poison_freed=True)
    assert np.array_equal(o1.array, o2.array) and t3.events[-1].live_after == 0


def test_tensor_split_size_caps_the_staged_slice():
    """run_pipeline(PassConfig(tensor_split_size=...)) bounds the database
    slice each chunk stages: 30000 x 32 f32 rows with a 1 MB split size plan
    several chunks and give the same answer as the unsplit call."""
    g = tb.build_knn(30000, 100, 32, 10, "l2", tb.DType.F32)
    x, q = tb.random_inputs(g, 6)
    cfg = tb.PassConfig(tensor_size_threshold=10**7, tensor_split_size=10**6)
    gp = tb.run_pipeline(g, cfg)
    assert G._split_cap_rows(gp, 32, 4) == 10**6 // 128
    p = tb.neighbors.plan(30000, 100, 32, 10, dtype=np.float32,
                          max_chunk_rows=G._split_cap_rows(gp, 32, 4))
    assert p.n_chunks >= 4 and p.chunk_rows * 32 * 4 <= 10**6
    (v1, i1), _ = tb.evaluate(g, [x, q])
    (v2, i2), _ = tb.evaluate(gp, [x, q])
    assert np.array_equal(i1.array, i2.array)
    assert rel_err(v2.array, v1.array) == 0.0


def test_mvm_budget_counts_the_fp64_buffers():
    """f32 MVM: x, y in f32 plus v and the output in fp64 = 24 n bytes on the
    device; a budget of 16 n (the f32 tensors alone) must raise."""
    n = 4096
    g = tb.build_kernel_mvm(n, tb.KernelSpec(), tb.DType.F32)
    xs = tb.random_inputs(g, 7)
    with pytest.raises(tb.BudgetExceeded):
        tb.evaluate(g, xs, budget=16 * n)
    out, trace = tb.evaluate(g, xs, budget=24 * n + 4 * 2**20)
    assert trace.peak_live_bytes >= 24 * n
