"""Exact-fallback throughput: every query forced through it (TB_FORCE_FALLBACK=1)
at the C2 database (1e6 x 128 f32), 2000 queries; checked against the
default (certified) answer.
    python tools/knn_fallback_bench.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_14148_b200 import neighbors

g = torch.Generator(device="cuda")
g.manual_seed(3)
n, m, d, k = 1_000_000, 2000, 128, 10
x = torch.randn((n, d), generator=g, device="cuda")
q = torch.randn((m, d), generator=g, device="cuda")
ref = neighbors.KnnOperator(n, m, d, k, memory_limit="1GB")
rd, ri = (t.clone() for t in ref.run(x, q))
os.environ["TB_FORCE_FALLBACK"] = "1"
op = neighbors.KnnOperator(n, m, d, k, memory_limit="1GB")
op.run(x, q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
dist, idx = op.run(x, q)
e1.record()
torch.cuda.synchronize()
print(json.dumps({"n": n, "m": m, "d": d, "fallback_queries": op.fallback_count(),
                  "ms": e0.elapsed_time(e1), "ms_per_query": e0.elapsed_time(e1) / m,
                  "same_idx": bool(torch.equal(idx, ri)),
                  "max_dist_rel": float(((dist - rd).abs().max() / rd.abs().max()).item())}))
