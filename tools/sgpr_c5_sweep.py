"""C5 (BASELINE.json configs[4]): SGPR Matern-3/2, N = 4e5, d = 3
(3droad-shaped synthetic), M swept 1e3 .. 2e4, memory_limit = 1 GB: planned
vs measured peak device bytes of the statistics pass, time, ELBO.  A point
whose statistics or packed O(M^3) tail cannot fit the limit is recorded as an
empty row (the
reference's bench CSV does the same for infeasible points, cli.py:184-186).

    python tools/sgpr_c5_sweep.py [--limit 1GB] [--out gpurun_out/c5.json]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2206_14148_b200 as tb

ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=400_000)
ap.add_argument("--limit", default="1GB")
ap.add_argument("--Ms", default="1000,2000,5000,10000,20000")
ap.add_argument("--out", default=None)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(3)
X = torch.randn((a.N, 3), generator=g, device="cuda")
y = torch.sin(X.double().sum(1)).float() + 0.1 * torch.randn(a.N, generator=g, device="cuda")
tb.SGPR(X[:4096], y[:4096], X[:256].contiguous(), "matern32", 1.0, 0.5, 0.01).elbo()  # warm-up
rows = []
for M in [int(v) for v in a.Ms.split(",")]:
    Z = X[torch.randperm(a.N, generator=g, device="cuda")[:M]].contiguous()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    torch.cuda.reset_peak_memory_stats()
    base = torch.cuda.memory_allocated() - (X.numel() + y.numel() + Z.numel()) * 4
    m = tb.SGPR(X, y, Z, "matern32", 1.0, 0.5, 0.01, memory_limit=a.limit)
    row = {"M": M, "N": a.N, "limit": a.limit}
    try:
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st = m.statistics()
        e1.record()
        torch.cuda.synchronize()
        row.update(stats_ms=e0.elapsed_time(e1),
                   peak_stats_mb=(torch.cuda.max_memory_allocated() - base) / 1e6,
                   planned_peak_mb=st.plan.peak_bytes / 1e6, chunk_n=int(st.plan.chunk_n),
                   chunk_buffers=int(st.plan.off[4]),
                   useful_tflops=a.N * M * (M + 1) / (e0.elapsed_time(e1) / 1e3) / 1e12)
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        row["elbo"] = m.elbo()            # packed in-place tail: inside the same budget
        t1.record()
        torch.cuda.synchronize()
        row["tail_ms"] = t0.elapsed_time(t1)
        row["peak_eval_mb"] = (torch.cuda.max_memory_allocated() - base) / 1e6
    except tb.BudgetExceeded as ex:
        row["infeasible"] = str(ex)[:160]
    rows.append(row)
    print(json.dumps(row), flush=True)
    del m
if a.out:
    with open(a.out, "w") as fh:
        json.dump(rows, fh, indent=1)
