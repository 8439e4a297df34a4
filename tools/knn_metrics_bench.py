"""kNN throughput per metric at the C2 shape (1e6 x 128 database, 1e4
queries, k = 10, f32, 1 GB) on one B200: l2 / cosine on tensor cores, l1 on
CUDA cores (no tensor-core form).

    python tools/knn_metrics_bench.py [--metrics l2,cosine,l1]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2206_14148_b200 import neighbors

ap = argparse.ArgumentParser()
ap.add_argument("--metrics", default="l2,cosine,l1")
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(1)
x = torch.randn((a.n, 128), generator=g, device="cuda")
q = torch.randn((10_000, 128), generator=g, device="cuda")
for metric in a.metrics.split(","):
    op = neighbors.KnnOperator(a.n, 10_000, 128, 10, metric=metric, memory_limit="1GB")
    op.run(x, q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        op.run(x, q)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    eng = {1: "tc3", 2: "simt", 3: "tc1"}[int(op.plan.engine)]
    print(json.dumps({"metric": metric, "engine": eng, "n": a.n, "ms": ms,
                      "queries_per_s": 1e4 / (ms / 1e3), "chunks": int(op.plan.n_chunks),
                      "cand": int(op.plan.cand), "fallback": op.fallback_count()}))
    del op
