"""C3 per-GPU shard (BASELINE.json configs[2]: 1e7 x 784 database over 8
B200 -> 1.25e6 x 784 per GPU, 1e4 queries, k = 10): one rank's fused kNN,
tcgen05 (streamed-query) engine vs the CUDA-core engine, on one B200.

    python tools/knn_c3_shard.py [--rows 1250000] [--engines tc3,simt]
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
ap.add_argument("--rows", type=int, default=1_250_000)
ap.add_argument("--m", type=int, default=10_000)
ap.add_argument("--d", type=int, default=784)
ap.add_argument("--engines", default="tc3,simt")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(7)
x = torch.randn((a.rows, a.d), generator=g, device="cuda")
q = torch.randn((a.m, a.d), generator=g, device="cuda")
for eng in a.engines.split(","):
    op = neighbors.KnnOperator(a.rows, a.m, a.d, 10, engine=eng, out_dtype=np.float64)
    n_ev = 2 * int(op.plan.n_chunks)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(n_ev)]
    for e in evs:             # materialise the cudaEvent_t handles
        e.record()
    op.run(x, q)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        d, i = op.run(x, q, events=evs)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    eng_ms = sum(evs[2 * c].elapsed_time(evs[2 * c + 1]) for c in range(n_ev // 2))
    useful = 2.0 * a.rows * a.m * a.d
    print(json.dumps({"engine": eng, "rows": a.rows, "m": a.m, "d": a.d, "ms": ms,
                      "queries_per_s": a.m / (ms / 1e3), "engine_ms": eng_ms,
                      "useful_tflops": useful / (eng_ms / 1e3) / 1e12,
                      "chunks": int(op.plan.n_chunks), "fallback": op.fallback_count()}))
    del op
