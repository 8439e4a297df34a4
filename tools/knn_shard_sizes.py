"""Per-rank C2 step time at the shard sizes of N = 1, 2, 4, 8 GPUs (the
database split, all 1e4 queries on every rank): what strong scaling can
reach before the all_gather + merge.
    python tools/knn_shard_sizes.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_14148_b200 import neighbors

g = torch.Generator(device="cuda")
g.manual_seed(1)
x = torch.randn((1_000_000, 128), generator=g, device="cuda")
q = torch.randn((10_000, 128), generator=g, device="cuda")
for world in (1, 2, 4, 8):
    n = 1_000_000 // world
    xs = x[:n]
    op = neighbors.KnnOperator(n, 10_000, 128, 10, memory_limit="1GB")
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record()
    for _ in range(3):
        op.run(xs, q)
    torch.cuda.synchronize()
    best, eng = 1e9, 0
    for _ in range(10):
        ev[2].record()
        op.run(xs, q, events=ev[:2])
        ev[3].record()
        torch.cuda.synchronize()
        t = ev[2].elapsed_time(ev[3])
        if t < best:
            best, eng = t, ev[0].elapsed_time(ev[1])
    print(json.dumps({"world": world, "rows": n, "step_ms": best, "engine_ms": eng,
                      "ideal_ms": None, "rows_per_tile_unit": None}))
    del op
