"""Engine time at C2 vs the seed-launch length (TB_TC_SEED tiles): the seed
publishes the per-query thresholds the main launch filters with.
    python tools/seed_sweep.py [4,8,16,32,64]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_14148_b200 import neighbors

seeds = [int(s) for s in (sys.argv[1] if len(sys.argv) > 1 else "4,8,16,32,64").split(",")]
n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda")
g.manual_seed(1)
x = torch.randn((n, d), generator=g, device="cuda")
q = torch.randn((m, d), generator=g, device="cuda")
res = {s: [] for s in seeds}
for rep in range(3):
    for s in seeds:
        os.environ["TB_TC_SEED"] = str(s)
        op = neighbors.KnnOperator(n, m, d, k, memory_limit="1GB")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        for e in ev:
            e.record()
        best = 1e9
        for _ in range(5):
            op.run(x, q, events=ev)
            torch.cuda.synchronize()
            best = min(best, ev[0].elapsed_time(ev[1]))
        res[s].append(best)
        del op
for s in seeds:
    print(json.dumps({"seed_tiles": s, "engine_ms": res[s]}))
