import os, sys, json
sys.path.insert(0, "/root/repo")
import torch
from paper_2206_14148_b200 import neighbors
g = torch.Generator(device="cuda"); g.manual_seed(1)
x = torch.randn((125_000, 128), generator=g, device="cuda")
q = torch.randn((10_000, 128), generator=g, device="cuda")
for rep in range(2):
    for s in (1, 2, 4, 8, 16):
        os.environ["TB_TC_SEED"] = str(s)
        op = neighbors.KnnOperator(125_000, 10_000, 128, 10, memory_limit="1GB")
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        for e in ev: e.record()
        for _ in range(3): op.run(x, q)
        best = 1e9
        for _ in range(8):
            ev[2].record(); op.run(x, q, events=ev[:2]); ev[3].record(); torch.cuda.synchronize()
            best = min(best, ev[2].elapsed_time(ev[3]))
        print(json.dumps({"seed": s, "step_ms": round(best, 4), "fallback": op.fallback_count()}))
