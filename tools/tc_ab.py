"""A/B timing of the tcgen05 engine on C2 (events around the engine only)."""
import sys, os, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda"); g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda"); q = torch.randn((m, d), generator=g, device="cuda")
op = neighbors.KnnOperator(n, m, d, k, engine=sys.argv[1] if len(sys.argv) > 1 else "tc3", memory_limit="1GB")
evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * int(op.plan.n_chunks))]
for e in evs: e.record()
for _ in range(3): op.run(x, q)
torch.cuda.synchronize()
t = []
for _ in range(5):
    op.run(x, q, events=evs); torch.cuda.synchronize()
    t.append([evs[2*c].elapsed_time(evs[2*c+1]) for c in range(int(op.plan.n_chunks))])
print(json.dumps({"TB_TC_DEBUG": os.environ.get("TB_TC_DEBUG", "0"), "chunk_ms": t[-1], "total_ms": min(sum(r) for r in t)}))
