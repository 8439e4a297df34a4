"""C2 with the single-pass bf16 engine (tc1): engine time, end-to-end time
and how many queries fail certification (exact fallback)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda"); g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda"); q = torch.randn((m, d), generator=g, device="cuda")
for eng in sys.argv[1:] or ["tc3", "tc1"]:
    op = neighbors.KnnOperator(n, m, d, k, engine=eng, memory_limit="1GB")
    out = op.alloc_outputs()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(2 * int(op.plan.n_chunks))]
    for e in evs: e.record()
    for _ in range(3): op.run(x, q, out)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); op.run(x, q, out, events=evs); b.record(); torch.cuda.synchronize()
    eng_ms = sum(evs[2*c].elapsed_time(evs[2*c+1]) for c in range(int(op.plan.n_chunks)))
    print(json.dumps({"engine": eng, "cand": int(op.plan.cand), "engine_ms": eng_ms,
                      "total_ms": a.elapsed_time(b), "fallback": op.fallback_count()}))
