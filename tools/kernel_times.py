"""Per-kernel GPU time of one C2 kNN call (CUPTI via torch.profiler), averaged
over a few calls: where the step goes outside the candidate engine."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda"); g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda"); q = torch.randn((m, d), generator=g, device="cuda")
op = neighbors.KnnOperator(n, m, d, k, dtype=np.float32, memory_limit="1GB")
out = op.alloc_outputs()
for _ in range(3): op.run(x, q, out)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
R = 5
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(R): op.run(x, q, out)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type.name == "CUDA":
        kname = e.name.split("(")[0][:60]
        agg[kname][0] += 1; agg[kname][1] += (e.time_range.end - e.time_range.start) / 1000
tot = sum(v[1] for v in agg.values())
print(f"per call: {tot / R:.3f} ms of GPU time")
for kname, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t / R:8.3f} ms/call {c // R:4d} launches/call  {kname}")
