"""Per-kernel GPU time of one SGPR statistics pass at C4 (CUPTI via
torch.profiler): the Gram engine vs the overlapped digit-plane producer."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2206_14148_b200 as tb
N, d, M = 2_000_000, 11, 10_000
g = torch.Generator(device="cuda"); g.manual_seed(77)
X = torch.randn((N, d), generator=g, device="cuda")
y = torch.sin(X.double().sum(1)).float()
g.manual_seed(5)
Z = torch.randn((M, d), generator=g, device="cuda")
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB")
m.statistics(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.statistics(); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0]); span = [1e30, 0]
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:60]
        agg[k][0] += 1; agg[k][1] += (e.time_range.end - e.time_range.start) / 1000
        span[0] = min(span[0], e.time_range.start); span[1] = max(span[1], e.time_range.end)
print(f"span {(span[1] - span[0]) / 1000:.1f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.2f} ms {c:5d}  {k}")
