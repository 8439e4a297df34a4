"""Per-kernel time of the packed SGPR tail at M = 1e4 (CUPTI via torch.profiler)."""
import sys, collections, torch
sys.path.insert(0, '/root/repo')
import paper_2206_14148_b200 as tb
N, M, d = 100000, 10000, 11
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((N, d), generator=g, device="cuda"); y = torch.randn(N, generator=g, device="cuda")
Z = X[:M].contiguous()
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01)
m.statistics(); m.elbo(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
m2 = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01)
m2.statistics(); torch.cuda.synchronize()
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m2.elbo(); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
span = [1e30, 0]
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:70]
        agg[k][0] += 1; agg[k][1] += (e.time_range.end - e.time_range.start) / 1000
        span[0] = min(span[0], e.time_range.start); span[1] = max(span[1], e.time_range.end)
print(f"span {(span[1]-span[0])/1000:.2f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f"{t:9.3f} ms {c:6d}  {k}")
