"""Per-kernel GPU time of one packed SGPR gradient (tb_sgpr_grad_run) at
C4 shape with N reduced (CUPTI via torch.profiler)."""
import collections, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2206_14148_b200 as tb
N = int(sys.argv[1]) if len(sys.argv) > 1 else 200_000
d, M = 11, 10_000
g = torch.Generator(device="cuda"); g.manual_seed(77)
X = torch.randn((N, d), generator=g, device="cuda")
y = torch.sin(X.double().sum(1)).float()
g.manual_seed(5)
Z = torch.randn((M, d), generator=g, device="cuda")
tb.SGPR(X[:4096], y[:4096], Z[:256].contiguous(), "rbf", 1.0, 1.0, 0.01).elbo_and_grads()
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB")
m.statistics(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.elbo_and_grads(); torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0]); span = [1e30, 0]
for e in prof.events():
    if e.device_type.name == "CUDA":
        k = e.name.split("(")[0][:60]
        agg[k][0] += 1; agg[k][1] += (e.time_range.end - e.time_range.start) / 1000
        span[0] = min(span[0], e.time_range.start); span[1] = max(span[1], e.time_range.end)
print(f"span {(span[1] - span[0]) / 1000:.1f} ms")
for k, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"{t:9.2f} ms {c:6d}  {k}")
