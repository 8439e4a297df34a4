"""CUPTI timeline of a few chunks of the C4 statistics pass: start/end of
every Gram and digit-plane generation launch (is generation c+1 overlapping
Gram c?)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
import paper_2206_14148_b200 as tb
N, d, M = 100_000, 11, 10_000
g = torch.Generator(device="cuda"); g.manual_seed(77)
X = torch.randn((N, d), generator=g, device="cuda"); y = torch.sin(X.double().sum(1)).float()
g.manual_seed(5); Z = torch.randn((M, d), generator=g, device="cuda")
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB"); m.statistics(); torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB")
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    m.statistics(); torch.cuda.synchronize()
ev = sorted((e.time_range.start, e.time_range.end, e.name.split("(")[0][-24:])
            for e in prof.events() if e.device_type.name == "CUDA")
t0 = ev[0][0]
for a, b, n in ev[:40]:
    print(f"{(a - t0) / 1000:8.3f} {(b - t0) / 1000:8.3f} {(b - a) / 1000:7.3f}  {n}")
