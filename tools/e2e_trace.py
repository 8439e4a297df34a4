"""CUPTI trace (torch.profiler) of the e2e host-buffer kNN step at C2, set up
exactly as bench.py does; prints the GPU activity timeline of one step."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
dev = torch.device("cuda", 0)
torch.cuda.set_device(0)
g = torch.Generator(device=dev)
g.manual_seed(1234)
x = torch.randn((n, d), generator=g, device=dev, dtype=torch.float32)
g.manual_seed(99)
q = torch.randn((m, d), generator=g, device=dev, dtype=torch.float32)
op = neighbors.KnnOperator(n, m, d, k, dtype=np.float32, out_dtype=np.float32, memory_limit=10**9, device=dev)
out = op.alloc_outputs()
for _ in range(13): op.run(x, q, out)
torch.cuda.synchronize()
xh = x.cpu().pin_memory(); qh = q.cpu().pin_memory()
op_h = neighbors.KnnOperator(n, m, d, k, dtype=np.float32, out_dtype=np.float32, memory_limit=10**9,
                             device=dev, max_chunk_rows=-(-n // 8))
staging = (x, q, out[0], out[1])
dh = torch.empty(out[0].shape, dtype=out[0].dtype).pin_memory()
ih = torch.empty(out[1].shape, dtype=out[1].dtype).pin_memory()
step = lambda: op_h.run_host(xh, qh, (dh, ih), staging=staging)
for _ in range(3): step()
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(3): step()
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type.name == "CUDA":
        evs.append((e.time_range.start, e.time_range.end, e.name[:60]))
evs.sort()
t0 = evs[0][0]
for s, e, nm in evs:
    print(f"{(s - t0) / 1000:9.3f} {(e - s) / 1000:8.3f}  {nm}")
