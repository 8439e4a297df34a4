"""Where the e2e (host-buffer) kNN step at C2 spends its time: chunked H2D
alone, compute alone on the same 8-chunk plan, and the overlapped run_host
call, each timed with CUDA events (one B200)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
parts = int(sys.argv[1]) if len(sys.argv) > 1 else 8
g = torch.Generator(device="cuda"); g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda"); q = torch.randn((m, d), generator=g, device="cuda")
if len(sys.argv) > 2:          # as bench.py: a 2-chunk operator alive and used first
    op2 = neighbors.KnnOperator(n, m, d, k, dtype=np.float32, out_dtype=np.float32,
                                memory_limit="1GB")
    out2 = op2.alloc_outputs()
    for _ in range(13): op2.run(x, q, out2)
    torch.cuda.synchronize()
xh, qh = x.cpu().pin_memory(), q.cpu().pin_memory()
op = neighbors.KnnOperator(n, m, d, k, memory_limit="1GB", max_chunk_rows=-(-n // parts))
out = op.alloc_outputs()
dh = torch.empty(out[0].shape, dtype=out[0].dtype).pin_memory()
ih = torch.empty(out[1].shape, dtype=torch.int64).pin_memory()
st = (x, q, out[0], out[1])
E = lambda: torch.cuda.Event(enable_timing=True)


def timed(fn, reps=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = E(), E()
    a.record()
    for _ in range(reps): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


cr = int(op.plan.chunk_rows)
def h2d_chunks():
    for c0 in range(0, n, cr):
        x[c0:c0 + cr].copy_(xh[c0:c0 + cr], non_blocking=True)
    q.copy_(qh, non_blocking=True)
res = {"parts": parts, "chunks": int(op.plan.n_chunks),
       "h2d_chunked_ms": timed(h2d_chunks),
       "compute_ms": timed(lambda: op.run(x, q, out=out)),
       "run_host_ms": timed(lambda: op.run_host(xh, qh, (dh, ih), staging=st))}
# per-chunk compute with events
evs = [E() for _ in range(2 * int(op.plan.n_chunks))]
for e in evs: e.record()
op.run(x, q, out=out, events=evs); torch.cuda.synchronize()
res["chunk_engine_ms"] = [round(evs[2*c].elapsed_time(evs[2*c+1]), 3) for c in range(int(op.plan.n_chunks))]
print(json.dumps(res))
