"""e2e (host buffers through tb_knn_run_host) vs the database chunk cap, C2."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2206_14148_b200 import neighbors
n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda"); g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda"); q = torch.randn((m, d), generator=g, device="cuda")
xh, qh = x.cpu().pin_memory(), q.cpu().pin_memory()
for parts in [int(v) for v in (sys.argv[1] if len(sys.argv) > 1 else "2,4,8,16").split(",")]:
    cap = (-(-n // parts) + 255) // 256 * 256          # whole tiles: `parts` chunks
    op = neighbors.KnnOperator(n, m, d, k, memory_limit="1GB", max_chunk_rows=cap)
    out = op.alloc_outputs()
    dh = torch.empty(out[0].shape, dtype=out[0].dtype).pin_memory()
    ih = torch.empty(out[1].shape, dtype=torch.int64).pin_memory()
    st = (x, q, out[0], out[1])
    for _ in range(3): op.run_host(xh, qh, (dh, ih), staging=st)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): op.run_host(xh, qh, (dh, ih), staging=st)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    # host cost of one call's enqueue (no synchronisation inside the call)
    import time
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    op.run_host(xh, qh, (dh, ih), staging=st, synchronize=False)
    enq = (time.perf_counter() - t0) * 1e3
    torch.cuda.synchronize()
    print(json.dumps({"parts": parts, "chunks": int(op.plan.n_chunks), "ms": ms, "qps": m / ms * 1e3,
                      "enqueue_ms": enq}))
    del op
