"""Pinned host->device bandwidth for 517 MB with 1/2/4 concurrent copy streams."""
import torch, json
n = 517_120_000 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = [(i * n // ns, (i + 1) * n // ns) for i in range(ns)]
    def go():
        cur = torch.cuda.current_stream()
        ev = torch.cuda.Event(); ev.record(cur)
        for s, (a, b) in zip(streams, parts):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                d[a:b].copy_(h[a:b], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
    for _ in range(2): go()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(5): go()
    b.record(); torch.cuda.synchronize()
    ms = a.elapsed_time(b) / 5
    print(json.dumps({"streams": ns, "ms": ms, "GBs": n * 4 / ms / 1e6}))
