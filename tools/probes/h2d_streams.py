"""Pinned host -> device copy bandwidth of the C2 database (512 MB): one
stream vs chunks alternating over two / four streams (copy engines)."""
import json, sys, torch
x = torch.randn((1_000_000, 128)).pin_memory()
d = torch.empty((1_000_000, 128), device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunks = 20
    rows = 1_000_000 // chunks
    def run():
        for c in range(chunks):
            s = streams[c % ns]
            with torch.cuda.stream(s):
                d[c * rows:(c + 1) * rows].copy_(x[c * rows:(c + 1) * rows], non_blocking=True)
    for _ in range(2): run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        e0.record(torch.cuda.current_stream())
        for s in streams: s.wait_event(e0)
        run()
        for s in streams: torch.cuda.current_stream().wait_stream(s)
        e1.record(torch.cuda.current_stream()); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(json.dumps({"streams": ns, "ms": best, "GB_s": 512e6 / (best / 1e3) / 1e9}))
