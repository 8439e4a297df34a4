"""SGPR timing on the GPU box: statistics pass + fp64 tail at a given size."""
import sys, os, time, json, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2206_14148_b200 as tb
ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=2_000_000); ap.add_argument("--M", type=int, default=10_000)
ap.add_argument("--d", type=int, default=11); ap.add_argument("--kernel", default="rbf")
ap.add_argument("--ls", type=float, default=1.0); ap.add_argument("--limit", default="1GB")
ap.add_argument("--engine", default="auto")
a = ap.parse_args()
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((a.N, a.d), generator=g, device="cuda")
y = torch.sin(X.double().sum(1)).float() + 0.1 * torch.randn(a.N, generator=g, device="cuda")
Z = X[torch.randperm(a.N, generator=g, device="cuda")[:a.M]].contiguous()
torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats(); base = torch.cuda.memory_allocated()
m = tb.SGPR(X, y, Z, a.kernel, 1.0, a.ls, 0.01, memory_limit=a.limit, engine=a.engine)
s0 = torch.cuda.Event(enable_timing=True); s1 = torch.cuda.Event(enable_timing=True)
s0.record(); st = m.statistics(); s1.record(); torch.cuda.synchronize()
stats_ms = s0.elapsed_time(s1); peak_stats = torch.cuda.max_memory_allocated() - base + (X.numel()+y.numel()+Z.numel())*4
t0 = time.perf_counter()
try:
    e = m.elbo()
except Exception as ex:          # debug modes (TB_I8_DEBUG) produce garbage statistics
    e = repr(ex)[:80]
torch.cuda.synchronize(); tail_s = time.perf_counter() - t0
flops = a.N * a.M * (a.M + 1)
print(json.dumps({"engine": a.engine, "N": a.N, "M": a.M, "d": a.d, "kernel": a.kernel, "elbo": e, "stats_ms": stats_ms,
  "stats_tflops": flops / (stats_ms / 1e3) / 1e12, "tail_s": tail_s, "chunk_n": int(st.plan.chunk_n),
  "peak_stats_mb": peak_stats / 1e6, "planned_peak_mb": st.plan.peak_bytes / 1e6}))
