"""Steady-state packed vs dense SGPR tail at M = 1e4 (C4 shape, N = 2e5)."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2206_14148_b200 as tb
N, M, d = 200000, 10000, 11
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((N, d), generator=g, device="cuda"); y = torch.randn(N, generator=g, device="cuda")
Z = X[:M].contiguous()
for tail in ("packed", "dense", "packed", "dense"):
    m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, tail=tail)
    m.statistics(); torch.cuda.synchronize(); torch.cuda.reset_peak_memory_stats()
    t0 = time.perf_counter(); e = m.elbo(); torch.cuda.synchronize()
    print(tail, f"{1e3 * (time.perf_counter() - t0):.1f} ms", e,
          f"peak {torch.cuda.max_memory_allocated() / 1e9:.2f} GB")
