"""SGPR ELBO + gradient timing (statistics pass, autograd tail, N-streaming
gradient pass) at a C4-shaped size on one B200.

    python tools/sgpr_grad_bench.py [--N 200000] [--M 10000] [--d 11]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_14148_b200 as tb
ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=200_000); ap.add_argument("--M", type=int, default=10_000)
ap.add_argument("--d", type=int, default=11); ap.add_argument("--kernel", default="rbf")
ap.add_argument("--chunk", type=int, default=8192)
a = ap.parse_args()
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((a.N, a.d), generator=g, device="cuda")
y = torch.sin(X.double().sum(1)).float() + 0.1 * torch.randn(a.N, generator=g, device="cuda")
Z = X[torch.randperm(a.N, generator=g, device="cuda")[:a.M]].contiguous()
tb.SGPR(X[:4096], y[:4096], Z[:256].contiguous(), a.kernel, 1.0, 1.0, 0.01).elbo_and_grads()
torch.cuda.synchronize()
m = tb.SGPR(X, y, Z, a.kernel, 1.0, [1.0] * a.d, 0.01)   # the gradient tail is O(M^2) > 1 GB at M = 1e4
t0 = time.perf_counter(); m.statistics(); torch.cuda.synchronize(); t1 = time.perf_counter()
e, gr = m.elbo_and_grads(chunk_n=a.chunk); torch.cuda.synchronize(); t2 = time.perf_counter()
print(json.dumps({"N": a.N, "M": a.M, "d": a.d, "kernel": a.kernel, "elbo": e,
                  "stats_s": t1 - t0, "tail_and_grad_s": t2 - t1,
                  "grad_gemm_flops": 2.0 * a.M * a.M * a.N,
                  "grad_variance": gr["variance"], "grad_noise": gr["noise_variance"],
                  "max_abs_grad_Z": float(abs(gr["Z"]).max()),
                  "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}))
