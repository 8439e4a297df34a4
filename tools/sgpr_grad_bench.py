"""SGPR ELBO + training gradient at the benchmarked C4 configuration on one
B200, inside memory_limit (the packed gradient tail, tb_sgpr_grad_run):
statistics pass, then the gradient; device peak measured against the limit.

    python tools/sgpr_grad_bench.py [--N 2000000] [--M 10000] [--d 11] [--limit 1GB]
                                    [--tail packed|dense]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200.sizes import as_limit
ap = argparse.ArgumentParser()
ap.add_argument("--N", type=int, default=2_000_000); ap.add_argument("--M", type=int, default=10_000)
ap.add_argument("--d", type=int, default=11); ap.add_argument("--kernel", default="rbf")
ap.add_argument("--limit", default="1GB"); ap.add_argument("--tail", default="packed")
a = ap.parse_args()
g = torch.Generator(device="cuda"); g.manual_seed(77)
X = torch.randn((a.N, a.d), generator=g, device="cuda")
y = (torch.sin(X.double().sum(1)) + 0.1 * torch.randn(a.N, generator=g, device="cuda",
                                                      dtype=torch.float64)).float()
g.manual_seed(5)
Z = torch.randn((a.M, a.d), generator=g, device="cuda")
tb.SGPR(X[:4096], y[:4096], Z[:256].contiguous(), a.kernel, 1.0, 1.0, 0.01).elbo_and_grads()
torch.cuda.synchronize()
limit = None if a.limit == "none" else a.limit
m = tb.SGPR(X, y, Z, a.kernel, 1.0, [1.0] * a.d, 0.01, memory_limit=limit, tail=a.tail)
base = torch.cuda.memory_allocated() - (X.numel() + y.numel() + Z.numel()) * 4
torch.cuda.reset_peak_memory_stats()
t0 = time.perf_counter()
e, gr = m.elbo_and_grads()
torch.cuda.synchronize()
t1 = time.perf_counter()
peak = torch.cuda.max_memory_allocated() - base
print(json.dumps({"N": a.N, "M": a.M, "d": a.d, "kernel": a.kernel, "tail": a.tail, "elbo": e,
                  "elbo_and_grads_s": t1 - t0, "grad_gemm_flops": 2.0 * a.M * a.M * a.N,
                  "grad_variance": gr["variance"], "grad_noise": gr["noise_variance"],
                  "grad_lengthscale0": float(gr["lengthscales"][0]),
                  "max_abs_grad_Z": float(abs(gr["Z"]).max()),
                  "peak_mb_incl_inputs": peak / 1e6,
                  "planned_peak_mb": m.grad_peak_bytes() / 1e6 if a.tail == "packed" else None,
                  "memory_limit": limit}))
