"""Kernel MVM at the paper's §5.1 size: y = K v, K the
n x n squared-exponential kernel over 1-D inputs (build_kernel_mvm,
frontend.py:34-54), n = 1e6, fp64 (the paper's "double precision").
Inputs resident on the device; CUDA events; prints one JSON line."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2206_14148_b200 import mvm

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=1_000_000)
ap.add_argument("--reps", type=int, default=3)
ap.add_argument("--dim", type=int, default=1)
a = ap.parse_args()
g = torch.Generator(device="cuda")
g.manual_seed(3)
x = torch.rand((a.n, a.dim), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
y = torch.rand((a.n, a.dim), generator=g, device="cuda", dtype=torch.float64) * 2 - 1
v = torch.rand(a.n, generator=g, device="cuda", dtype=torch.float64) * 2 - 1
mvm.kernel_mvm(x[:4096], y, v, "rbf", 1.0, 0.1)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    out = mvm.kernel_mvm(x, y, v, "rbf", 1.0, 0.1)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
ms = min(ts)
print(json.dumps({"workload": f"se_kernel_mvm_n{a.n}_d{a.dim}_f64", "ms": ms, "mvm_per_s": 1e3 / ms,
                  "kernel_evals_per_s": a.n * a.n / (ms * 1e-3), "checksum": float(out.sum())}))
