"""C3 at full size on ONE B200 (BASELINE.json configs[2]: 1e7 x 784 f32
database, 1e4 queries, k = 10, sharded over 8 ranks): the 8 shards of the
multi-GPU partition (distributed.shard_range) are processed one after the
other by the same per-rank code path (KnnOperator on the shard, fp64 output,
index_base = the shard's first global row), their lists are merged by
tb_topk_merge (the NCCL all_gather is the only step not exercised), and the
result is checked against the exact fp64 oracle over the WHOLE 1e7-row
database for a query sample.  Prints one JSON line: per-shard times (the
per-GPU cost of an 8-GPU run) and the parity report.

    python tools/knn_c3_full.py [--rows 10000000] [--check 16]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2206_14148_b200 import distributed, neighbors
from oracle import knn as oknn

ap = argparse.ArgumentParser()
ap.add_argument("--rows", type=int, default=10_000_000)
ap.add_argument("--m", type=int, default=10_000)
ap.add_argument("--d", type=int, default=784)
ap.add_argument("--world", type=int, default=8)
ap.add_argument("--check", type=int, default=16)
a = ap.parse_args()
k = 10
g = torch.Generator(device="cuda")
g.manual_seed(11)
x = torch.randn((a.rows, a.d), generator=g, device="cuda")
q = torch.randn((a.m, a.d), generator=g, device="cuda")
dl, il, shard_ms = [], [], []
for r in range(a.world):
    s, e = distributed.shard_range(a.rows, r, a.world)
    op = neighbors.KnnOperator(e - s, a.m, a.d, k, out_dtype=np.float64)
    xs = x[s:e]
    op.run(xs, q, index_base=s)                          # warm-up (plan, maps)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    d, i = op.run(xs, q, index_base=s)
    e1.record()
    torch.cuda.synchronize()
    shard_ms.append(e0.elapsed_time(e1))
    dl.append(d.clone())
    il.append(i.clone())
    del op
dls, ils = torch.stack(dl), torch.stack(il)
distributed.merge_topk(dls, ils)                         # warm-up (lazy module load)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
od, oi = distributed.merge_topk(dls, ils)
e1.record()
torch.cuda.synchronize()
merge_ms = e0.elapsed_time(e1)
# exact fp64 check over the whole database for a query sample
sel = np.random.default_rng(0).choice(a.m, a.check, replace=False)
xh = x.cpu().numpy()
qh = q[torch.from_numpy(sel).cuda()].cpu().numpy()
t0 = time.time()
ref_d, ref_i = oknn.exact(xh, qh, k)
rep = oknn.compare(od[torch.from_numpy(sel).cuda()].cpu().numpy(),
                   oi[torch.from_numpy(sel).cuda()].cpu().numpy(), ref_d, ref_i, xh, qh)
print(json.dumps({"workload": f"knn_c3_{a.rows}x{a.d}_q{a.m}_k{k}_shards{a.world}",
                  "shard_ms": shard_ms, "max_shard_ms": max(shard_ms), "merge_ms": merge_ms,
                  "queries_per_s_8gpu_projection": a.m / ((max(shard_ms) + merge_ms) / 1e3),
                  "note": "per-GPU time of an 8-GPU run = max shard + merge (NCCL all_gather of "
                          "2 x 1.6 MB not included)",
                  "oracle_check_queries": int(a.check), "oracle_s": time.time() - t0,
                  "parity": rep}))
