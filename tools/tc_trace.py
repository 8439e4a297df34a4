"""Timing study of the tc1 engine (TB_TC_DEBUG bit 16): clock64 stamps of the
MMA issuer and of epilogue warp 2 for the first 64 tiles of every CTA's main
launch, read back from the candidate-index region.  Prints where the
issuer waits (tempty, efull, full stages) and the epilogue's per-tile span.
    TB_TC_DEBUG=16 python tools/tc_trace.py [extra debug bits, e.g. 7]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2206_14148_b200._lib as _L
_L.LIB_PATH = os.path.join(os.path.dirname(_L.LIB_PATH), "libtb_pairwise_trace.so")   # make -C ... trace

extra = int(sys.argv[1]) if len(sys.argv) > 1 else 0
t0 = int(sys.argv[2]) if len(sys.argv) > 2 else 0       # first traced tile of each CTA
os.environ["TB_TC_DEBUG"] = str(16 | extra | (t0 << 8))
from paper_2206_14148_b200 import neighbors

n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda")
g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda")
q = torch.randn((m, d), generator=g, device="cuda")
op = neighbors.KnnOperator(n, m, d, k, engine="auto", memory_limit="1GB")
for _ in range(3):
    op.run(x, q)
torch.cuda.synchronize()
import ctypes
from paper_2206_14148_b200 import _lib
tr = np.zeros((148, 2048), np.int64)
assert _lib.load().tb_debug_tc_trace(ctypes.c_void_p(tr.ctypes.data)) == 0
mma = tr[:, :512].reshape(148, 64, 8).astype(np.float64)
epi = tr[:, 1024:1536].reshape(148, 64, 8).astype(np.float64)
sl = slice(8, 60)        # steady state
mm = mma[:, sl]
ee = epi[:, sl]
per_tile = np.diff(mma[:, sl, 0], axis=1)
print(f"debug={16 | extra} tiles {t0}..{t0 + 63}  MMA issuer, cycles per tile (median over CTAs): "
      f"{np.median(per_tile):.0f}")
names = ["wait tempty", "wait full kb0", "kb0->full kb1", "kb1->end(commit)"]
segs = [mm[..., 1] - mm[..., 0], mm[..., 3] - mm[..., 1],
        mm[..., 4] - mm[..., 3], mm[..., 7] - mm[..., 4]]
for nm, sg in zip(names, segs):
    print(f"  {nm:18s} median {np.median(sg):7.0f}  mean {np.mean(sg):7.0f}")
ep_tile = np.diff(epi[:, sl, 0], axis=1)
print(f"epilogue warp 2: cycles per tile {np.median(ep_tile):.0f}")
names = ["wait tfull", "loads->release", "release->publish", "publish->next"]
segs = [ee[..., 1] - ee[..., 0], ee[..., 2] - ee[..., 1], ee[..., 3] - ee[..., 2],
        epi[:, 9:61, 0] - ee[..., 3]]
for nm, sg in zip(names, segs):
    print(f"  {nm:18s} median {np.median(sg):7.0f}  mean {np.mean(sg):7.0f}")
segs = [ee[..., 5] - ee[..., 3], epi[:, 9:61, 4] - ee[..., 5], ee[..., 0] - ee[..., 4]]
for nm, sg in zip(["publish->end", "end->top(i+1)", "top->ready"], segs):
    print(f"  {nm:18s} median {np.median(sg):7.0f}  mean {np.mean(sg):7.0f}")
# latency from the issuer's commit of tile i to the epilogue seeing tfull
lat = ee[..., 1] - mm[..., 7]
print(f"  commit(i) -> epilogue sees tfull(i): median {np.median(lat):.0f}")
rel = mma[:, 10:62, 1] - ee[..., 2]
print(f"  epilogue release(i) -> issuer passes tempty(i+2): median {np.median(rel):.0f}")
