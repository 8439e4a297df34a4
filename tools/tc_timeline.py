"""Whole-launch timeline of the tc1 engine at C2 (trace build:
make -C paper_2206_14148_b200/csrc trace): per CTA %globaltimer at entry,
every 32nd tile of the MMA issuer and exit, for the seed and the main
launch.  Prints launch spans, the spread of CTA start/end times (tail
imbalance) and the chip-wide tile rate in time bins (slow early phase).
    [TB_TC_DEBUG=8] python tools/tc_timeline.py   (8: no insertions, timing only)"""
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2206_14148_b200._lib as _L
_L.LIB_PATH = os.path.join(os.path.dirname(_L.LIB_PATH), "libtb_pairwise_trace.so")
from paper_2206_14148_b200 import _lib, neighbors

n, m, d, k = 1_000_000, 10_000, 128, 10
g = torch.Generator(device="cuda")
g.manual_seed(0)
x = torch.randn((n, d), generator=g, device="cuda")
q = torch.randn((m, d), generator=g, device="cuda")
op = neighbors.KnnOperator(n, m, d, k, engine="auto", memory_limit="1GB")
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for e in ev:
    e.record()          # creates the underlying cudaEvent_t
for _ in range(3):
    op.run(x, q, events=ev)
torch.cuda.synchronize()
cn = np.zeros(8, np.uint64)
_lib.load().tb_debug_tc_census(ctypes.c_void_p(cn.ctypes.data), 1)
op.run(x, q, events=ev)
torch.cuda.synchronize()
_lib.load().tb_debug_tc_census(ctypes.c_void_p(cn.ctypes.data), 0)
tl = np.zeros((2, 148, 128), np.uint64)
assert _lib.load().tb_debug_tc_timeline(ctypes.c_void_p(tl.ctypes.data)) == 0
tl = tl.astype(np.float64)
t0 = tl[:, :, 0][tl[:, :, 0] > 0].min()
out = {"engine_ms_events": ev[0].elapsed_time(ev[1]),
       "census": {name: {"warp_events": int(cn[4 * li]), "lanes": int(cn[4 * li + 1]),
                         "candidates": int(cn[4 * li + 2]),
                         "candidates_per_query": float(cn[4 * li + 2]) / m}
                  for li, name in ((0, "seed"), (1, "main"))}}
for li, name in ((0, "seed"), (1, "main")):
    a = tl[li][tl[li, :, 0] > 0]          # CTAs of this launch
    start, end, tiles = a[:, 0] - t0, a[:, 127] - t0, a[:, 126]
    first = a[:, 1] - t0
    out[name] = {"entry_us": [float(start.min() / 1e3), float(start.max() / 1e3)],
                 "first_tile_us": [float(first.min() / 1e3), float(np.median(first) / 1e3)],
                 "exit_us": [float(end.min() / 1e3), float(np.median(end) / 1e3),
                             float(end.max() / 1e3)],
                 "tiles_per_cta": [int(tiles.min()), int(np.median(tiles)), int(tiles.max())]}
    if name == "main":
        # ns per tile per CTA in consecutive 32-tile windows
        nt = int(np.median(tiles)) // 32
        w = np.diff(a[:, 1:1 + min(nt, 124)], axis=1) / 32.0      # ns per tile
        prof = np.median(w, axis=0)
        out[name]["ns_per_tile_by_window"] = [round(float(v), 1) for v in prof[::4]]
        out[name]["ns_per_tile_median"] = float(np.median(w))
        out[name]["ns_per_tile_first_256"] = float(np.median(w[:, :8]))
        out[name]["ns_per_tile_last_256"] = float(np.median(w[:, -8:]))
        # time from the last stamp to exit (tail of units)
        out[name]["busy_fraction"] = float(np.sum(end - start) / (len(a) * (end.max() - start.min())))
print(json.dumps(out, indent=1))
