"""Engine tc1 (fp16 single pass, measured-residual bound) vs tc3 (bf16x3)
across data distributions at 2e5 x d, 2000 queries, k = 10: exactness vs
the fp64 oracle on a query subset, uncertified (fallback) queries, time.

    python tools/knn_engine_robustness.py
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import knn as oknn
from paper_2206_14148_b200 import neighbors

n, m, k = 200_000, 2000, 10
rng = np.random.default_rng(0)
cases = {
    "gauss_d128": lambda: rng.standard_normal((n + m, 128)),
    "uniform01_d128": lambda: rng.random((n + m, 128)),
    "offset100_d64": lambda: rng.standard_normal((n + m, 64)) + 100.0,
    "lowrank_d256": lambda: rng.standard_normal((n + m, 8)) @ rng.standard_normal((8, 256)),
    "clustered_d32": lambda: (rng.standard_normal((200, 32)) * 10)[rng.integers(0, 200, n + m)]
                             + 0.01 * rng.standard_normal((n + m, 32)),
    "quantized_d96": lambda: np.round(rng.random((n + m, 96)) * 255) / 255,
    "heavytail_d64": lambda: rng.standard_cauchy((n + m, 64)).clip(-1e4, 1e4),
}
for name, gen in cases.items():
    a = gen().astype(np.float32)
    x, q = a[:n].copy(), a[n:].copy()
    d = x.shape[1]
    sub = np.arange(0, m, 10)
    ref_d, ref_i = oknn.exact(x, q[sub], k)
    xt, qt = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    for eng in ("tc1", "tc3"):
        op = neighbors.KnnOperator(n, m, d, k, engine=eng)
        out = op.alloc_outputs()
        op.run(xt, qt, out); torch.cuda.synchronize()
        t0 = time.perf_counter(); op.run(xt, qt, out); torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        dist, idx = out[0].cpu().numpy(), out[1].cpu().numpy()
        rep = oknn.compare(dist[sub], idx[sub], ref_d, ref_i, x, q[sub])
        print(json.dumps({"case": name, "engine": eng, "ok": bool(rep["ok"]),
                          "fallback": op.fallback_count(), "ms": round(ms, 3)}))
