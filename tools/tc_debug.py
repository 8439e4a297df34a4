"""Quick tcgen05-engine sanity check on the GPU box (prints, never hangs long)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2206_14148_b200 as tb
from oracle import knn as oknn

for (n, m, d, k, eng) in [(512, 128, 64, 10, "tc3"), (256, 128, 64, 10, "tc3"), (5000, 300, 128, 10, "tc3"),
                          (5000, 300, 128, 10, "tc1"), (100000, 1000, 128, 10, "tc3"), (3000, 77, 16, 5, "tc3")]:
    rng = np.random.default_rng(n + d)
    x = rng.standard_normal((n, d)).astype(np.float32)
    q = rng.standard_normal((m, d)).astype(np.float32)
    t = time.time()
    res = tb.knn(x, q, k, engine=eng, return_result=True)
    dt = time.time() - t
    ref_d, ref_i = oknn.exact(x, q, k)
    rep = oknn.compare(res.dist, res.idx, ref_d, ref_i, x, q)
    print(n, m, d, k, eng, f"{dt:.2f}s", "fallback", res.fallback_queries,
          {kk: rep[kk] for kk in ("ok", "identical", "tie_swaps", "mismatches", "bad_index", "dist_rel_err")}, flush=True)
