import sys, os, json
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np
import test_knn_fuzz_gpu as T
import paper_2206_14148_b200 as tb
from oracle import knn as oknn
seed = int(sys.argv[1])
rng = np.random.default_rng(1000 + seed)
metric = ["l2", "cosine", "l1"][seed % 3]
kind = ["gauss", "offset", "quantized", "clustered", "duplicates"][seed % 5]
n = int(rng.integers(1, 30_000)); m = int(rng.integers(1, 300))
d = int(rng.choice([1, 3, 8, 31, 64, 96, 128, 130, 300])); k = int(rng.integers(1, min(64, n) + 1))
dtype = np.float32 if seed % 2 else np.float64
engine = "simt" if metric == "l1" else str(rng.choice(["auto", "tc1", "tc3", "simt"]))
if metric == "cosine" and engine == "simt": engine = "tc1"
x, q = (a.astype(dtype) for a in T._data(rng, kind, n, m, d))
if metric == "cosine":
    x[np.all(x == 0, axis=1)] = 1.0; q[np.all(q == 0, axis=1)] = 1.0
print(metric, kind, n, m, d, k, dtype, engine)
inputs = (n + m) * d * np.dtype(dtype).itemsize
limit = None
if rng.random() < 0.5:
    full = tb.neighbors.plan(n, m, d, k, metric=metric, dtype=dtype, engine=engine).peak_bytes
    limit = inputs + max(int((full - inputs) * rng.uniform(0.3, 0.9)), 4 * 2**20)
res = tb.knn(x, q, k, metric=metric, engine=engine, memory_limit=limit, out_dtype=np.float64, return_result=True)
ref_d, ref_i = oknn.exact(x, q, k, metric=metric)
rep = oknn.compare(res.dist, res.idx, ref_d, ref_i, x, q, metric=metric)
print({kk: v for kk, v in rep.items() if kk != "bad"} if isinstance(rep, dict) else rep)
bad = np.argwhere(res.idx != ref_i)
print("limit", limit, "fallback", res.fallback_queries, "n_bad_positions", len(bad))
for r, c in bad[:8]:
    gi, ri = res.idx[r, c], ref_i[r, c]
    print(r, c, "got", gi, res.dist[r, c], "ref", ri, ref_d[r, c], "x_got", x[gi], "x_ref", x[ri], "q", q[r])
dd = np.abs(res.dist - ref_d)
r, c = np.unravel_index(np.argmax(dd), dd.shape)
print("max diff at", r, c, "got", res.dist[r], "ref", ref_d[r], "idx got", res.idx[r], "ref", ref_i[r])
print("rel_err denominators: max|ref|", np.max(np.abs(ref_d)), "max|diff|", dd.max())
