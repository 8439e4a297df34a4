import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_2206_14148_b200._lib as _L
if os.environ.get("FBLIB"): _L.LIB_PATH = os.path.join(os.path.dirname(_L.LIB_PATH), os.environ["FBLIB"])
from paper_2206_14148_b200 import neighbors
n, m, k = 200_000, 2000, 10
rng = np.random.default_rng(0)
a = ((rng.standard_normal((200, 32)) * 10)[rng.integers(0, 200, n + m)]
     + 0.01 * rng.standard_normal((n + m, 32))).astype(np.float32)
x, q = torch.from_numpy(a[:n]).cuda(), torch.from_numpy(a[n:]).cuda()
op = neighbors.KnnOperator(n, m, 32, k, engine="tc1")
for _ in range(2):
    op.run(x, q)
torch.cuda.synchronize()
print("fallback", op.fallback_count(), "plan lists/cand", int(op.plan.cand))
