import sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200 import synthetic
X, y, Z, Xs = synthetic.sgpr_data(3000, 3, 96, seed=1, n_test=50, dtype=np.float32)
m = tb.SGPR(X, y, Z, "matern32", 1.0, 0.7, 0.05)
m.elbo()
print("engine", m.engine, "cond_lb", m.cond_kuu_lb)
