import sys, time
sys.path.insert(0, "/root/repo")
import torch
import paper_2206_14148_b200 as tb
g = torch.Generator(device="cuda"); g.manual_seed(77)
X = torch.randn((2_000_000, 11), generator=g, device="cuda")
y = (torch.sin(X.double().sum(1)) + 0.1 * torch.randn(X.shape[0], generator=g, device="cuda", dtype=torch.float64)).float()
g.manual_seed(5)
Z = torch.randn((10_000, 11), generator=g, device="cuda")
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01, memory_limit="1GB")
t0 = time.time(); e = m.elbo(); torch.cuda.synchronize()
print("C4 elbo", e, "cond_kuu_lb %.3e" % m.cond_kuu_lb, "engine", m.engine, "s %.3f" % (time.time() - t0))
