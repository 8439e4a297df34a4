import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2206_14148_b200 as tb
N, M, d = 50000, 10000, 11
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((N, d), generator=g, device="cuda"); y = torch.randn(N, generator=g, device="cuda")
m = tb.SGPR(X, y, X[:M].contiguous(), "rbf", 1.0, 1.0, 0.01)
m.elbo(); torch.cuda.synchronize()
