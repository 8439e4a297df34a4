import sys, time, torch, math
sys.path.insert(0, '/root/repo')
import paper_2206_14148_b200 as tb
from paper_2206_14148_b200.sgpr import kernel_matrix
N, M, d = 200000, 10000, 11
g = torch.Generator(device="cuda"); g.manual_seed(0)
X = torch.randn((N, d), generator=g, device="cuda"); y = torch.randn(N, generator=g, device="cuda")
Z = X[:M].contiguous()
m = tb.SGPR(X, y, Z, "rbf", 1.0, 1.0, 0.01)
s = m.statistics(); torch.cuda.synchronize()
def T(label, f):
    torch.cuda.synchronize(); t0 = time.perf_counter(); r = f(); torch.cuda.synchronize()
    print(f"{label:28s} {1e3*(time.perf_counter()-t0):8.1f} ms"); return r
for rep in range(2):
    Kuu = T("kernel_matrix Kuu", lambda: kernel_matrix(m.Z, m.Z, "rbf", 1.0, m.lengthscales))
    L = T("cholesky Kuu", lambda: torch.linalg.cholesky(Kuu))
    S = T("unpack Sigma", lambda: s.full_sigma())
    tmp = T("trsm L^-1 Sigma", lambda: torch.linalg.solve_triangular(L, S, upper=False))
    AAT = T("trsm (.)L^-T", lambda: torch.linalg.solve_triangular(L, tmp.mT, upper=False).mT)
    AAT = T("symmetrize+scale", lambda: 0.5 * (AAT + AAT.mT) / 0.01)
    LB = T("cholesky B", lambda: torch.linalg.cholesky(AAT + torch.eye(M, device="cuda", dtype=torch.float64)))
    T("full _tail()", lambda: m._tail())
