import sys, os, json, torch
sys.path.insert(0, "/root/repo")
import paper_2206_14148_b200 as tb
g = torch.Generator(device="cuda"); g.manual_seed(1)
Z = torch.randn((10000, 11), generator=g, device="cuda"); Xs = torch.randn((200000, 11), generator=g, device="cuda")
w = torch.randn(10000, generator=g, device="cuda", dtype=torch.float64)
for _ in range(2): tb.kernel_mvm(Xs, Z, w, "rbf", 1.0, [1.0]*11)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): tb.kernel_mvm(Xs, Z, w, "rbf", 1.0, [1.0]*11)
e1.record(); torch.cuda.synchronize()
print(json.dumps({"predict_ms": e0.elapsed_time(e1) / 5}))
