"""Measured INT8 tensor-core peak on this B200 via cuBLASLt (torch._int_mm),
the i8 analogue of MEASURED_PEAKS.json's bf16 figure: best of 10 (burst) and
back to back for ~3 s (sustained)."""
import json
import time

import torch

n = 8192
a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda")
b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device="cuda").t().contiguous().t()
for _ in range(3):
    torch._int_mm(a, b)
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); torch._int_mm(a, b); e1.record(); e1.synchronize()
    best = max(best, 2 * n ** 3 / (e0.elapsed_time(e1) * 1e-3) / 1e12)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps, t0 = 0, time.time()
e0.record()
while time.time() - t0 < 3.0:
    for _ in range(20):
        torch._int_mm(a, b)
    reps += 20
    torch.cuda.synchronize()
e1.record(); e1.synchronize()
sus = 2 * n ** 3 * reps / (e0.elapsed_time(e1) * 1e-3) / 1e12
print(json.dumps({"int8_tops_burst": best, "int8_tops_sustained": sus,
                  "how": "torch._int_mm 8192^3 int8->int32 (cuBLASLt), best of 10 / 3 s loop"}))
