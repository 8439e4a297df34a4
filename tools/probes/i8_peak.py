"""Measured INT8 tensor-core peak for the SGPR roofline: the tcgen05 kind::i8
probe (tools/probes/i8_peak_probe, the Gram's own instruction on all SMs,
burst + a >= 4 s sustained launch) with nvidia-smi clocks sampled during the
sustained launch, plus cuBLASLt int8 (torch._int_mm) for comparison.
Writes one JSON object (profiles/r02_i8_peak.json)."""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

HERE = os.path.dirname(os.path.abspath(__file__))
secs = float(sys.argv[1]) if len(sys.argv) > 1 else 5.0
q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.sw_power_cap,"
     "clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown")
smi = subprocess.Popen(["nvidia-smi", "-i", "0", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                        "-lms", "100"], stdout=subprocess.PIPE, text=True)
lines = []
threading.Thread(target=lambda: [lines.append(l.strip()) for l in smi.stdout], daemon=True).start()
time.sleep(1.0)
t0 = time.time()
out = subprocess.run([os.path.join(HERE, "i8_peak_probe"), str(secs)], capture_output=True,
                     text=True).stdout.strip().splitlines()[-1]
t1 = time.time()
smi.terminate()
res = json.loads(out)
sm, pw, reasons = [], [], set()
for l in lines[int(1.0 / 0.1) + 3:]:          # samples inside the probe's run (skip warm-up)
    p = [v.strip() for v in l.split(",")]
    try:
        sm.append(float(p[0])); pw.append(float(p[2]))
    except (ValueError, IndexError):
        continue
    for name, v in zip(("sw_power_cap", "hw_slowdown", "sw_thermal_slowdown"), p[3:6]):
        if v.lower().startswith("active"):
            reasons.add(name)
res["clocks"] = {"sm_mhz_median": statistics.median(sm) if sm else None,
                 "power_w_max": max(pw) if pw else None, "reasons": sorted(reasons),
                 "samples": len(sm)}
if sm:
    f = statistics.median(sm) * 1e6
    res["i8_tops_floor_at_median_clock"] = 16384 * res["sms"] * f / 1e12
try:
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
    res["cublaslt_int8_tops_burst"] = best
except Exception as exc:             # pragma: no cover
    res["cublaslt_int8_tops_burst"] = repr(exc)[:80]
res["how"] = ("tools/probes/i8_peak.py: all-SM tcgen05 kind::i8 M128N128K32 loop, best of 5 x "
              "20k-iteration launches (burst) and one launch of ~%.0f s (sustained); "
              "floor = 16384 int8 ops/cycle/SM at the median sampled SM clock" % secs)
print(json.dumps(res))
