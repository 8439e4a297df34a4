"""Aggregate an ncu --metrics gpu__time_duration.sum --csv launch list."""
import csv, sys
lines = [l for l in open(sys.argv[1]) if l.startswith('"')]
rows = list(csv.reader(lines))
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value"); ui = h.index("Metric Unit")
agg = {}
order = []
for r in rows[1:]:
    n = r[ki].split("(")[0].replace("void ", "")
    scale = {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(r[ui], 1e-3)
    if n not in agg: order.append(n)
    agg.setdefault(n, []).append(float(r[vi].replace(",", "")) * scale)
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'mean_us':>10s} {'share':>7s}")
for n in order:
    v = agg[n]
    print(f"{n[:48]:48s} {len(v):8d} {sum(v)/len(v):10.1f} {sum(v)/tot:7.1%}")
