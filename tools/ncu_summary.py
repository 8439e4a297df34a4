"""Summarise an ncu --set full report (run here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active": "hmma_inst_pct",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed": "l1_throughput_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "launch__shared_mem_per_block_dynamic": "dyn_smem",
}

UNIT_SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
              "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0,
              "nsecond": 1e-9, "second": 1.0}


def ncu_csv(rep, page, extra=()):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv", *extra],
                         capture_output=True, text=True, check=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    rows = ncu_csv(rep, "raw")
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120]}
        for k, name in KEYS.items():
            if k in hdr:
                i = hdr.index(k)
                v = vals[i].replace(",", "")
                try:
                    f = float(v)
                except ValueError:
                    d[name] = v
                    continue
                u = units[i]
                if name in ("dram_read", "dram_write"):
                    f = f * UNIT_SCALE.get(u, 1)
                elif name == "duration":
                    f = f * UNIT_SCALE.get(u, 1e-9) * 1e3   # -> ms
                elif name == "sm_clock":
                    f = f * (1e9 if u.lower().startswith("g") else 1e6 if u.lower().startswith("m") else 1) / 1e9
                d[name] = f
        res.append(d)
    # stall reasons from the source page
    try:
        src = ncu_csv(rep, "source", ("--print-source", "sass"))
        h = src[1]
        stalls = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
        tot = {s: 0.0 for s in stalls}
        for r in src[2:]:
            for s in stalls:
                try:
                    tot[s] += float(r[h.index(s)] or 0)
                except ValueError:
                    pass
        total = sum(tot.values()) or 1.0
        res[0]["stall_share"] = {k: round(v / total, 3) for k, v in
                                 sorted(tot.items(), key=lambda kv: -kv[1])[:6]}
    except Exception as exc:  # pragma: no cover
        res[0]["stall_share"] = f"unavailable: {exc}"
    return res


if __name__ == "__main__":
    r = summarise(sys.argv[1])
    if "--json" in sys.argv:
        print(json.dumps(r, indent=1))
    else:
        for d in r:
            for k, v in d.items():
                print(f"{k:28s} {v}")
