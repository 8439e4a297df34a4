"""Per-kernel SASS census of the built library objects: counts of the
instructions that prove the sm_100a paths (tcgen05 MMA: UTCHMMA / UTCIMMA /
UTCQMMA; TMA: UTMALDG / UBLKCP; TMEM loads: LDTM; DMMA: DMMA; fp64 FMA: DFMA;
mbarrier waits: SYNCS.PHASECHK).  Run here (no GPU):
    python tools/sass_census.py > profiles/r02_sass_census.txt"""
import glob
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OPS = ("UTCHMMA", "UTCIMMA", "UTCQMMA", "UTMALDG", "UBLKCP", "LDTM", "DMMA", "DFMA",
       "SYNCS.PHASECHK", "ELECT")
objs = sorted(glob.glob(os.path.join(ROOT, "paper_2206_14148_b200", "csrc", "build", "*.o")))
objs = [o for o in objs if "trace" not in o]
print(f"{'object':14s} {'kernel':70s} " + " ".join(f"{o.split('.')[0][:8]:>8s}" for o in OPS))
for obj in objs:
    sass = subprocess.run(["cuobjdump", "-sass", obj], capture_output=True, text=True).stdout
    for block in re.split(r"\n\s*Function : ", sass)[1:]:
        name = block.split("\n", 1)[0].strip()
        demangled = subprocess.run(["c++filt", name], capture_output=True, text=True).stdout.strip()
        counts = [len(re.findall(r"\b" + re.escape(op) + r"\b", block)) for op in OPS]
        if not any(counts[:8]):
            continue
        short = re.sub(r"\(.*", "", demangled)[:70]
        print(f"{os.path.basename(obj):14s} {short:70s} " + " ".join(f"{c:8d}" for c in counts))
