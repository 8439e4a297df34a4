"""Same-box A/B of two builds of the C-ABI library: run a tool script
(default tools/tc_ab.py) against paper_2206_14148_b200/<libname> (build the
alternative .so next to the default one first).

    python tools/probes/ab_lib.py libtb_pairwise_old.so [--script tools/e2e_chunks.py] [args]
"""
import sys, os
sys.path.insert(0, "/root/repo")
import paper_2206_14148_b200._lib as L
L.LIB_PATH = os.path.join(os.path.dirname(L.LIB_PATH), sys.argv[1])
rest = sys.argv[2:]
script = "/root/repo/tools/tc_ab.py"
if rest[:1] == ["--script"]:
    script = os.path.join("/root/repo", rest[1])
    rest = rest[2:]
sys.argv = [script] + rest
exec(open(script).read())
