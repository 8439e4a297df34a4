"""Same-box A/B of two builds of the C-ABI library: run tools/tc_ab.py
against paper_2206_14148_b200/<libname> (build the alternative .so next to
the default one first).

    python tools/probes/ab_lib.py libtb_pairwise_old.so tc1
"""
import sys, os
sys.path.insert(0, "/root/repo")
import paper_2206_14148_b200._lib as L
L.LIB_PATH = os.path.join(os.path.dirname(L.LIB_PATH), sys.argv[1])
sys.argv = [sys.argv[0]] + sys.argv[2:]
exec(open("/root/repo/tools/tc_ab.py").read())
