import os, sys, json
sys.path.insert(0, "/root/repo")
import paper_2206_14148_b200._lib as _L
_L.LIB_PATH = os.path.join(os.path.dirname(_L.LIB_PATH), "libtb_pairwise_trace.so")
exec(open("/root/repo/tools/knn_shard_sizes.py").read())
