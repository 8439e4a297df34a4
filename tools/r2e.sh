timeout 300 python -m pytest tests/test_knn_gpu.py -q -x 2>&1 | grep -E "^E |passed|failed" | head
python tools/probes/ab_lib.py libtb_pairwise_old.so tc3
python tools/probes/ab_lib.py libtb_pairwise.so tc3
python tools/probes/ab_lib.py libtb_pairwise_old.so tc3
python tools/probes/ab_lib.py libtb_pairwise.so tc3
