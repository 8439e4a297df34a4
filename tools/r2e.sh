timeout 300 python -m pytest tests/test_knn_gpu.py -q -x 2>&1 | grep -E "^E |passed|failed" | head -5
python tools/tc_trace.py 0 1000 | head -6
python tools/tc_trace.py 1 1000 | head -6
bash tools/lib_ab.sh 0
