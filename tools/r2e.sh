python tools/tc_trace.py 0 1000
python tools/tc_trace.py 1 1000
bash tools/lib_ab.sh 0 1
