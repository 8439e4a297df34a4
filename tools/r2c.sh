export PYTHONUNBUFFERED=1
mkdir -p gpurun_out/r2c
TB_TC_STAGES=5 TB_TC_EXTBUF=3 timeout 600 python -m pytest tests/test_knn_gpu.py -q -x -k "golden or c2" 2>&1 | tail -2
bash tools/tc_env_ab.sh 2>&1 | tee gpurun_out/r2c/ab.txt
