export PYTHONUNBUFFERED=1
TB_TC_STAGES=5 TB_TC_EXTBUF=3 timeout 600 python -m pytest tests/test_knn_gpu.py -q -x -k "golden or c2" 2>&1 | grep -E "Error|assert|FAIL|passed|failed" | head -20
timeout 600 python -m pytest tests/test_knn_gpu.py -q -x -k "golden or c2" 2>&1 | tail -2
cat > /tmp/ab.txt <<'EOT'
TB_TC_MC=0
TB_TC_MC=0 TB_TC_DEBUG=3
TB_TC_MC=0 TB_TC_DEBUG=1
TB_TC_DEBUG=7
TB_TC_MC=0 TB_TC_DEBUG=7
TB_TC_DEBUG=2
EOT
bash tools/tc_env_ab.sh /tmp/ab.txt
