export PYTHONUNBUFFERED=1
O=gpurun_out/r2b
mkdir -p $O
./tools/probes/tmem_ld_probe > $O/tmem_probe.txt 2>&1
cat $O/tmem_probe.txt
timeout 900 python -m pytest tests/test_sgpr_gpu.py -q -x -k "c4" > $O/sgpr_c4_tests.log 2>&1
tail -15 $O/sgpr_c4_tests.log
