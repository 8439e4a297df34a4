export PYTHONUNBUFFERED=1
O=gpurun_out/r2a
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 900 python -m pytest tests -q -m gpu -x > $O/gpu_tests.log 2>&1
tail -3 $O/gpu_tests.log
timeout 600 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
tail -c 600 $O/bench_n1.json
