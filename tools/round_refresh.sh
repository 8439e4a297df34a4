#!/bin/bash
# One GPU call that refreshes every committed measurement: the GPU test
# suite, the bench line (ours + reference arm), the C3 shard, the launch
# list of the bench command, and ncu --set full captures of the kNN engine
# and the SGPR Gram.  Outputs land in gpurun_out/refresh/ (copied into
# profiles/ by hand).
export PYTHONUNBUFFERED=1
O=gpurun_out/refresh
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt
timeout 1200 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
tail -3 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
tail -c 400 $O/bench_n1.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 python tools/knn_c3_shard.py --engines tc1,tc3 > $O/c3_shard.jsonl 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-sgpr --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_tc -s 3 -c 1 \
  -o $O/knn_tc1 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sgpr \
  > $O/ncu_knn.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sgpr_gram_i8 -s 2 -c 1 \
  -o $O/sgpr_gram_i8 python tools/sgpr_bench.py > $O/ncu_sgpr.log 2>&1
ls -la $O
