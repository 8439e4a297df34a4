#!/bin/bash
# One GPU call that refreshes every committed measurement: the GPU test
# suite, the bench line (ours + reference arm), the launch list of the bench
# command, and ncu --set full captures of the kNN engine and the tail potrf.
# Outputs land in gpurun_out/refresh/ (copied into profiles/ by hand).
export PYTHONUNBUFFERED=1
O=gpurun_out/refresh
mkdir -p $O
timeout 900 python -m pytest tests -q -m gpu > $O/gpu_tests.log 2>&1
tail -3 $O/gpu_tests.log
timeout 900 python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
tail -c 400 $O/bench_n1.json
timeout 600 python bench.py --impl reference > $O/bench_ref.json 2> $O/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file $O/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline \
  --no-sgpr --no-e2e > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:knn_tc -s 3 -c 1 \
  -o $O/knn_tc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --no-sgpr \
  > $O/ncu_knn.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tail_potrf -s 3 -c 1 \
  -o $O/tail_potrf python tools/probes/tail_kernels.py > $O/ncu_potrf.log 2>&1
ls -la $O
