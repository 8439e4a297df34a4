mkdir -p gpurun_out/r2f
python tools/probes/i8_peak.py 6 > gpurun_out/r2f/i8_peak.json; cat gpurun_out/r2f/i8_peak.json
./tools/probes/fp64_peak_probe | tee gpurun_out/r2f/fp64_peak.json
python tools/mvm_bench.py --n 1000000 --reps 2 | tee gpurun_out/r2f/mvm_1e6.json
ncu --set full --clock-control none -k regex:kernel_mvm -c 1 -o gpurun_out/r2f/mvm python tools/mvm_bench.py --n 200000 --reps 1 > gpurun_out/r2f/ncu_mvm.log 2>&1
tail -2 gpurun_out/r2f/ncu_mvm.log
