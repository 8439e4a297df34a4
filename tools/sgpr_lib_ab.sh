#!/bin/bash
# Same-box A/B of two library builds on the SGPR C4 statistics pass
# (tools/sgpr_bench.py), alternating old / new.
for rep in 1 2; do
  for lib in libtb_pairwise_old.so libtb_pairwise.so; do
    out=$(timeout 300 python tools/probes/ab_lib.py $lib --script tools/sgpr_bench.py "$@" 2>&1 | tail -1)
    echo "$lib :: $out"
  done
done
