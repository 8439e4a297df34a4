#!/bin/bash
# Same-box A/B of N library builds on the C2 tc1 engine, alternating, 3 reps:
#   tools/lib_abn.sh libtb_pairwise_v0.so libtb_pairwise_vp.so ...
for rep in 1 2 3; do
  for lib in "$@"; do
    out=$(TB_TC_DEBUG=${MODE:-0} timeout 300 python tools/probes/ab_lib.py $lib auto 2>&1 | tail -1)
    echo "$lib :: $out"
  done
done
