#!/bin/bash
# Same-box A/B of two library builds (old = libtb_pairwise_old.so) on the
# C2 tc1 engine, alternating, for each TB_TC_DEBUG mode given (default 0;
# modes other than 0 act only in study builds: make trace, -DTB_TC_TRACE).
modes="${@:-0}"
for rep in 1 2 3; do
  for mode in $modes; do
    for lib in libtb_pairwise_old.so libtb_pairwise.so; do
      out=$(TB_TC_DEBUG=$mode timeout 300 python tools/probes/ab_lib.py $lib auto 2>&1 | tail -1)
      echo "$lib mode=$mode :: $out"
    done
  done
done
