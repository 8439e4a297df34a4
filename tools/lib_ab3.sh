#!/bin/bash
# same-box A/B/C of library builds on the C2 tc1 engine: bash tools/lib_ab3.sh libA.so libB.so ...
for rep in 1 2 3; do
  for lib in "$@"; do
    out=$(timeout 300 python tools/probes/ab_lib.py $lib auto 2>&1 | tail -1)
    echo "$lib :: $out"
  done
done
