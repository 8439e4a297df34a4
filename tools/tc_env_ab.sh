#!/bin/bash
# Same-box A/B of tc1 engine knobs: each line = one env setting, C2 engine ms
# (tools/tc_ab.py, min over 5 calls), repeated twice in alternating order.
for rep in 1 2; do
  while read -r envs; do
    [ -z "$envs" ] && continue
    out=$(env $envs timeout 300 python tools/tc_ab.py auto 2>&1 | tail -1)
    echo "$envs :: $out"
  done < "${1:-tools/tc_env_ab.txt}"
done
