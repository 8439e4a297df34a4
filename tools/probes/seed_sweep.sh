# Same-box sweep of the seed-launch length (TB_TC_SEED) on C2, engines tc1/tc3.
for i in 1 2; do
  for s in 8 2 3 4 6 16; do echo "seed=$s"; TB_TC_SEED=$s python tools/tc_ab.py tc1; done
done
