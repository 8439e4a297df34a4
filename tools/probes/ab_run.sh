for dbg in 0 1 2 4 8; do
  for o in 8 4; do echo "dbg=$dbg ovh4=$o"; TB_TC_DEBUG=$dbg TB_TC_OVH4=$o python tools/tc_ab.py tc1; done
done
