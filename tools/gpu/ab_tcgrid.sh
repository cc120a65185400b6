# A/B: tensor-core screen grid cap vs concurrent k-means lanes (cfg5 steps)
for g in 0 128 112 96; do
  echo "== CSC_TC_GRID=$g"; CSC_TC_GRID=$g timeout 600 python tools/cfg5_steps.py --steps 3 2>&1 | grep "^step" | cut -c1-120
done
