# cfg5 steps: concurrent lanes vs one stream (k-means phase variance)
for mode in 0 1 0 1; do
  echo "== CSC_KMEANS_SERIAL=$mode"; CSC_KMEANS_SERIAL=$mode timeout 900 python tools/cfg5_steps.py --steps 8 2>&1 | grep "step" | sed 's/.*step \([0-9.]*\) ms.*kmeans \([0-9.]*\).*/step \1 kmeans \2/'
done
