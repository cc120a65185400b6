# cfg5 step variance vs the stream-ordered pool's release threshold
for keep in 2 1000 2 1000; do
  echo "== CSC_POOL_KEEP_GB=$keep"; CSC_POOL_KEEP_GB=$keep timeout 900 python tools/cfg5_steps.py --steps 8 2>&1 | grep "step" | sed 's/.*step \([0-9.]*\) ms.*laplacian \([0-9.]*\).*kmeans \([0-9.]*\) |.*/\1(L\2,K\3)/'
done
