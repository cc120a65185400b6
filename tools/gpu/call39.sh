# feasibility: cfg3 sweep time per order at narrow widths (contiguous n x d blocks)
for d in 8 16 32 128; do
  echo "d=$d $(timeout 300 python tools/time_sweep.py --workload cfg3 --precision fp64 --d $d --orders 20 2>/dev/null)"
done
