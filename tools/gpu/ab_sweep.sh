# A/B of sweep library variants (abv/sw_*.so) on one box: ms per order via tools/time_sweep.py
WL=${WL:-cfg4}; D=${D:-64}
for round in 1 2; do
  for v in "$@"; do
    for p in fp32 fp64; do
      echo "== $v $p round $round $(CSC_LIB=abv/sw_$v.so timeout 300 python tools/time_sweep.py --workload $WL --precision $p --d $D --orders 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_order"],3), round(d["gbs_bmin"]))')"
    done
  done
done
