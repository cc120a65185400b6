# A/B of the sweep's row-group width / vectors per lane at one workload (env knobs CSC_SWEEP_G, CSC_VPL)
WL=${WL:-cfg5}; D=${D:-48}; P=${P:-fp64}
for round in 1 2; do
  for cfg in "0 0" "8 0" "16 0" "32 0" "8 4" "16 4" "4 0"; do
    set -- $cfg
    echo "== G=$1 VPL=$2 round $round $(CSC_SWEEP_G=$1 CSC_VPL=$2 timeout 300 python tools/time_sweep.py --workload $WL --precision $P --d $D --orders 20 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["ms_per_order"],3), round(d["gbs_bmin"]))')"
  done
done
