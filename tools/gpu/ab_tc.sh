# A/B of tc screen variants (abv/tc_*.so) on one box: host-driven Lloyd iterations, screen per-launch times
for round in 1 2; do
  for v in "$@"; do
    echo "== $v round $round"
    CSC_LIB=abv/tc_$v.so timeout 300 python tools/profile_screen_iter.py 60 tc 2>&1 | grep "per-iteration screen\|GPU total"
  done
done
