# round 2: cfg5 step variance across configurations (phase-synced)
for p in 0.5 0.25 0.5 0.0 0.5; do
  echo "== p=$p"; timeout 600 python tools/cfg5_steps.py --steps 4 --p $p 2>&1 | grep -v "Warn\|warn"
done > gpurun_out/c36_var.log 2>&1
