# cfg5 step outliers: per-step phases + replay counter, clocks sampled alongside
nvidia-smi --query-gpu=timestamp,clocks.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.sw_power_cap,clocks_event_reasons.hw_slowdown,clocks_event_reasons.sw_thermal_slowdown --format=csv -lms 100 > gpurun_out/c50_clocks.csv &
SMI=$!
timeout 900 python tools/cfg5_steps.py --steps 10 > gpurun_out/c50.log 2>&1
kill $SMI
