timeout 120 python tools/tc_screen_check.py --n 20000 > gpurun_out/c8_tc.log 2>&1; echo "tc small rc=$?"; cat gpurun_out/c8_tc.log | tail -8
timeout 120 python tools/tc_screen_check.py --n 2000000 >> gpurun_out/c8_tc.log 2>&1; echo "tc big rc=$?"; tail -4 gpurun_out/c8_tc.log
timeout 120 python tools/tc_screen_check.py --n 300000 --d 128 --k 100 >> gpurun_out/c8_tc.log 2>&1; echo "tc cfg3 rc=$?"; tail -4 gpurun_out/c8_tc.log
python tools/kmeans_cfg5_profile.py > gpurun_out/c8_km.log 2>&1; tail -40 gpurun_out/c8_km.log
