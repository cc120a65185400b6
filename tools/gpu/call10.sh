timeout 120 python tools/tc_screen_check.py --n 20000 > gpurun_out/c10_tc.log 2>&1; echo "tc small rc=$?"; tail -3 gpurun_out/c10_tc.log
timeout 120 python tools/tc_screen_check.py --n 2000000 >> gpurun_out/c10_tc.log 2>&1; echo "tc big rc=$?"; tail -3 gpurun_out/c10_tc.log
timeout 120 python tools/tc_screen_check.py --n 300000 --d 128 --k 100 >> gpurun_out/c10_tc.log 2>&1; echo "tc cfg3 rc=$?"; tail -3 gpurun_out/c10_tc.log
timeout 600 python -m pytest tests/test_gpu_kmeans_fused.py -x -q > gpurun_out/c10_tests.log 2>&1; echo "km tests rc=$?"; tail -5 gpurun_out/c10_tests.log
CSC_KMEANS_TC=1 timeout 300 python tools/kmeans_cfg5_profile.py --reps 3 > gpurun_out/c10_km_tc.log 2>&1; echo "tc rc=$?"; grep "^kmeans" gpurun_out/c10_km_tc.log
CSC_KMEANS_TC=0 timeout 300 python tools/kmeans_cfg5_profile.py --reps 3 > gpurun_out/c10_km_simt.log 2>&1; echo "simt rc=$?"; grep "^kmeans" gpurun_out/c10_km_simt.log
