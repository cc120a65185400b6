timeout 120 python tools/tc_screen_check.py --n 2000000 > gpurun_out/c17_tc.log 2>&1; echo "tc big rc=$?"; tail -3 gpurun_out/c17_tc.log
timeout 120 python tools/tc_screen_check.py --n 300000 --d 128 --k 100 >> gpurun_out/c17_tc.log 2>&1; echo "tc cfg3 rc=$?"; tail -2 gpurun_out/c17_tc.log
timeout 600 python -m pytest tests/test_gpu_kmeans_fused.py -x -q > gpurun_out/c17_tests.log 2>&1; echo "km tests rc=$?"; tail -3 gpurun_out/c17_tests.log
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c17_iter.log 2>&1; echo "iter rc=$?"; grep -v "Warning\|warn" gpurun_out/c17_iter.log | grep -A14 "mode="
timeout 300 python tools/cfg5_steps.py > gpurun_out/c17_cfg5.log 2>&1; echo "cfg5 rc=$?"; tail -6 gpurun_out/c17_cfg5.log
