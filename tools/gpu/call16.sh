timeout 120 python tools/tc_screen_check.py --n 2000000 > gpurun_out/c16_tc.log 2>&1; echo "tc big rc=$?"; tail -3 gpurun_out/c16_tc.log
timeout 600 python -m pytest tests/test_gpu_kmeans_fused.py -x -q > gpurun_out/c16_tests.log 2>&1; echo "km tests rc=$?"; tail -3 gpurun_out/c16_tests.log
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c16_iter.log 2>&1; echo "iter rc=$?"; grep -v "Warning\|warn" gpurun_out/c16_iter.log | grep -A12 "mode="
python tools/profile_screen_iter.py 6 tc > gpurun_out/c16_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_screen -s 2 -c 1 -o gpurun_out/c16_tc python tools/profile_screen_iter.py 6 tc > gpurun_out/c16_ncu.log 2>&1
echo "ncu rc=$?"
