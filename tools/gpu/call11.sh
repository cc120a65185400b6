timeout 600 python -m pytest tests/test_gpu_kmeans_fused.py tests/test_gpu_parity.py -x -q > gpurun_out/c11_tests.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/c11_tests.log
CSC_KMEANS_TC=1 timeout 300 python tools/kmeans_cfg5_profile.py --reps 3 > gpurun_out/c11_km_tc.log 2>&1; echo "tc rc=$?"; grep "^kmeans" gpurun_out/c11_km_tc.log
CSC_KMEANS_TC=1 python tools/kmeans_cfg5_profile.py --restarts 1 --reps 1 > gpurun_out/c11_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"screen|update|assign|bound_kernel|cost_kernel|sums_finish" -c 700 --csv --log-file gpurun_out/c11_ncu_tc.csv python tools/kmeans_cfg5_profile.py --restarts 1 --reps 1 > gpurun_out/c11_ncu_tc.log 2>&1
CSC_KMEANS_TC=0 python tools/kmeans_cfg5_profile.py --restarts 1 --reps 1 > gpurun_out/c11_plain0.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"screen|update|assign|bound_kernel|cost_kernel|sums_finish" -c 700 --csv --log-file gpurun_out/c11_ncu_simt.csv python tools/kmeans_cfg5_profile.py --restarts 1 --reps 1 > gpurun_out/c11_ncu_simt.log 2>&1
echo done
