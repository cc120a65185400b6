timeout 600 python -m pytest tests/test_gpu_kmeans_fused.py -x -q > gpurun_out/c9_tests.log 2>&1; echo "km tests rc=$?"; tail -15 gpurun_out/c9_tests.log
CSC_KMEANS_TC=1 timeout 300 python tools/kmeans_cfg5_profile.py --reps 3 > gpurun_out/c9_km_tc.log 2>&1; echo "tc rc=$?"; grep "^kmeans" gpurun_out/c9_km_tc.log
CSC_KMEANS_TC=0 timeout 300 python tools/kmeans_cfg5_profile.py --reps 3 > gpurun_out/c9_km_simt.log 2>&1; echo "simt rc=$?"; grep "^kmeans" gpurun_out/c9_km_simt.log
