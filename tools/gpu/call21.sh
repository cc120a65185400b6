# round 2: exact fixed-point centroid sums -- parity, then per-iteration kernel times and cfg5 steps
timeout 900 python -m pytest tests/test_gpu_kmeans_fused.py tests/test_gpu_parity.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/c21_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c21_iter.log 2>&1; echo "iter rc=$?"
timeout 600 python tools/cfg5_steps.py --steps 3 > gpurun_out/c21_cfg5.log 2>&1; echo "cfg5 rc=$?"
