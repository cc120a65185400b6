# round 2: TC screen pipeline ordering fix -- parity at many tiles, cfg3 k-means, per-iteration screen times, cfg5 steps
timeout 900 python -m pytest tests/test_gpu_kmeans_fused.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/c19_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/profile_screen_iter.py 100 simt,tc > gpurun_out/c19_iter.log 2>&1; echo "iter rc=$?"
timeout 600 python tools/cfg5_steps.py --steps 3 > gpurun_out/c19_cfg5.log 2>&1; echo "cfg5 rc=$?"
