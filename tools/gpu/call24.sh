# round 2: TC screen with a raw ring read directly as A_hi + separate lo ring
timeout 300 python tools/tc_screen_check.py --n 2000000 --d 96 --k 64 > gpurun_out/c24_check.log 2>&1; echo "check rc=$?"
timeout 300 python tools/tc_screen_check.py --n 1000000 --d 128 --k 100 >> gpurun_out/c24_check.log 2>&1; echo "check2 rc=$?"
timeout 900 python -m pytest tests/test_gpu_kmeans_fused.py tests/test_gpu_scale.py -m gpu -q -x > gpurun_out/c24_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c24_iter.log 2>&1; echo "iter rc=$?"
