# round 2: staging loops without per-element divisions -- full GPU suite + iteration profile
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c43_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c43_iter.log 2>&1; echo "iter rc=$?"
