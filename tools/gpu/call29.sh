# round 2: full GPU suite + cfg5 step phases after the k-means changes
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c29_tests.log 2>&1; echo "tests rc=$?"
timeout 600 python tools/cfg5_steps.py --steps 3 > gpurun_out/c29_cfg5.log 2>&1; echo "cfg5 rc=$?"
