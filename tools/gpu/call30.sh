# round 2: device generators
timeout 900 python -m pytest tests/test_gpu_generators.py -m gpu -q -x > gpurun_out/c30_tests.log 2>&1; echo "tests rc=$?"
