# round 2: device generators in the bench and scale tests
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/c31_tests.log 2>&1; echo "tests rc=$?"
timeout 900 python bench.py > gpurun_out/c31_bench.json 2> gpurun_out/c31_bench.err; echo "bench rc=$?"
