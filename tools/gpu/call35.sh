# round 2: full bench with the cfg5 matrix
timeout 1200 python bench.py > gpurun_out/c35_bench.json 2> gpurun_out/c35_bench.err; echo "bench rc=$?"
