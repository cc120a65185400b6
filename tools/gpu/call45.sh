# round 2: bench with the cfg3 end-to-end pipeline
timeout 1200 python bench.py > gpurun_out/c45_bench.json 2> gpurun_out/c45_bench.err; echo "bench rc=$?"
