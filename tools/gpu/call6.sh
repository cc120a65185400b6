python -m pytest tests -m gpu -x -q -s -k "not scale" > gpurun_out/c6_tests.log 2>&1; tail -4 gpurun_out/c6_tests.log
python -m pytest tests/test_gpu_scale.py -x -q -s --durations=0 > gpurun_out/c6_scale.log 2>&1; tail -30 gpurun_out/c6_scale.log
for wl in "cfg3 fp64 128" "cfg3 fp32 128" "cfg4 fp32 64" "cfg4 fp64 64" "cfg5 fp64 96" "cfg5 fp64 48"; do set -- $wl
python tools/time_sweep.py --workload $1 --precision $2 --d $3 --orders 30 >> gpurun_out/c6_t.json 2>&1
done
CSC_PREFETCH=0 python tools/time_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 30 >> gpurun_out/c6_t.json 2>&1
cut -c1-250 gpurun_out/c6_t.json
