python -m pytest tests -m gpu -x -q > gpurun_out/c4_tests.log 2>&1; tail -5 gpurun_out/c4_tests.log
for pf in 1 0; do
CSC_PREFETCH=$pf python tools/time_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 40 >> gpurun_out/c4_t.json 2>&1
CSC_PREFETCH=$pf python tools/time_sweep.py --workload cfg4 --precision fp64 --d 64 --orders 40 >> gpurun_out/c4_t.json 2>&1
CSC_PREFETCH=$pf python tools/time_sweep.py --workload cfg3 --precision fp64 --d 128 --orders 40 >> gpurun_out/c4_t.json 2>&1
CSC_PREFETCH=$pf python tools/time_sweep.py --workload cfg3 --precision fp32 --d 128 --orders 40 >> gpurun_out/c4_t.json 2>&1
done
cat gpurun_out/c4_t.json
