python -m pytest tests -m gpu -x -q > gpurun_out/c2_tests.log 2>&1; tail -15 gpurun_out/c2_tests.log
for b in 1 0; do
CSC_ROW_BINNING=$b python tools/time_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 40 >> gpurun_out/c2_t.json 2>&1
CSC_ROW_BINNING=$b python tools/time_sweep.py --workload cfg4 --precision fp64 --d 64 --orders 40 >> gpurun_out/c2_t.json 2>&1
done
python tools/time_sweep.py --workload cfg3 --precision fp64 --d 128 --orders 40 >> gpurun_out/c2_t.json 2>&1
cat gpurun_out/c2_t.json
