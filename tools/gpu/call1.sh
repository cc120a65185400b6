set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python tools/time_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 40 > gpurun_out/c1_t32.json 2>&1
python tools/time_sweep.py --workload cfg4 --precision fp64 --d 64 --orders 40 > gpurun_out/c1_t64.json 2>&1
python tools/profile_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 3 > gpurun_out/c1_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/c1_cfg4_fp32 python tools/profile_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 3 > gpurun_out/c1_ncu.log 2>&1
cat gpurun_out/c1_t32.json gpurun_out/c1_t64.json
tail -3 gpurun_out/c1_ncu.log
