python tools/profile_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 3 > gpurun_out/c3_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 3 -c 1 -o gpurun_out/c3_cfg4_fp32_binned python tools/profile_sweep.py --workload cfg4 --precision fp32 --d 64 --orders 3 > gpurun_out/c3_ncu.log 2>&1
tail -3 gpurun_out/c3_ncu.log
