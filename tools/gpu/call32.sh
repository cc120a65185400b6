# round 2: bench launch list (headline path) + full ncu captures of the cfg4 fp32/fp64 sweep (stall breakdown, L2 hit)
B="python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-dynamic --no-variants --no-cfg4 --no-cfg5"
$B > gpurun_out/c32_plain.json 2> gpurun_out/c32_plain.err && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/c32_launches.csv $B > gpurun_out/c32_ncu_bench.log 2>&1; echo "launches rc=$?"
for p in fp32 fp64; do
  python tools/capture_traffic.py --workload cfg4 --precision $p > gpurun_out/c32_cfg4_$p.plain 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:sweep_kernel -s 2 -c 1 -o gpurun_out/c32_cfg4_$p python tools/capture_traffic.py --workload cfg4 --precision $p > gpurun_out/c32_ncu_$p.log 2>&1; echo "cfg4 $p rc=$?"
done
