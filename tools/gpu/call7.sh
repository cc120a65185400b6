python bench.py > gpurun_out/c7_bench.json 2> gpurun_out/c7_bench.err; echo "bench rc=$?"; tail -5 gpurun_out/c7_bench.err
for wl in "cfg3 fp64" "cfg3 fp32" "cfg4 fp32" "cfg4 fp64"; do set -- $wl
python tools/capture_traffic.py --workload $1 --precision $2 > gpurun_out/traffic_$1_$2.json 2> gpurun_out/traffic_$1_$2.err && \
ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sweep_kernel --csv --log-file gpurun_out/traffic_$1_$2.csv python tools/capture_traffic.py --workload $1 --precision $2 > gpurun_out/traffic_$1_$2.json 2>> gpurun_out/traffic_$1_$2.err
echo "$1 $2 rc=$?"
done
python tools/kmeans_cfg5_profile.py > gpurun_out/c7_km.log 2>&1; tail -40 gpurun_out/c7_km.log
