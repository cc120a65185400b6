for lib in w3 w0; do for pf in 1 0; do
for wl in "cfg3 fp64 128" "cfg3 fp32 128" "cfg4 fp32 64" "cfg4 fp64 64"; do set -- $wl
echo -n "$lib pf=$pf " >> gpurun_out/c5_t.json
CSC_LIB=abv/$lib.so CSC_PREFETCH=$pf python tools/time_sweep.py --workload $1 --precision $2 --d $3 --orders 30 >> gpurun_out/c5_t.json 2>&1
done; done; done
cat gpurun_out/c5_t.json | cut -c1-200
