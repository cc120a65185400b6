timeout 600 python tools/profile_screen_iter.py 40 > gpurun_out/c12_iter.log 2>&1; echo "iter rc=$?"; grep -v "Warning\|warn" gpurun_out/c12_iter.log | tail -48
timeout 600 python tools/relabel_sweep.py > gpurun_out/c12_relabel.log 2>&1; echo "relabel rc=$?"; tail -4 gpurun_out/c12_relabel.log
