timeout 900 python tools/profile_screen_iter.py 100 simt,tc,changes > gpurun_out/c18_iter.log 2>&1; echo "iter rc=$?"; grep -v "Warning\|warn" gpurun_out/c18_iter.log | grep -A30 "mode=simt"
