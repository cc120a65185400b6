python tools/profile_screen_iter.py 6 tc > gpurun_out/c14_plain.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:tc_screen -s 2 -c 1 -o gpurun_out/c14_tc python tools/profile_screen_iter.py 6 tc > gpurun_out/c14_ncu.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/c14_ncu.log
