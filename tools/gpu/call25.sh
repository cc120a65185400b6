# round 2: TC screen timing A/B (distance hook + host-driven Lloyd iterations)
timeout 300 python tools/tc_screen_check.py --n 2000000 --d 96 --k 64 > gpurun_out/c25_check.log 2>&1; echo "check rc=$?"
timeout 600 python tools/profile_screen_iter.py 100 tc > gpurun_out/c25_iter.log 2>&1; echo "iter rc=$?"
