# round 2: label changes, Hamerly candidates and screen-undecided rows per cfg5 Lloyd iteration
timeout 900 python tools/profile_screen_iter.py 100 changes > gpurun_out/c20_changes.log 2>&1; echo "rc=$?"
