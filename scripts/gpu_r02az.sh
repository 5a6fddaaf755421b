cd $GRAFT_REPO_ROOT
O=gpurun_out
for k in 1 2 3; do SAMG_SETUP_TIMING=1 timeout 300 python scripts/first_call.py 2>&1 | grep -h 'L0 upload\|call 0' | head -2 >> $O/r02az_first.txt; done
