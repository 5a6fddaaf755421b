cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_timeline.py C1 ilu0 > $O/r02aa_tl_ilu.txt 2>&1
