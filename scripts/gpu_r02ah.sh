cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02ah_setup_c4_launches.csv python scripts/setup_phases.py C4 > $O/r02ah_ncu.log 2>&1
