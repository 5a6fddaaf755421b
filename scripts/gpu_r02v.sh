cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/r02v_setup_c1.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02v_setup_c4.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02v_setup_c1_launches.csv python scripts/setup_phases.py C1 > /dev/null 2>&1
