# ncu --set full of the pull SpGEMM numeric pass (level-0 R*A and (RA)*P), C1 and C4; raw CSV exported on the box
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:k_spgemm_pull -c 2 -o /tmp/pull_c1 python scripts/setup_phases.py C1 > $O/pull_c1.log 2>&1
ncu -i /tmp/pull_c1.ncu-rep --page raw --csv > $O/pull_c1_raw.csv 2>/dev/null
timeout 1200 ncu --set full --clock-control none -k regex:k_spgemm_pull -c 2 -o /tmp/pull_c4 python scripts/setup_phases.py C4 > $O/pull_c4.log 2>&1
ncu -i /tmp/pull_c4.ncu-rep --page raw --csv > $O/pull_c4_raw.csv 2>/dev/null
ls -la $O/pull_*
