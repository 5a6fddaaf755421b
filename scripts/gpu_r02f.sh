cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_vtail -s 20 -c 1 -o $O/r02f_vtail python scripts/profile_solve.py 12 > $O/r02f_ncu_vtail.log 2>&1
timeout 600 python scripts/iter_timeline.py C1 --json $O/r02f_timeline_c1.json > $O/r02f_timeline_c1.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 --json $O/r02f_timeline_c1_notail.json > $O/r02f_timeline_c1_notail.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_L2_HINTS=0 SAMG_VTAIL=0 --json $O/r02f_timeline_c1_nohint.json > $O/r02f_timeline_c1_nohint.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_VTAIL=0' 'SAMG_VTAIL=0 SAMG_L2_HINTS=0' > $O/r02f_sweep_c1.jsonl 2>&1
