cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 ncu --set full --clock-control none -k regex:'k_trailing|k_panel_reg|k_moves_apply' -s 30 -c 6 -o $O/r02ao_gj python scripts/setup_phases.py C1 > $O/r02ao_ncu.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02ao_c1_setup_launches.csv python scripts/setup_phases.py C1 > /dev/null 2>&1
