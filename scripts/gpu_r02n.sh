cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_CG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none -k regex:'^k_bsr3$' -s 45 -c 9 -o $O/r02n_coarse python scripts/profile_solve.py 8 > $O/r02n_ncu.log 2>&1
