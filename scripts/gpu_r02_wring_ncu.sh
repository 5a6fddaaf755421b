# ncu --set full of the level-1 kernels: register kernel (k_bsr3<32,...>) vs warp-ring (k_bsr3_wring);
# raw pages exported as CSV on the box (the reports exceed the 64 MiB return limit)
cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_WRING=0 timeout 900 ncu --set full --clock-control none -k regex:'^k_bsr3$' -s 26 -c 13 -o /tmp/wrn_reg python scripts/ncu_solve_small.py 6 spai0 > $O/wrn_reg.log 2>&1
ncu -i /tmp/wrn_reg.ncu-rep --page raw --csv > $O/wrn_reg_raw.csv 2>/dev/null
SAMG_WRING=1 timeout 900 ncu --set full --clock-control none -k regex:'k_bsr3_wring' -s 6 -c 3 -o /tmp/wrn_ring python scripts/ncu_solve_small.py 6 spai0 > $O/wrn_ring.log 2>&1
ncu -i /tmp/wrn_ring.ncu-rep --page raw --csv > $O/wrn_ring_raw.csv 2>/dev/null
ls -la $O/wrn_*; tail -n 3 $O/wrn_reg.log; tail -n 3 $O/wrn_ring.log
