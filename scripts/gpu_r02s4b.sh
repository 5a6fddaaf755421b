# full ncu sections for the level >= 1 V-cycle kernels of one C1 iteration
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python scripts/ncu_solve_small.py 6 > $O/s4b_plain.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_bsr3|k_dense_gemv|k_cg_update|k_p_update' -s 48 -c 34 -o $O/s4b_iter_full \
  python scripts/ncu_solve_small.py 6 > $O/s4b_ncu.log 2>&1
tail -3 $O/s4b_ncu.log
