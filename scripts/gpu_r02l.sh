cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_timeline.py C1 > $O/r02l_tl.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_EPI_PREFETCH=0' 'SAMG_SPMV_LONGROW_BPL=0' 'SAMG_SPMV_LONGROW_BPL=4' 'SAMG_EPI_PREFETCH=0 SAMG_SPMV_LONGROW_BPL=0' > $O/r02l_sweep_c1.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 '' 'SAMG_EPI_PREFETCH=0 SAMG_SPMV_LONGROW_BPL=0' > $O/r02l_sweep_c4.jsonl 2>&1
