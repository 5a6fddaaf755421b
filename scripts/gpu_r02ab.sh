cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_L2_PREFETCH_MB=0' 'SAMG_GEMV_EVICT_FIRST=0' 'SAMG_L2_PREFETCH_MB=0 SAMG_GEMV_EVICT_FIRST=0' > $O/r02ab_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 > $O/r02ab_tl.txt 2>&1
