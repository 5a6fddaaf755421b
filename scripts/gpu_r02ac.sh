cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_EVICT_FIRST_MB=0' 'SAMG_EVICT_FIRST_MB=30' > $O/r02ac_sweep_c1.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 '' 'SAMG_EVICT_FIRST_MB=0' > $O/r02ac_sweep_c4.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 > $O/r02ac_tl.txt 2>&1
