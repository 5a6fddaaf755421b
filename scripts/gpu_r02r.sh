cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_timeline.py C4 --json $O/r02r_tl_c4.json > $O/r02r_tl_c4.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 '' > $O/r02r_sweep_c4.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' > $O/r02r_sweep_c1.jsonl 2>&1
