cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 SAMG_L2_PERSIST_MB=70 --json $O/r02h_tl_persist70.json > $O/r02h_tl_persist70.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 SAMG_L2_PERSIST_MB=200 --json $O/r02h_tl_persist200.json > $O/r02h_tl_persist200.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 'SAMG_VTAIL=0' 'SAMG_VTAIL=0 SAMG_L2_PERSIST_MB=70' 'SAMG_VTAIL=0 SAMG_L2_PERSIST_MB=200' 'SAMG_L2_PERSIST_MB=200' > $O/r02h_sweep_c1.jsonl 2>&1
