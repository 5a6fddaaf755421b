cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "tail" > $O/r02e_tail_test.log 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_VTAIL=0' 'SAMG_VTAIL_MB=200' 'SAMG_VTAIL_MB=30' > $O/r02e_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 --json $O/r02e_timeline_c1.json > $O/r02e_timeline_c1.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 --json $O/r02e_timeline_c1_notail.json > $O/r02e_timeline_c1_notail.txt 2>&1
