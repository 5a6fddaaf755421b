cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_timeline.py C1 > $O/r02k_tl.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_GEMV_TMA=0' > $O/r02k_sweep_c1.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/r02k_pytest.log 2>&1
