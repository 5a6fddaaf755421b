cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $O/r02s_pytest.log 2>&1
timeout 600 python scripts/iter_timeline.py C4 > $O/r02s_tl_c4.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 > $O/r02s_tl_c1.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' > $O/r02s_sweep_c1.jsonl 2>&1
