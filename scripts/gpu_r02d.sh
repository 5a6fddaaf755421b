cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "vtail or tail" > $O/r02d_tail_test.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $O/r02d_pytest.log 2>&1
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_VTAIL=0' 'SAMG_VTAIL_MB=200' 'SAMG_VTAIL_MB=30' > $O/r02d_sweep_c1.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 '' 'SAMG_VTAIL=0' 'SAMG_VTAIL_MB=200' > $O/r02d_sweep_c4.jsonl 2>&1
SAMG_CG_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/r02d_cg_iter.csv python scripts/profile_solve.py 4 > $O/r02d_cg_iter.log 2>&1
