# warp-ring SpMV (variant 4) A/B: parity tests, C1/C4 solve sweep, per-kernel timelines
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coarse.py -x -q -m gpu > $O/wr_pytest.log 2>&1; echo "exit $?" >> $O/wr_pytest.log
timeout 600 python scripts/solve_env_sweep.py C1 'SAMG_WRING=0' 'SAMG_WRING=1' 'SAMG_WRING_SHAPE=33' 'SAMG_WRING_SHAPE=32' 'SAMG_WRING=1 SAMG_L2_HINTS=0' 'SAMG_WRING_MIN_ROWS=1' > $O/wr_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_WRING=0 > $O/wr_tl_c1_off.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_WRING=1 > $O/wr_tl_c1_on.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_WRING_SHAPE=33 > $O/wr_tl_c1_33.txt 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 'SAMG_WRING=0' 'SAMG_WRING=1' 'SAMG_WRING_SHAPE=33' > $O/wr_sweep_c4.jsonl 2>&1
tail -3 $O/wr_pytest.log; cat $O/wr_sweep_c1.jsonl $O/wr_sweep_c4.jsonl
