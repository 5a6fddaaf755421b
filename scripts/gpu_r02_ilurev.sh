# ILU(0) sweeps: per-kernel times and solve time, reference and latest_last backward order
cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "ilu" 2>&1 | tail -n 3
SWEEP_SMOOTHER=ilu0 timeout 900 python scripts/solve_env_sweep.py C1 'SAMG_ILU_ORDER=reference' 'SAMG_ILU_ORDER=latest_last' > $O/ir_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 SAMG_ILU_ORDER=latest_last > $O/ir_tl_c1_rev.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 SAMG_ILU_ORDER=reference > $O/ir_tl_c1_ref.txt 2>&1
cat $O/ir_sweep_c1.jsonl | cut -c1-200; head -4 $O/ir_tl_c1_rev.txt; head -4 $O/ir_tl_c1_ref.txt
