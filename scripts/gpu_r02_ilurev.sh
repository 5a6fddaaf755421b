# ILU(0) backward sweep with the subtraction chain over descending columns (relaxed order)
cd $GRAFT_REPO_ROOT
O=gpurun_out
SWEEP_SMOOTHER=ilu0 timeout 900 python scripts/solve_env_sweep.py C1 'SAMG_ILU_BWD_REV=0' 'SAMG_ILU_BWD_REV=1' > $O/ir_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 SAMG_ILU_BWD_REV=1 > $O/ir_tl_c1_rev.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 SAMG_ILU_BWD_REV=0 > $O/ir_tl_c1_ref.txt 2>&1
cat $O/ir_sweep_c1.jsonl | cut -c1-260; grep -h "ilu_sweep" $O/ir_tl_c1_rev.txt $O/ir_tl_c1_ref.txt | head -20
