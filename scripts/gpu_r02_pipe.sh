# long-row register kernel variants: col one iteration ahead (pipe) under different register budgets
# (the sweep that picked variant 2; the experiment values 1 / 3 / 5 / 6 of SAMG_LONG_PIPE selected builds that
# no longer exist -- the shipped switch is 0: variant 1, 1: G = 32 only, 2: also G = 64; results in profiles/r02_long_pipe.txt)
cd $GRAFT_REPO_ROOT
O=gpurun_out
for v in 0 1 3 5 6; do
  timeout 600 python scripts/iter_timeline.py C1 SAMG_LONG_PIPE=$v > $O/pp_tl_c1_$v.txt 2>&1
done
timeout 600 python scripts/solve_env_sweep.py C1 'SAMG_LONG_PIPE=0' 'SAMG_LONG_PIPE=1' 'SAMG_LONG_PIPE=3' 'SAMG_LONG_PIPE=5' 'SAMG_LONG_PIPE=6' > $O/pp_sweep_c1.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 'SAMG_LONG_PIPE=0' 'SAMG_LONG_PIPE=3' 'SAMG_LONG_PIPE=5' 'SAMG_LONG_PIPE=6' > $O/pp_sweep_c4.jsonl 2>&1
cat $O/pp_sweep_c1.jsonl $O/pp_sweep_c4.jsonl | cut -c1-180; grep -h "us/it.*k_bsr3<32" $O/pp_tl_c1_?.txt | head -40
