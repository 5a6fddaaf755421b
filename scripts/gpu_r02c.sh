cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python scripts/solve_env_sweep.py C1 '' 'SAMG_TMA_MIN_CHUNKS=8' 'SAMG_TMA_MIN_CHUNKS=4' 'SAMG_TMA_MIN_CHUNKS=2' 'SAMG_SPMV_BLOCKS_PER_LANE=4' 'SAMG_SPMV_BLOCKS_PER_LANE=12' 'SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_BLOCKED=1' > $O/r02c_sweep_c1.jsonl 2>&1
timeout 900 python scripts/solve_env_sweep.py C4 '' 'SAMG_TMA_MIN_CHUNKS=8' 'SAMG_TMA_MIN_CHUNKS=4' > $O/r02c_sweep_c4.jsonl 2>&1
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_probe.py > $O/r02c_san_$t.log 2>&1; echo "rc=$?" >> $O/r02c_san_$t.log
done
