cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1200 python scripts/solve_env_sweep.py C1 'SAMG_VTAIL=0' 'SAMG_VTAIL=0 SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_GMAX=16' 'SAMG_VTAIL=0 SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_GMAX=8' 'SAMG_VTAIL=0 SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_GMAX=32' > $O/r02j_sweep_c1.jsonl 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_GMAX=16 > $O/r02j_tl_g16.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 SAMG_VTAIL=0 SAMG_TMA_MIN_CHUNKS=8 SAMG_TMA_GMAX=8 > $O/r02j_tl_g8.txt 2>&1
