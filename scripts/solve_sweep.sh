#!/bin/bash
# SpMV dispatch settings vs C1 solve time and per-operator SpMV rates.
out=${1:-gpurun_out/solve_sweep.txt}
: > "$out"
for cfg in "" "SAMG_TMA_MIN_CHUNKS=8" "SAMG_TMA_MIN_CHUNKS=4" "SAMG_TMA_MIN_CHUNKS=1" \
           "SAMG_SPMV_BLOCKS_PER_LANE=4" "SAMG_SPMV_BLOCKS_PER_LANE=12"; do
  echo "== $cfg" >> "$out"
  env $cfg timeout 120 python scripts/solve_time.py >> "$out" 2>&1
  env $cfg timeout 120 python scripts/level_spmv.py >> "$out" 2>&1
done
