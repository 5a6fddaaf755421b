# mixed-precision V-cycle probe: C1 SPAI0 solve and the fp64 SpMV bench under
# TMA ring budgets / chunk assignment
run() { timeout 300 python scripts/configs.py C1 --smoother spai0 --precision $1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1', d['gpu_solve_s'], d['gpu_iterations'])"; }
for b in 0 1; do for sm in 226000 160000 110000; do
  echo "blocked=$b smem32=$sm"; SAMG_TMA_BLOCKED=$b SAMG_TMA_SMEM32=$sm SAMG_TMA_G=4 run mixed
done; done
for b in 0 1; do for sm in 226000 160000; do
  printf "fp64 bench blocked=$b smem=$sm: "; SAMG_TMA_BLOCKED=$b SAMG_TMA_SMEM=$sm timeout 300 python bench.py --steps 500 --warmup 10 --amg-repeats 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['amg']['solve_s'])"
done; done
