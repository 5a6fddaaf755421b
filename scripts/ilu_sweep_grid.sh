timeout 300 python -m pytest tests -m gpu -q -x -k "ilu" 2>&1 | tail -2
for c in 1 2; do for k in 2 4 8 16 64 100000; do printf "ctas/sm %s ahead %s: " $c $k; SAMG_ILU_CTAS_PER_SM=$c SAMG_ILU_AHEAD=$k timeout 300 python scripts/configs.py C1 --smoother ilu0 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['gpu_solve_s'], d['gpu_iterations'])"; done; done
