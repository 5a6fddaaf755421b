python -m pytest tests -m gpu -q -x 2>&1 | tail -3
python bench.py --no-cpu-baseline --steps 500 > gpurun_out/bench8.json 2> gpurun_out/bench8.err; echo bench rc=$?; tail -3 gpurun_out/bench8.err
for c in 16 32 64 128 182; do SAMG_GJ_CTAS=$c python scripts/configs.py C1 2>&1 | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('gj_ctas', $c, d['gpu_setup_s'], d['gpu_solve_s'])"; done
SAMG_CONFIGS_REF_SOLVE=0 python scripts/configs.py C2 --max-it 1000 --out gpurun_out/configs_d.jsonl 2>&1 | tail -2
python scripts/configs.py C3 --max-it 4000 --out gpurun_out/configs_d.jsonl 2>&1 | tail -1
