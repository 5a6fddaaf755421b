#!/bin/bash
# SpMV variant sweep on C1: register-streaming (1) vs TMA-fed (3)
cd "$(dirname "$0")/.."
for cfg in "SAMG_SPMV_VARIANT=1" "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=0" "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=1" \
           "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=2" "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=3" \
           "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=4" "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=0 SAMG_TMA_SMEM=160000" \
           "SAMG_SPMV_VARIANT=3 SAMG_TMA_CFG=2 SAMG_TMA_SMEM=160000"; do
  env $cfg timeout 300 python bench.py --steps 2000 --warmup 20 --amg-repeats 2 --no-cpu-baseline > /tmp/b.json 2>/tmp/b.err
  python - "$cfg" <<'PY'
import json,sys
try:
    d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1])
    a=d.get('amg') or {}
    print(sys.argv[1], 'spmv %.0f frac %.3f'%(d['value'],d['roofline']['frac']), 'setup',a.get('setup_s'),'solve',a.get('solve_s_all'),'it',a.get('iterations'))
except Exception as e:
    print(sys.argv[1], 'FAILED', open('/tmp/b.err').read()[-800:])
PY
done
