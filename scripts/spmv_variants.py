"""Time the BSR SpMV variants on C1 (one subprocess per env setting)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CONFIGS = [
    {"SAMG_SPMV_VARIANT": "1"},
    {"SAMG_SPMV_VARIANT": "2"},
    {"SAMG_SPMV_VARIANT": "1", "SAMG_SPMV_GROUP": "4"},
    {"SAMG_SPMV_VARIANT": "2", "SAMG_SPMV_GROUP": "4"},
    {"SAMG_SPMV_VARIANT": "1", "SAMG_SPMV_BLOCKS_PER_LANE": "2"},
    {"SAMG_SPMV_VARIANT": "1", "SAMG_SPMV_BLOCKS_PER_LANE": "6"},
    {"SAMG_SPMV_VARIANT": "1", "SAMG_CG_GRAPH": "0"},
]
extra = sys.argv[1:]
for cfg in CONFIGS:
    env = dict(os.environ, **cfg)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--no-cpu-baseline",
                          "--steps", "2000"] + extra, env=env, capture_output=True, text=True)
    try:
        d = json.loads(out.stdout.strip().splitlines()[-1])
        amg = d.get("amg") or {}
        print(cfg, f"spmv {d['value']:.0f} GB/s frac {d['roofline']['frac']:.3f}",
              f"setup {amg.get('setup_s_all')} solve {amg.get('solve_s_all')} it {amg.get('iterations')}",
              flush=True)
    except Exception:
        print(cfg, "FAILED", out.stdout[-500:], out.stderr[-2000:], flush=True)
