set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
SAMG_CG_GRAPH=0 python -m pytest tests/test_gpu_parity.py -x -q -k "cube6 or zero or breakdown" 2>&1 | tail -3
python scripts/spmv_variants.py --amg-repeats 3
