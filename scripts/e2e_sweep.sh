# e2e SpMV pipeline: CTA cap of the SpMV inside samg_bsr3_spmv_batch (3 runs each)
for c in 0 108 96 84 74; do printf "SAMG_BATCH_CTAS=$c:"; for r in 1 2 3; do SAMG_BATCH_CTAS=$c timeout 300 python bench.py --steps 300 --warmup 10 --amg-repeats 1 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(' %d' % d['e2e']['value'], end='')"; done; echo; done
