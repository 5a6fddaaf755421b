# verification of the head commit: full GPU tests, smoke, bench line + reference arm (outputs under gpurun_out/r02v_*)
cd $GRAFT_REPO_ROOT
O=gpurun_out
P=r02v
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${P}_smi.txt
(timeout 1500 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${P}_pytest.log)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1; echo "smoke exit $?" >> $O/${P}_smoke.log
timeout 900 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
tail -n 3 $O/${P}_pytest.log; tail -n 2 $O/${P}_smoke.log; cut -c1-600 $O/${P}_bench.json; cut -c1-300 $O/${P}_bench_ref.json
