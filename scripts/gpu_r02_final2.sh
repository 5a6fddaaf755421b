# round-2 closing evidence run: full GPU tests, smoke, bench line + reference arm, bench launch list,
# one full ncu capture of the headline kernel, in-loop per-kernel timelines (SPAI0 C1/C4, ILU C1),
# setup phases (outputs under gpurun_out/r02z_*)
cd $GRAFT_REPO_ROOT
O=gpurun_out
P=r02z
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${P}_smi.txt
(timeout 1500 python -m pytest tests -m gpu -x -q > $O/${P}_pytest.log 2>&1; echo "pytest exit $?" >> $O/${P}_pytest.log)
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${P}_smoke.log 2>&1
timeout 900 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv \
  python bench.py --steps 20 --warmup 5 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_bsr3_tma -s 3 -c 2 -o /tmp/${P}_spmv_full \
  python bench.py --steps 10 --warmup 3 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/${P}_ncu_full.log 2>&1
ncu -i /tmp/${P}_spmv_full.ncu-rep --page raw --csv > $O/${P}_spmv_full_raw.csv 2>/dev/null
timeout 600 python scripts/iter_timeline.py C1 --json $O/${P}_tl_c1.json > $O/${P}_tl_c1.txt 2>&1
timeout 600 python scripts/iter_timeline.py C4 --json $O/${P}_tl_c4.json > $O/${P}_tl_c4.txt 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 > $O/${P}_tl_c1_ilu0.txt 2>&1
SAMG_ILU_ORDER=latest_last timeout 600 python scripts/iter_timeline.py C1 ilu0 > $O/${P}_tl_c1_ilu0_latest_last.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/${P}_setup_c1.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/${P}_setup_c4.txt 2>&1
tail -n 3 $O/${P}_pytest.log; tail -n 1 $O/${P}_smoke.log; cut -c1-400 $O/${P}_bench.json; cut -c1-300 $O/${P}_bench_ref.json; head -3 $O/${P}_tl_c1.txt
