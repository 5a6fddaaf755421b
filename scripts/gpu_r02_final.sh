# round-2 evidence run: bench line, reference arm, bench launch list, one
# full ncu capture of the headline kernel, in-loop per-kernel timelines,
# setup phases (all outputs under gpurun_out/r02f_*)
cd $GRAFT_REPO_ROOT
O=gpurun_out
P=${1:-r02fin}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/${P}_smi.txt
timeout 900 python bench.py > $O/${P}_bench.json 2> $O/${P}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/${P}_bench_ref.json 2> $O/${P}_bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/${P}_launches.csv \
  python bench.py --steps 20 --warmup 5 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/${P}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsr3_tma -s 3 -c 2 -o $O/${P}_spmv_full \
  python bench.py --steps 10 --warmup 3 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/${P}_ncu_full.log 2>&1
timeout 600 python scripts/iter_timeline.py C1 --json $O/${P}_tl_c1.json > $O/${P}_tl_c1.txt 2>&1
timeout 600 python scripts/iter_timeline.py C4 --json $O/${P}_tl_c4.json > $O/${P}_tl_c4.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/${P}_setup_c1.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/${P}_setup_c4.txt 2>&1
