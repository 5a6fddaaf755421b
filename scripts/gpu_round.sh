set -x
python -m pytest tests -m gpu -x -q 2>&1 | tail -5
python -c "import __graft_entry__ as g; g.smoke()"
python bench.py > gpurun_out/bench2.json 2> gpurun_out/bench2.err; echo bench rc=$?
SMALL="python bench.py --steps 20 --warmup 5 --amg-repeats 1 --no-cpu-baseline"
$SMALL > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches2.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
SM2="python bench.py --steps 10 --warmup 3 --amg-repeats 0 --no-cpu-baseline"
$SM2 > gpurun_out/plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_bsr3 -s 5 -c 2 -o gpurun_out/prof_spmv2 $SM2 > gpurun_out/ncu_full.log 2>&1; echo ncu2 rc=$?
