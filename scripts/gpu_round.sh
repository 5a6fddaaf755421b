./paper_2202_09056_b200/csrc/build/shim_test; echo shim rc=$?
python -m pytest tests -m gpu -q 2>&1 | tail -5
python bench.py --no-cpu-baseline --steps 500 > gpurun_out/bench4.json 2> gpurun_out/bench4.err; echo bench rc=$?
SMALL="python bench.py --steps 20 --warmup 5 --amg-repeats 1 --no-cpu-baseline"
$SMALL > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches4.csv $SMALL > gpurun_out/ncu_launch.log 2>&1; echo ncu1 rc=$?
