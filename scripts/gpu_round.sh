python -m pytest tests -m gpu -q -x 2>&1 | tail -4
python bench.py --no-cpu-baseline --steps 1000 > gpurun_out/bench7.json 2> gpurun_out/bench7.err; echo bench rc=$?; tail -3 gpurun_out/bench7.err
python scripts/spmv_variants.py --amg-repeats 2 2>&1 | head -4
SAMG_CG_GRAPH=0 python scripts/profile_solve.py 5 > gpurun_out/ps.log 2>&1 && \
SAMG_CG_GRAPH=0 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_bsr3|k_smooth|k_dense|k_cg|k_p_update|k_dot|k_fill" --csv --log-file gpurun_out/solve_launches3.csv python scripts/profile_solve.py 5 > gpurun_out/ncu_solve.log 2>&1; echo rc=$?
