cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "shim" > $O/r02b_shim.log 2>&1
# bench launch list (contract pass)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/r02b_launches_bench.csv \
  python bench.py --steps 20 --warmup 5 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/r02b_ncu_bench.log 2>&1
# full capture of the headline kernel (2 launches)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_bsr3_tma -s 3 -c 2 -o $O/r02b_spmv_full \
  python bench.py --steps 10 --warmup 3 --amg-repeats 1 --no-cpu-baseline --no-c4 > $O/r02b_ncu_full.log 2>&1
# per-kernel table of one CG iteration (host loop so every launch is visible)
SAMG_CG_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/r02b_cg_iter.csv python scripts/profile_solve.py 4 > $O/r02b_cg_iter.log 2>&1
SAMG_NODE6=1 SAMG_CG_GRAPH=0 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
  --log-file $O/r02b_cg_iter_node6.csv python scripts/profile_solve.py 4 > $O/r02b_cg_iter_node6.log 2>&1
# force-dist at N=1 vs single GPU
timeout 900 python bench.py --force-dist --steps 200 --warmup 10 --no-cpu-baseline --no-c4 > $O/r02b_forcedist.json 2> $O/r02b_forcedist.err
