cd $GRAFT_REPO_ROOT
O=gpurun_out
for e in "SAMG_TMA_MIN_CHUNKS=8" "SAMG_SPMV_GROUP=16" "SAMG_SPMV_GROUP=64"; do
  echo "== $e" >> $O/r02t_tl.txt
  timeout 600 python scripts/iter_timeline.py C1 $e 2>&1 | sed -n 3,18p >> $O/r02t_tl.txt
done
