cd $GRAFT_REPO_ROOT
O=gpurun_out
for e in "" "SAMG_VTAIL_SLEEP=100" "SAMG_VTAIL_G=64" "SAMG_VTAIL_G=128"; do
  echo "== $e" >> $O/r02i_trace.log
  env $e SAMG_VTAIL_TRACE=1 SAMG_CG_GRAPH=0 timeout 300 python scripts/profile_solve.py 20 2>&1 | grep -v '^{\|^P ' >> $O/r02i_trace.log
done
