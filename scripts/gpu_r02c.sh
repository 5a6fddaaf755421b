cd $GRAFT_REPO_ROOT
O=gpurun_out
# sanitizers
for t in memcheck racecheck synccheck; do
  timeout 1200 compute-sanitizer --tool $t --print-limit 20 python scripts/sanitize_probe.py > $O/r02b_san_$t.log 2>&1; echo "rc=$?" >> $O/r02b_san_$t.log
done
