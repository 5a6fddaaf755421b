# TMA team shapes for the long-row (level >= 1) operators: per-kernel timeline of one C1 iteration
cd $GRAFT_REPO_ROOT
O=gpurun_out
python scripts/row_stats.py C1 > $O/s4a_rowstats.txt 2>&1
for cfg in "SAMG_TMA_TW32=8" "SAMG_TMA_TW32=8 SAMG_TMA_MIN_CHUNKS=8" "SAMG_TMA_TW32=4" "SAMG_TMA_TW32=4 SAMG_TMA_MIN_CHUNKS=8" \
           "SAMG_TMA_TW32=2" "SAMG_TMA_TW32=2 SAMG_TMA_MIN_CHUNKS=8" "SAMG_TMA_TW32=4 SAMG_TMA_SLACK=1.4" "SAMG_TMA_TW32=2 SAMG_TMA_SLACK=1.5 SAMG_TMA_MIN_CHUNKS=8"; do
  tag=$(echo "$cfg" | tr ' =' '__')
  echo "== $cfg" >> $O/s4a_timelines.txt
  env $cfg SAMG_TMA_DEBUG=1 timeout 300 python scripts/iter_timeline.py C1 2> $O/s4a_err_$tag.txt | sed -n '/^C1:/p;/one iteration/,$p' >> $O/s4a_timelines.txt
  sort $O/s4a_err_$tag.txt | uniq -c | sort -rn | head -12 >> $O/s4a_timelines.txt
  env $cfg timeout 300 python scripts/solve_time.py >> $O/s4a_timelines.txt 2>&1
done
