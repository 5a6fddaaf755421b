cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python scripts/iter_bytes.py C1 0.481 > $O/r02p_iter_bytes_c1.json 2>&1
timeout 600 python scripts/iter_bytes.py C4 13.93 > $O/r02p_iter_bytes_c4.json 2>&1
timeout 600 python scripts/iter_timeline.py C4 --json $O/r02p_tl_c4.json > $O/r02p_tl_c4.txt 2>&1
timeout 1200 python bench.py --force-dist --steps 200 --warmup 10 --no-cpu-baseline > $O/r02p_forcedist.json 2> $O/r02p_forcedist.err
