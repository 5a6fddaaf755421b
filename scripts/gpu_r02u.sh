cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 2400 bash scripts/pipelines.sh $O/r02u_pipelines.jsonl C0 C1 > $O/r02u_pipelines.log 2>&1
