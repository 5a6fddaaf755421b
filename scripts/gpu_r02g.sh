cd $GRAFT_REPO_ROOT
O=gpurun_out
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/grid_barrier scripts/micro/grid_barrier.cu && timeout 120 /tmp/grid_barrier > $O/r02g_grid_barrier.txt 2>&1
SAMG_VTAIL_TRACE=1 SAMG_CG_GRAPH=0 timeout 300 python scripts/profile_solve.py 20 > $O/r02g_trace.log 2>&1
SAMG_VTAIL_TRACE=1 timeout 300 python scripts/profile_solve.py 20 > $O/r02g_trace_graph.log 2>&1
