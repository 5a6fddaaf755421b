cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_TMA_DEBUG=1 timeout 600 python scripts/solve_env_sweep.py C4 'SAMG_TMA_DEBUG=1' > $O/r02q_dbg.txt 2>&1
SAMG_TMA_DEBUG=1 timeout 600 python - > $O/r02q_dbg2.txt 2>&1 <<'PY'
import sys; sys.path.insert(0,'.')
import paper_2202_09056_b200 as pb, torch
dp = pb.generate_hex_device(pb.ProblemParams(nx=199, ny=199, nz=199, dirichlet="eliminate", noise=0.01, seed=2022), device=0)
x = torch.ones(dp.n, dtype=torch.float64, device="cuda"); y = torch.zeros_like(x)
dp.A.spmv_device(x.data_ptr(), y.data_ptr()); torch.cuda.synchronize(); print("spmv ok", float(y.sum()))
print(dp.A.shape)
PY
