cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ilu or pipeline or parity" > $O/r02bd_pytest.log 2>&1
SAMG_PROBE_SMOOTHER=ilu0 SAMG_SETUP_TIMING=1 timeout 300 python scripts/setup_phases.py C1 > $O/r02bd_ilu_setup.txt 2>&1
