cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > $O/r02ai_pytest.log 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/r02ai_setup_c1.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02ai_setup_c4.txt 2>&1
