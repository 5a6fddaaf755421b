cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_config_parity.py tests/test_gpu_parity.py -m gpu -q -x > $O/r02ar_pytest.log 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/r02ar_setup_c1.txt 2>&1
SAMG_GJ_LOOKAHEAD=0 SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/r02ar_setup_c1_nola.txt 2>&1
