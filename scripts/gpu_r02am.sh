cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse.py tests/test_gpu_config_parity.py -m gpu -q -x > $O/r02am_pytest.log 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02am_setup_c4.txt 2>&1
