cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse.py -m gpu -q -x > $O/r02ad_pytest.log 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02ad_setup_c4.txt 2>&1
for f in 1.5 1.0; do SAMG_POOL_RESERVE=$f SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02ad_setup_c4_$f.txt 2>&1; done
