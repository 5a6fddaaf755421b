cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "ilu or pipeline or parity" > $O/r02ae_pytest.log 2>&1
timeout 600 python scripts/iter_timeline.py C1 ilu0 > $O/r02ae_tl_ilu.txt 2>&1
