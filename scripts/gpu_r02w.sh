cd $GRAFT_REPO_ROOT
O=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "column_range or shim or tail" > $O/r02w_pytest.log 2>&1
timeout 300 python scripts/pcie_probe.py > $O/r02w_pcie.txt 2>&1
timeout 900 python bench.py > $O/r02w_bench.json 2> $O/r02w_bench.err
