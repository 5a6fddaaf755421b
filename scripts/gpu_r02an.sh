cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C4 > $O/r02an_setup_c4.txt 2>&1
SAMG_SETUP_TIMING=1 timeout 600 python scripts/setup_phases.py C1 > $O/r02an_setup_c1.txt 2>&1
timeout 600 python scripts/coarse_sym_probe.py C1 C4 > $O/r02an_sym.txt 2>&1
