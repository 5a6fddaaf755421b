cd $GRAFT_REPO_ROOT
O=gpurun_out
SAMG_CG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:'k_bsr3<' -s 40 -c 12 -o $O/r02m_coarse python scripts/profile_solve.py 8 > $O/r02m_ncu.log 2>&1
SAMG_CG_GRAPH=0 timeout 900 ncu --set full --import-source on --clock-control none --cache-control none -k regex:'k_cg_update_smooth|k_p_update_u|k_dense_gemv' -s 6 -c 3 -o $O/r02m_vec python scripts/profile_solve.py 8 > $O/r02m_ncu2.log 2>&1
