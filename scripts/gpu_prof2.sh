cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_eig|k_solve_u|k_svd_warp" -s 3 -c 3 -f -o gpurun_out/prof_c3 python scripts/prof_c3.py c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?"
cat gpurun_out/prof_plain.log; tail -2 gpurun_out/ncu_full.log
