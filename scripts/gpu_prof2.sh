cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram" -s 2 -c 1 -f -o gpurun_out/prof_c3 python scripts/prof_c3.py c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?"
cat gpurun_out/prof_plain.log; tail -2 gpurun_out/ncu_full.log
