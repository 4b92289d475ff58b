# full ncu capture of one kernel (regex in $K) from the config-3 stage run
cd $GRAFT_REPO_ROOT
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"$K" -s ${S:-0} -c 1 -f -o gpurun_out/prof_k python scripts/prof_c3.py c3 > gpurun_out/ncu_k.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/ncu_k.log
