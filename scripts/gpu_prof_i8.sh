# launch list + one full ncu capture of k_gram_i8 on config 3
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_i8.csv python scripts/prof_c3.py c3 > gpurun_out/ncu_l.log 2>&1; echo "launches exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram_i8|k_slice" -s 0 -c 2 -f -o gpurun_out/prof_i8 python scripts/prof_c3.py c3 > gpurun_out/ncu_k.log 2>&1; echo "ncu exit $?"; tail -3 gpurun_out/ncu_k.log
