# one ncu --set full capture of the kernels matching $K (default k_solve_u) on config $CFG
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
REPS=2 timeout 300 python scripts/prof_c3.py ${CFG:-c3} > gpurun_out/prof_plain.log 2>&1 && \
REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"${K:-k_solve_u}" -s ${SKIP:-1} -c ${CNT:-1} -f -o gpurun_out/${OUT:-prof_k} python scripts/prof_c3.py ${CFG:-c3} > gpurun_out/ncu_k.log 2>&1; echo "ncu exit $?"
tail -3 gpurun_out/ncu_k.log
