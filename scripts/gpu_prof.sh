cd $GRAFT_REPO_ROOT
timeout 600 python bench.py --steps 3 --warmup 3 --stages --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -2 gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 300 python scripts/prof_c3.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram|k_svd|k_solve_u|k_eig" -s 4 -c 4 -f -o gpurun_out/prof_c3 python scripts/prof_c3.py > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?"
cat gpurun_out/prof_plain.log; tail -3 gpurun_out/ncu_full.log
