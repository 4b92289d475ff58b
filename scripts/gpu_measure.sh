# round measurement: bench line (value/e2e/roofline/cpu_baseline), reference arm,
# ncu launch list of the same bench command, full ncu captures of the stage kernels
cd $GRAFT_REPO_ROOT
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/nvsmi.txt 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 --stages > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench exit $?" >> gpurun_out/bench.err
tail -1 gpurun_out/bench.err; cut -c1-600 gpurun_out/bench.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref exit $?"; cut -c1-300 gpurun_out/bench_ref.json
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches exit $?"
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_gram|k_svd_warp|k_solve_u|k_eig|k_select|k_normal" -s 7 -c 7 -f -o gpurun_out/prof_full python scripts/prof_c3.py c3 > gpurun_out/ncu_full.log 2>&1; echo "ncu full exit $?"
