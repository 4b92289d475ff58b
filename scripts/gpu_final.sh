# round-final run: smoke, full GPU suite, then the round measurement and the all-config table
cd $GRAFT_REPO_ROOT
timeout 300 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/smoke.log
timeout 1500 python -m pytest tests -q -m gpu -x --timeout 600 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/smoke.log; tail -4 gpurun_out/pytest_gpu.log
bash scripts/gpu_measure.sh
timeout 600 python scripts/all_configs.py > gpurun_out/configs.jsonl 2> gpurun_out/configs.err; echo "configs exit $?"
