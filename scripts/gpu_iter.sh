# test + bench + stage timings (one call)
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1; echo "prof exit $?"; cat gpurun_out/prof_plain.log
