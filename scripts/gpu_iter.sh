# test + stage timings (one call); VARIANTS="ENV=.. ENV=.." adds extra timing runs
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_cpp_dropin.py -q -m gpu -x --timeout 300 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
REPS=3 timeout 300 python scripts/prof_c3.py c3 > gpurun_out/prof_plain.log 2>&1; echo "prof exit $?"; cut -c1-250 gpurun_out/prof_plain.log
for v in $VARIANTS; do echo "== $v"; env $(echo $v | tr , " ") REPS=3 timeout 300 python scripts/prof_c3.py c3 2>&1 | cut -c1-250; done
