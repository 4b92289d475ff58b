# full GPU suite + stage timings (one call); VARIANTS="ENV=..,ENV=.. ENV=.." adds extra timing runs
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests -q -m gpu -x --timeout 300 ${TESTS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/pytest_gpu.log
tail -15 gpurun_out/pytest_gpu.log
REPS=9 timeout 300 python scripts/prof_c3.py ${CFG:-c3} > gpurun_out/prof_plain.log 2>&1; echo "prof exit $?"; grep median gpurun_out/prof_plain.log
for v in $VARIANTS; do echo "== $v"; env $(echo $v | tr , " ") REPS=9 timeout 300 python scripts/prof_c3.py ${CFG:-c3} 2>&1 | grep median; done
