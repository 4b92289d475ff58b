# stage timings per variant env (VARIANTS="A=1,B=2 A=3"), with the harvest/decompose parity tests per variant
cd $GRAFT_REPO_ROOT
for v in base $VARIANTS; do
  ev=""; [ "$v" != base ] && ev=$(echo $v | tr , " ")
  echo "== $v"
  env $ev timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_coverage.py -q -m gpu -x --timeout 300 -k "${TESTK:-harvest or decompose}" 2>&1 | tail -2
  env $ev REPS=3 timeout 300 python scripts/prof_c3.py ${CFG:-c3} 2>&1 | tail -2 | cut -c1-200
done
