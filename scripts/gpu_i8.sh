cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 120 python scripts/i8_check.py config1 > gpurun_out/i8_c1.log 2>&1; echo "exit $?" >> gpurun_out/i8_c1.log
cat gpurun_out/i8_c1.log
if grep -q '"config": "config1"' gpurun_out/i8_c1.log; then
  timeout 600 python scripts/i8_check.py config2 config3 config4 > gpurun_out/i8_all.log 2>&1; echo "exit $?" >> gpurun_out/i8_all.log
  cat gpurun_out/i8_all.log
fi
