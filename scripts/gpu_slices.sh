# stage-3 digit-count experiment: S = 5, 6, 7 against the FP64 kernel, plus
# the full-size reference fixtures at S = 5
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for S in 5 6 7; do
  RSM_I8_SLICES=$S timeout 600 python scripts/i8_check.py config1 config2 config3 config4 > gpurun_out/slices_$S.log 2>&1; echo "S=$S exit $?" >> gpurun_out/slices_$S.log
  cat gpurun_out/slices_$S.log
done
RSM_I8_SLICES=5 timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x > gpurun_out/slices5_tests.log 2>&1; echo "tests exit $?" >> gpurun_out/slices5_tests.log
tail -5 gpurun_out/slices5_tests.log
