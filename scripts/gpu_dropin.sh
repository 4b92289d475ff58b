cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_dropin_utils.py tests/test_cpp_dropin.py -q -m gpu > gpurun_out/dropin.log 2>&1; echo "pytest exit $?" >> gpurun_out/dropin.log
tail -30 gpurun_out/dropin.log
for t in test_core test_sampler test_spectra test_solver; do (cd /tmp && timeout 300 $GRAFT_REPO_ROOT/oracle/_ref/dropin_$t > $GRAFT_REPO_ROOT/gpurun_out/dropin_$t.log 2>&1; echo "exit $?" >> $GRAFT_REPO_ROOT/gpurun_out/dropin_$t.log); tail -3 gpurun_out/dropin_$t.log; done
