# compute-sanitizer memcheck, racecheck, synccheck on scripts/sanitize_cases.py
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python scripts/sanitize_cases.py > gpurun_out/san_plain.log 2>&1; echo "plain exit $?" >> gpurun_out/san_plain.log
tail -3 gpurun_out/san_plain.log
for tool in ${TOOLS:-memcheck synccheck racecheck}; do
  timeout ${TLIM:-900} compute-sanitizer --tool $tool --target-processes all --print-limit 50 ${SANFLAGS:-} python scripts/sanitize_cases.py ${CASES:-} > gpurun_out/san_$tool.log 2>&1; echo "$tool exit $?" >> gpurun_out/san_$tool.log
  grep -E "ERROR SUMMARY|exit|Hazard|Invalid|race|RACECHECK SUMMARY" gpurun_out/san_$tool.log | head -20
done
