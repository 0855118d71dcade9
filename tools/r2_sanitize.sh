export UM_SANITIZE=1
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --print-limit 50 --log-file gpurun_out/r2_sanitize_$tool.log \
    python tools/sanitize_cases.py > gpurun_out/r2_sanitize_$tool.out 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitize_rc.txt
done
cat gpurun_out/r2_sanitize_rc.txt
tail -3 gpurun_out/r2_sanitize_*.out
