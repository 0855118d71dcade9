for t in memcheck synccheck racecheck; do
  timeout 900 compute-sanitizer --tool $t python tools/sanitize_cases.py > gpurun_out/s3v_sanitize_$t.log 2>&1
done
timeout 1800 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/s3v_gputest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3v_smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/s3v_bench.log 2>&1
