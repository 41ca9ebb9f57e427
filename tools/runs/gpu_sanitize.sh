mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool python tools/sanitize_cases.py > gpurun_out/r1_sanitizer6_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/r1_sanitizer6_$tool.log
done
