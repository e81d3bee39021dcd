mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_workload.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|SANITIZE_WORKLOAD_OK|RACECHECK SUMMARY' gpurun_out/sanitize_$tool.log | tr '\n' ' ')"
done
