# compute-sanitizer memcheck / racecheck / synccheck over scripts/sanitize_cases.py
# (run under gpurun; writes gpurun_out/sanitizer_<tool>.txt)
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
      python scripts/sanitize_cases.py > gpurun_out/sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitizer_summary.txt
done
