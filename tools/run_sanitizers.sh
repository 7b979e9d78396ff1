# compute-sanitizer over the library's kernel families (one gpurun call); summaries in gpurun_out/
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 7 python tools/sanitize_probe.py 256 \
      > gpurun_out/r02_sanitizer_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r02_sanitizer_summary.txt
done
