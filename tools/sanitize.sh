#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py: memcheck, racecheck, synccheck,
# initcheck. Summaries to gpurun_out/sanitize_<tool>.txt.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 --error-exitcode 9 \
      python tools/sanitize_run.py > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.txt
done
