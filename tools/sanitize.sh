#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck / initcheck over small
# invocations of every hot kernel (tools/sanitize_cases.py); summaries under
# gpurun_out/sanitize_<tool>.log (copy to profiles/ with the round tag).
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report analysis"
  timeout 1500 compute-sanitizer --tool $tool $extra --print-limit 50 --error-exitcode 9 \
    python tools/sanitize_cases.py > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"; tail -3 gpurun_out/sanitize_$tool.log
done
