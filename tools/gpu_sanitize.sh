#!/bin/bash
# compute-sanitizer over tools/sanitize_run.py (every kernel variant at small shapes).
# Each tool under its own timeout; summaries land in gpurun_out/sanitize_<tool>.log.
mkdir -p gpurun_out
for tool in ${SAN_TOOLS:-memcheck synccheck racecheck initcheck}; do
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool --print-limit 50 \
    python tools/sanitize_run.py > gpurun_out/sanitize_${tool}.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_${tool}.log
  echo "$tool: $(tail -3 gpurun_out/sanitize_${tool}.log | tr '\n' ' ')"
done
