#!/bin/bash
# Runs compute-sanitizer memcheck / racecheck / synccheck over every kernel family (small inputs) and
# keeps the logs in gpurun_out/sanitize/.  Usage (GPU box): bash tools/sanitize.sh [family ...]
set -u
out=gpurun_out/sanitize; mkdir -p "$out"
fams=${*:-"small stream chunked large tc batched stats symbols variants"}
for tool in memcheck racecheck synccheck; do
  for f in $fams; do
    timeout 300 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 20 \
      python tools/sanitize_driver.py $f > "$out/${tool}_${f}.log" 2>&1
    echo "$tool $f rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' "$out/${tool}_${f}.log" | tail -1)"
  done
done
