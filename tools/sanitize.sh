#!/bin/bash
# compute-sanitizer memcheck / racecheck / synccheck over every libvba kernel family
# (tools/sanitize_run.py); summaries into gpurun_out/sanitize_<tool>.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck racecheck; do
  for part in solve tc dense preint; do
    timeout 1200 $CS --tool $tool --print-limit 20 --error-exitcode 9 python tools/sanitize_run.py $part \
      > gpurun_out/sanitize_${tool}_${part}.log 2>&1
    echo "$tool $part rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|sanitize_run ok' gpurun_out/sanitize_${tool}_${part}.log | tr '\n' ' ')"
  done
done | tee gpurun_out/sanitize_summary.txt
