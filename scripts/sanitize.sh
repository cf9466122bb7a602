#!/bin/bash
# compute-sanitizer on small configurations: memcheck, racecheck and
# synccheck over the DP kernel's ring / mbarrier-free release-acquire protocol, the
# persistent scheduler, the cluster (DSMEM) variant, traceback, path and ragged batches.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py \
     > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
done
cat gpurun_out/sanitize_summary.txt
