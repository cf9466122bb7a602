#!/bin/bash
# compute-sanitizer on small configurations: memcheck, racecheck and
# synccheck over the DP kernel's ring / mbarrier-free release-acquire protocol, the
# persistent scheduler, the cluster (DSMEM) variant, traceback, path and ragged batches.
cd "$(dirname "$0")/.."
O=${1:-gpurun_out}
mkdir -p $O
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool --error-exitcode 9 --print-limit 20 python scripts/sanitize_cases.py \
     > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_summary.txt
done
cat $O/sanitize_summary.txt
