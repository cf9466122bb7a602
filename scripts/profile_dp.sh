#!/bin/bash
# ncu evidence for the DP kernel.  Usage: scripts/profile_dp.sh <tag> [bench args]
cd "$(dirname "$0")/.."
TAG=${1:-r01}; shift
mkdir -p gpurun_out
# launch list of a bench run (cold, serialised: shares only)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/${TAG}_launches.csv python bench.py --config c2 --steps 2 --warmup 3 \
   --no-cpu-baseline --no-e2e "$@" > gpurun_out/${TAG}_launches_bench.json 2>&1
# full section set on one DP launch (c2 workload)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o gpurun_out/${TAG}_dp python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e "$@" \
   > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
