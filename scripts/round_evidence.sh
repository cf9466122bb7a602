#!/bin/bash
# Bench line + ncu evidence for the default configuration.  Usage: scripts/round_evidence.sh <tag>
cd "$(dirname "$0")/.."
TAG=${1:-r01}
mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv > gpurun_out/${TAG}_smi.csv 2>&1
timeout 900 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
# launch list of the default bench command (serialised, cold: shares only)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/${TAG}_launches_bench.json 2>&1
# one full-section capture of the DP kernel (c2 workload keeps the replays short)
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o gpurun_out/${TAG}_dp python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e \
   > gpurun_out/${TAG}_ncu_full.log 2>&1
echo done
# DRAM traffic of one DP launch of the bench workload (roofline.traffic)
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
   -k regex:sdtw_dp -s 3 -c 1 --csv --log-file gpurun_out/${TAG}_traffic.csv \
   python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/ncu_traffic.py gpurun_out/${TAG}_traffic.csv c3 512 2000 10000000 && cp profiles/traffic_c3.json gpurun_out/ 
