#!/bin/bash
# ncu evidence for the speculative-segment schedule at Z=64 (config 3 strong-scaled to 8 GPUs)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
Z=64 N=2000 M=10000000 REPS=2 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
   --log-file gpurun_out/spec_z64_launches.csv python scripts/prof_one.py > /dev/null 2>&1
Z=64 N=2000 M=10000000 REPS=2 timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp_kernel \
   -s 1 -c 1 -o gpurun_out/spec_z64_dp python scripts/prof_one.py > gpurun_out/spec_z64_ncu.log 2>&1
Z=64 N=2000 M=10000000 REPS=2 OPT_SCHED=1 timeout 600 ncu --metrics gpu__time_duration.sum,sm__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv \
   --log-file gpurun_out/seq_z64_launches.csv python scripts/prof_one.py > /dev/null 2>&1
tail -3 gpurun_out/spec_z64_ncu.log; ls -la gpurun_out/spec_z64*
