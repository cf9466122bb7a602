#!/bin/bash
# r02 call BK: ncu --set full of the config-5 N = 1,000 DP launch (2-warp rings, checkpointed start) + launch list
O=gpurun_out/r02bk; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o $O/c5_1000_dp python bench.py --config c5_1000 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c5.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c5_1000.csv \
   python bench.py --config c5_1000 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_c5_bench.json 2>&1
tail -3 $O/ncu_c5.log
