#!/bin/bash
# r02 call M: the new full-size parity tests (config 4 on one GPU, all config-5 lengths, the
# straddle worst case); DRAM traffic of the config-3 DP launch (twice: reproducibility)
O=gpurun_out/r02m; mkdir -p $O
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -rf --tb=short --durations=0 2>&1 | tail -30 > $O/fullsize.log
for k in 1 2; do
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none -k regex:sdtw_dp -s 3 -c 1 --csv \
   python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/traffic_c3_$k.csv 2> $O/traffic_$k.err
done
