#!/bin/bash
# r02 call L: uint8 pruning in the unclamped 5+1-SASS form (parity, bench), column-call error
# paths, ncu --set full of the uint8 DP launch at config 2
O=gpurun_out/r02l; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_q8.py tests/test_gpu_refsplit.py tests/test_gpu_spec.py -q -rf --tb=short 2>&1 | tail -25 > $O/tests.log
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 --q8-prune 96 > $O/bench_c3_q8p96.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e --q8 > $O/bench_c3_q8.json 2>> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp2 -s 3 -c 1 \
   -o $O/c2_q8 python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --q8 > $O/ncu_q8.log 2>&1
