#!/bin/bash
# r02 call BA: 2-warp rings for short fixed-length queries -- tests, config-5 lines, N = 1,500 probe, ragged lanes
O=gpurun_out/r02ba; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_start_ckpt.py tests/test_gpu_spec.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_path.py tests/test_gpu_tail_skip.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for c in c5_500 c5_1000; do timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
timeout 900 python bench.py --config c5_1000 --steps 5 --no-cpu-baseline --path > $O/bench_c5_1000_path.json 2>> $O/bench.err
Z=512 N=1500 M=1000000 CONFIGS='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 4}]' timeout 900 python scripts/sweep.py > $O/n1500.jsonl 2>&1
TRACE=1 Z=512 N=1500 M=1000000 CONFIGS='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 4}]' timeout 900 python scripts/sweep.py >> $O/n1500.jsonl 2>&1
CASES=";OPT_LANES=2;OPT_LANES=4;OPT_LANES=8" timeout 900 python scripts/ragged_sweep.py > $O/ragged_lanes.jsonl 2>&1
LMIN=500 LMAX=2000 CASES=";OPT_LANES=2;OPT_LANES=4" timeout 900 python scripts/ragged_sweep.py >> $O/ragged_lanes.jsonl 2>&1
cat $O/tests.log $O/n1500.jsonl $O/ragged_lanes.jsonl
