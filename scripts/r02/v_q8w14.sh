#!/bin/bash
# r02 call V: W = 14 default for uint8 (parity + benches), half at W = 14 vs 30
O=gpurun_out/r02v; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_q8.py tests/test_gpu_half.py -q -rf --tb=short 2>&1 | tail -15 > $O/tests.log
Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_PRECISION": 16}, {"OPT_PRECISION": 16, "OPT_SEGMENT_W": 14}, {"OPT_PRECISION": 16, "OPT_SEGMENT_W": 14, "OPT_LANES": 8}]' timeout 900 python scripts/sweep.py > $O/sweep_half_w.jsonl 2>&1
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 > $O/bench_c3_q8.json 2>> $O/bench.err
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 --q8-prune 96 > $O/bench_c3_q8p96.json 2>> $O/bench.err
timeout 900 python bench.py --config c2 --steps 3 --no-cpu-baseline --q8 > $O/bench_c2_q8.json 2>> $O/bench.err
