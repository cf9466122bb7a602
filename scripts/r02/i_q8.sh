#!/bin/bash
# r02 call I: uint8-codebook variant (NEXT-3) parity + the packed-half refactor regression; q8 benches
O=gpurun_out/r02i; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_q8.py tests/test_gpu_half.py -q -rf --tb=short 2>&1 | tail -30 > $O/tests.log
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 > $O/bench_c3_q8.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 --q8-prune 96 > $O/bench_c3_q8p96.json 2>> $O/bench.err
timeout 600 python bench.py --config c3 --steps 3 --no-cpu-baseline --no-e2e --half > $O/bench_c3_half.json 2>> $O/bench.err
timeout 600 python bench.py --config c2 --steps 5 --no-cpu-baseline --q8 > $O/bench_c2_q8.json 2>> $O/bench.err
