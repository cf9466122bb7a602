#!/bin/bash
# r02 call BB: ragged batches on 4-warp rings -- ragged / refsplit / spec tests and the c6 line
O=gpurun_out/r02bb; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_spec.py tests/test_gpu_refsplit.py tests/test_gpu_half.py tests/test_gpu_q8.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
timeout 900 python bench.py --config c6_ragged --steps 5 --no-cpu-baseline > $O/bench_c6_ragged.json 2>> $O/bench.err
cat $O/tests.log; tail -3 $O/bench.err
