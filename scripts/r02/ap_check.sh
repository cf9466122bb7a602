#!/bin/bash
# r02 call AP: schedule tables copied in stream order (event-guarded) -- spec / parity / ragged /
# refsplit / nccl / tail-skip tests, config 2 and 3 bench lines
O=gpurun_out/r02ap; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_tail_skip.py tests/test_gpu_spec.py tests/test_gpu_parity.py tests/test_gpu_ragged.py tests/test_gpu_refsplit.py tests/test_gpu_nccl.py tests/test_gpu_start_ckpt.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
timeout 600 python bench.py --config c2 --steps 10 --no-cpu-baseline > $O/bench_c2.json 2>> $O/bench.err
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2>> $O/bench.err
cat $O/tests.log; tail -3 $O/bench.err
