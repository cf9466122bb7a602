#!/bin/bash
# r02 call AX: auto correction length N + half a round -- spec / start / fullsize tests and the config-5 lines
O=gpurun_out/r02ax; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_spec.py tests/test_gpu_start_ckpt.py tests/test_gpu_fullsize.py tests/test_gpu_ragged.py tests/test_gpu_half.py tests/test_gpu_q8.py tests/test_gpu_path.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for c in c5_500 c5_1000 c5_4000 c5_8000 c2 c6_ragged; do timeout 900 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
cat $O/tests.log; tail -3 $O/bench.err
