#!/bin/bash
# r02 call AU: tail skip as early stop + nominal-end publish (no extra live registers), ported to
# the half / uint8 kernels; unit-log slot in shared memory -- tests and the affected bench lines
O=gpurun_out/r02au; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_tail_skip.py tests/test_gpu_spec.py tests/test_gpu_parity.py tests/test_gpu_half.py tests/test_gpu_q8.py tests/test_gpu_start_ckpt.py tests/test_gpu_ragged.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for c in c2 c5_500 c5_1000; do timeout 600 python bench.py --config $c --steps 5 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2>> $O/bench.err
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --half > $O/bench_c3_half.json 2>> $O/bench.err
timeout 900 python bench.py --config c2 --steps 5 --no-cpu-baseline --half > $O/bench_c2_half.json 2>> $O/bench.err
cat $O/tests.log; tail -3 $O/bench.err
