#!/bin/bash
O=gpurun_out/r02ae; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_start_ckpt.py tests/test_gpu_ragged.py tests/test_gpu_spec.py -q -rf --tb=short 2>&1 | tail -8 > $O/tests.log
for c in c5_8000 c5_4000 c6_ragged; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rf --tb=short -k "c5_8000" 2>&1 | tail -3 > $O/fullsize.log
