#!/bin/bash
# r02 call E: checkpointed start index -- parity and C5 benches
O=gpurun_out/r02e; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_start_ckpt.py -q -x --tb=short 2>&1 | tail -30 > $O/tests_ckpt.log
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py tests/test_gpu_path.py -q -x --tb=short 2>&1 | tail -20 > $O/tests_parity.log
for c in c5_500 c5_1000 c5_4000 c5_8000; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench.err
done
