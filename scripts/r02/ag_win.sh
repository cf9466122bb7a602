#!/bin/bash
# r02 call AG: strip-wise window DP of the checkpointed start index -- parity and C5 rates
O=gpurun_out/r02ag; mkdir -p $O
timeout 1500 python -m pytest tests/test_gpu_start_ckpt.py tests/test_gpu_path.py tests/test_gpu_spec.py -q -rf --tb=short 2>&1 | tail -8 > $O/tests.log
for c in c5_500 c5_1000 c5_4000 c5_8000; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 900 python bench.py --config c5_1000 --steps 3 --no-cpu-baseline --path > $O/bench_c5_1000_path.json 2>> $O/bench.err
timeout 1200 python -m pytest tests/test_gpu_fullsize.py -q -rf --tb=short -k "config5" 2>&1 | tail -3 > $O/fullsize.log
