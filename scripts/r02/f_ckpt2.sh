#!/bin/bash
# r02 call F: checkpointed start index v2 (one launch, end-round first windows); cost-only C5 rates
O=gpurun_out/r02f; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_start_ckpt.py tests/test_gpu_spec.py -q -x --tb=short 2>&1 | tail -20 > $O/tests.log
for c in c5_500 c5_1000 c5_4000 c5_8000; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > $O/bench_$c.json 2>> $O/bench.err
done
for n in 500 1000 4000 8000; do
  Z=512 N=$n M=1000000 CONFIGS='[{}]' timeout 300 python scripts/sweep.py >> $O/costonly_c5.jsonl 2>&1
done
