#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_half.py tests/test_gpu_spec.py -q -x 2>&1 | tail -4 > gpurun_out/spec7_tests.log
CASES="512:2000:10000000:OPT_PRECISION=16,OPT_SCHED=2;512:2000:10000000:OPT_PRECISION=16;64:2000:10000000:OPT_PRECISION=16,OPT_SCHED=1;64:2000:10000000:OPT_PRECISION=16" timeout 900 python scripts/spec_sweep.py > gpurun_out/spec_half.jsonl 2>&1
timeout 600 python bench.py --half --steps 3 > gpurun_out/bench_half.json 2>/dev/null
cat gpurun_out/spec7_tests.log gpurun_out/spec_half.jsonl | cut -c1-200; cut -c1-400 gpurun_out/bench_half.json
