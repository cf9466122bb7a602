#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py tests/test_gpu_ragged.py tests/test_gpu_half.py -q -x 2>&1 | tail -8 > gpurun_out/spec5_tests.log
CASES=";OPT_SCHED=2;OPT_SCHED=3,OPT_SEGMENTS=2;OPT_SCHED=3,OPT_SEGMENTS=4;OPT_SCHED=3,OPT_SEGMENTS=6;OPT_SCHED=3,OPT_LANES=4" timeout 900 python scripts/ragged_sweep.py > gpurun_out/ragged_spec.jsonl 2>&1
cat gpurun_out/spec5_tests.log gpurun_out/ragged_spec.jsonl | cut -c1-220
