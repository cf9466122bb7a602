#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -12 > gpurun_out/gpu_tests.log
TRACE=1 CASES="64:1000:10000000:OPT_SCHED=1;64:1000:10000000:;512:1000:10000000:;64:4000:10000000:OPT_SCHED=1;64:4000:10000000:" timeout 900 python scripts/spec_sweep.py > gpurun_out/spec_trace.jsonl 2>&1
cat gpurun_out/gpu_tests.log gpurun_out/spec_trace.jsonl
