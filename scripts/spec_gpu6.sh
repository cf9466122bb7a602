#!/bin/bash
mkdir -p gpurun_out
CASES=";OPT_SCHED=3,OPT_SEGMENTS=3;OPT_SCHED=3,OPT_SEGMENTS=4;OPT_SCHED=3,OPT_SEGMENTS=5;OPT_SCHED=3,OPT_SEGMENTS=8;OPT_SCHED=2" timeout 900 python scripts/ragged_sweep.py > gpurun_out/ragged_spec2.jsonl 2>&1
LMIN=500 LMAX=2000 CASES=";OPT_SCHED=2" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_spec2.jsonl 2>&1
LMIN=2000 LMAX=8000 CASES=";OPT_SCHED=2" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_spec2.jsonl 2>&1
timeout 600 python -m pytest tests/test_gpu_ragged.py tests/test_gpu_spec.py -q -x 2>&1 | tail -2 >> gpurun_out/ragged_spec2.jsonl
cat gpurun_out/ragged_spec2.jsonl | cut -c1-200
