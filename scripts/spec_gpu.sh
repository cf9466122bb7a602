#!/bin/bash
# speculative segments: GPU parity + small-batch timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spec.py -x -q 2>&1 | tail -15 > gpurun_out/spec_tests.log
C=""
for Z in 64; do for S in 7 28 56; do C="$C;$Z:2000:10000000:OPT_SCHED=3,OPT_SEGMENTS=$S"; done; done
for Z in 200 300 444; do C="$C;$Z:2000:10000000:OPT_SCHED=2;$Z:2000:10000000:OPT_SCHED=3"; done
C="$C;64:2000:10000000:OPT_SCHED=3,OPT_WORKERS=2"
CASES="${CASES:-${C#;}}" timeout 1200 python scripts/spec_sweep.py > gpurun_out/spec_sweep2.jsonl 2> gpurun_out/spec_sweep.err
cat gpurun_out/spec_tests.log gpurun_out/spec_sweep2.jsonl; tail -5 gpurun_out/spec_sweep.err
