#!/bin/bash
# r02 call Y: per-level recomputation workspaces (nested speculative re-runs), spec / start / q8 suites
O=gpurun_out/r02y; mkdir -p $O
timeout 1800 python -m pytest tests/test_gpu_spec.py tests/test_gpu_start_ckpt.py tests/test_gpu_q8.py tests/test_gpu_ragged.py tests/test_gpu_refsplit.py -q -rf --tb=short 2>&1 | tail -15 > $O/tests.log
timeout 900 python bench.py --config c3_straddle --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_straddle.json 2>> $O/bench.err
