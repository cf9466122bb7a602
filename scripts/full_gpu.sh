#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > gpurun_out/gpu_tests.log
timeout 600 python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
CASES="64:2000:10000000:;32:2000:10000000:;128:2000:10000000:;16:2000:10000000:" timeout 600 python scripts/spec_sweep.py > gpurun_out/spec_auto.jsonl 2>&1
cat gpurun_out/gpu_tests.log gpurun_out/bench_c3.json gpurun_out/spec_auto.jsonl; tail -3 gpurun_out/bench_c3.err
