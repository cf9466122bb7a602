#!/bin/bash
# r02 call G (session 2 re-entry): full GPU suite + smoke + benches on HEAD (checkpointed start index)
O=gpurun_out/r02g; mkdir -p $O
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; nvcc --version | tail -2) > $O/env.txt 2>&1
timeout 1800 python -m pytest tests -m gpu -q -rf --tb=short 2>&1 | tail -40 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 600 python bench.py --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
timeout 600 python bench.py --config c2 --steps 5 --no-cpu-baseline > $O/bench_c2.json 2>> $O/bench.err
