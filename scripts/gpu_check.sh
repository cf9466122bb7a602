#!/bin/bash
# One GPU-box session: smoke, parity tests, short benches. Outputs under gpurun_out/.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
{ nvidia-smi -L; nproc; lscpu | grep -E 'Model name|Socket|Core|Thread' ; } > gpurun_out/box.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout ${PYTEST_TIMEOUT:-1200} python -m pytest tests -m gpu -q --timeout 400 ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err
tail -n 3 gpurun_out/smoke.log gpurun_out/pytest_gpu.log; cat gpurun_out/bench_c2.json gpurun_out/bench_c3.json
