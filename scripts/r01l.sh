#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -6 > gpurun_out/r01l_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r01l_smoke.log 2>&1
bash scripts/round_evidence.sh r01l > /dev/null 2>&1
for c in c2 c5_1000 c6_ragged; do timeout 600 python bench.py --config $c --steps 3 > gpurun_out/r01l_bench_$c.json 2>/dev/null; done
timeout 600 python bench.py --half --steps 3 > gpurun_out/r01l_bench_half.json 2>/dev/null
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/r01l_bench_ref.json 2>/dev/null
cat gpurun_out/r01l_gpu_tests.log gpurun_out/r01l_smoke.log; cut -c1-300 gpurun_out/r01l_bench.json gpurun_out/r01l_bench_c2.json gpurun_out/r01l_bench_c5_1000.json gpurun_out/r01l_bench_ref.json; ls gpurun_out | grep r01l
