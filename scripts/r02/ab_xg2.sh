#!/bin/bash
# r02 call AB: XG = rows + wrap ring in global memory -- parity, C5 / ragged / C3 rates
O=gpurun_out/r02ab; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_start_ckpt.py tests/test_gpu_ragged.py -q -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for n in 8000 4000; do
TRACE=1 Z=512 N=$n M=1000000 CONFIGS='[{"OPT_QUERY_ROWS": 1}, {}, {"OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py >> $O/sweep_c5.jsonl 2>&1
done
Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_QUERY_ROWS": 1}, {}, {"OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py > $O/sweep_c3.jsonl 2>&1
timeout 900 python bench.py --config c6_ragged --steps 3 --no-cpu-baseline > $O/bench_c6_ragged.json 2>> $O/bench.err
timeout 900 python bench.py --config c5_8000 --steps 3 --no-cpu-baseline > $O/bench_c5_8000.json 2>> $O/bench.err
