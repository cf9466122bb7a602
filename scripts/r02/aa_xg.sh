#!/bin/bash
# r02 call AA: query rows in global memory (XG) -- parity, and C5 / C3 rates auto vs forced layouts
O=gpurun_out/r02aa; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -rf --tb=short -k "query_rows or config1 or ragged or config5_shape or long_queries" 2>&1 | tail -15 > $O/tests.log
for n in 8000 4000 1000; do
TRACE=1 Z=512 N=$n M=1000000 CONFIGS='[{}, {"OPT_QUERY_ROWS": 1}, {"OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py >> $O/sweep_c5.jsonl 2>&1
done
Z=512 N=8000 M=1000000 CONFIGS='[{}, {"OPT_QUERY_ROWS": 1}, {"OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py > $O/sweep_n8000_costonly.jsonl 2>&1
Z=512 N=2000 M=10000000 CONFIGS='[{}, {"OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py > $O/sweep_c3.jsonl 2>&1
