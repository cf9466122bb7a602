#!/bin/bash
# r02 call AC: rows-only XG -- bench lines of the long-query workloads, ragged auto vs forced
O=gpurun_out/r02ac; mkdir -p $O
for c in c5_8000 c5_4000 c6_ragged; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -rf --tb=short -k "config5" 2>&1 | tail -5 > $O/fullsize_c5.log
