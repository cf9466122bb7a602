#!/bin/bash
# r02 call BN: full GPU suite + smoke + default bench line on the final library (after the 2-warp ring-depth rule)
O=gpurun_out/r02bn; mkdir -p $O
timeout 2700 python -m pytest tests -m gpu -q -rf --tb=short --durations=5 2>&1 | tail -20 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
for c in c2 c5_500 c5_1000 c5_4000 c5_8000 c6_ragged; do timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err; done
tail -3 $O/gpu_tests.log; cat $O/smoke.log | cut -c1-80
