#!/bin/bash
# r02 call B: full GPU suite (incl. full-size parity), smoke, ncu of the C3 DP launch, benches
O=gpurun_out/r02b; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -rf --tb=short 2>&1 | tail -40 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o $O/c3_dp python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c3.log 2>&1
timeout 600 python bench.py --steps 5 > $O/bench_c3.json 2> $O/bench_c3.err
for c in c2 c5_500 c5_1000 c5_4000 c5_8000; do
  timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
