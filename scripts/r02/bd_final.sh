#!/bin/bash
# r02 call BD: final evidence of the round (2-warp rings for short queries, correction N + half a round, 4-warp ragged rings)
# line, its launch list, ncu --set full of the config-3 DP launch, and the other workloads' lines
O=gpurun_out/r02bd; mkdir -p $O
(nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv; nvcc --version | tail -2) > $O/env.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q -rf --tb=short --durations=15 2>&1 | tail -45 > $O/gpu_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 900 python bench.py > $O/bench_c3.json 2> $O/bench_c3.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c3.csv \
   python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_bench.json 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o $O/c3_dp python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c3.log 2>&1
for c in c2 c5_500 c5_1000 c5_4000 c5_8000 c6_ragged c3_straddle; do
  timeout 900 python bench.py --config $c --steps 3 --no-cpu-baseline > $O/bench_$c.json 2>> $O/bench.err
done
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --half > $O/bench_c3_half.json 2>> $O/bench.err
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 > $O/bench_c3_q8.json 2>> $O/bench.err
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline --q8 --q8-prune 96 > $O/bench_c3_q8p96.json 2>> $O/bench.err
timeout 900 python bench.py --config c5_1000 --steps 3 --no-cpu-baseline --path > $O/bench_c5_1000_path.json 2>> $O/bench.err
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 3 -c 1 \
   -o $O/c2_dp python bench.py --config c2 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > $O/ncu_c2.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
   python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_c2_bench.json 2>&1
