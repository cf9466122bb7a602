#!/bin/bash
# r02 call K: speculative worst case (c3_straddle) with the new vs the r01 fixup; C2 schedule
# sweep; ncu of the uint8 DP launch
O=gpurun_out/r02k; mkdir -p $O
timeout 600 python bench.py --config c3_straddle --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_straddle.json 2>> $O/bench.err
SDTW_LIB=$PWD/variants/fixseq.so timeout 900 python bench.py --config c3_straddle --steps 3 --no-cpu-baseline --no-e2e > $O/bench_c3_straddle_fixseq.json 2>> $O/bench.err
Z=512 N=2000 M=100000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 1}, {"OPT_LANES": 5}, {"OPT_LANES": 6}, {"OPT_LANES": 3}, {"OPT_LANES": 5, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 3, "OPT_SPEC_ROUNDS": 1}, {"OPT_SCHED": 2}, {"OPT_SCHED": 2, "OPT_LANES": 5}, {"OPT_CHUNK": 64}, {"OPT_WORKERS": 3}]' timeout 900 python scripts/sweep.py > $O/sweep_c2.jsonl 2>&1
Z=512 N=2000 M=10000000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 1}, {"OPT_LANES": 5}]' timeout 900 python scripts/sweep.py > $O/sweep_c3.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp2 -s 3 -c 1 \
   -o $O/c3_q8 python bench.py --config c3 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e --q8 > $O/ncu_q8.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/q8_launches.csv \
   python bench.py --config c3 --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --q8 > $O/ncu_q8_list.log 2>&1
