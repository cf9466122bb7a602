#!/bin/bash
# r02 call AI: tail skip (warps beyond M in the last round stop early) + cached grab order /
# unit table -- parity, C2 A/B, M sweep around the C2 shape, C3 regression
O=gpurun_out/r02ai; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_tail_skip.py tests/test_gpu_spec.py tests/test_gpu_parity.py tests/test_gpu_ragged.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for i in 1 2; do
  timeout 600 python bench.py --config c2 --steps 10 --no-cpu-baseline > $O/bench_c2_skip_$i.json 2>> $O/bench.err
  SDTW_NO_TAIL_SKIP=1 timeout 600 python bench.py --config c2 --steps 10 --no-cpu-baseline > $O/bench_c2_noskip_$i.json 2>> $O/bench.err
done
for M in 99840 100000 103680; do
  Z=512 N=2000 M=$M CONFIGS='[{}]' timeout 600 python scripts/sweep.py >> $O/sweep_m.jsonl 2>&1
  SDTW_NO_TAIL_SKIP=1 Z=512 N=2000 M=$M CONFIGS='[{}]' timeout 600 python scripts/sweep.py >> $O/sweep_m_noskip.jsonl 2>&1
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_c2.csv \
   python bench.py --config c2 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > $O/launches_c2_bench.json 2>&1
timeout 900 python bench.py --config c3 --steps 3 --no-cpu-baseline > $O/bench_c3.json 2>> $O/bench.err
cat $O/tests.log
