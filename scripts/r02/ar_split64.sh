#!/bin/bash
# r02 call AR: two-segment plan split at 16/25 of the rounds -- tests, M map (Pr = 25..30), C2 line
O=gpurun_out/r02ar; mkdir -p $O
timeout 1200 python -m pytest tests/test_gpu_spec.py tests/test_gpu_start_ckpt.py tests/test_gpu_tail_skip.py tests/test_gpu_ragged.py tests/test_gpu_half.py tests/test_gpu_q8.py -q -x -rf --tb=short 2>&1 | tail -15 > $O/tests.log
for M in 96000 99840 100000 103680 107520 111360 115200; do
  Z=512 N=2000 M=$M CONFIGS='[{}, {}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"M\": $M, \"r\": /; s/$/}/" >> $O/mmap.jsonl 2>&1
done
for Z in 256 384; do
  Z=$Z N=2000 M=100000 CONFIGS='[{}, {"OPT_SEGMENTS": 3}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"Z\": $Z, \"r\": /; s/$/}/" >> $O/zmap.jsonl 2>&1
done
Z=512 N=4000 M=200000 CONFIGS='[{}, {"OPT_SEGMENTS": 3}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"N\": 4000, \"r\": /; s/$/}/" >> $O/zmap.jsonl 2>&1
for i in 1 2; do timeout 600 python bench.py --config c2 --steps 10 --no-cpu-baseline > $O/bench_c2_$i.json 2>> $O/bench.err; done
cat $O/tests.log
