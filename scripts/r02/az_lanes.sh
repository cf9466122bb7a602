#!/bin/bash
# r02 call AZ: warps per ring (OPT_LANES) under the speculative schedule, cost/end and checkpointed start
O=gpurun_out/r02az; mkdir -p $O
L='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 3}, {"OPT_LANES": 4}, {"OPT_LANES": 2}]'
for N in 500 1000 2000 4000 8000; do
  Z=512 N=$N M=1000000 CONFIGS="$L" timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": $N, \"M\": 1000000, \"trace\": 0, \"r\": /; s/$/}/" >> $O/lanes.jsonl 2>&1
done
for N in 2000 4000 8000; do
  TRACE=1 Z=512 N=$N M=1000000 CONFIGS="$L" timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": $N, \"M\": 1000000, \"trace\": 1, \"r\": /; s/$/}/" >> $O/lanes.jsonl 2>&1
done
Z=512 N=2000 M=100000 CONFIGS="$L" timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": 2000, \"M\": 100000, \"trace\": 0, \"r\": /; s/$/}/" >> $O/lanes.jsonl 2>&1
Z=512 N=2000 M=10000000 CONFIGS='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 3}]' timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": 2000, \"M\": 10000000, \"trace\": 0, \"r\": /; s/$/}/" >> $O/lanes.jsonl 2>&1
cat $O/lanes.jsonl
