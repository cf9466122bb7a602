#!/bin/bash
# r02 call BC: config-5 segment counts with the new ring widths / correction length (checkpointed start)
O=gpurun_out/r02bc; mkdir -p $O
for N in 500 1000; do
TRACE=1 Z=512 N=$N M=1000000 CONFIGS='[{}, {"OPT_SEGMENTS": 6}, {"OPT_SEGMENTS": 20}, {"OPT_SEGMENTS": 30}, {}]' timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": $N, \"r\": /; s/$/}/" >> $O/seg.jsonl 2>&1
done
for N in 4000 8000; do
TRACE=1 Z=512 N=$N M=1000000 CONFIGS='[{}, {"OPT_SEGMENTS": 4}, {"OPT_SEGMENTS": 8}, {"OPT_SEGMENTS": 12}, {}]' timeout 900 python scripts/sweep.py | sed "s/^/{\"N\": $N, \"r\": /; s/$/}/" >> $O/seg.jsonl 2>&1
done
for N in 500 1000 4000 8000; do SDTW_DEBUG_PLAN=1 TRACE=1 Z=512 N=$N M=1000000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py 2>&1 | grep plan | head -1 >> $O/plans.txt; done
cat $O/seg.jsonl $O/plans.txt
