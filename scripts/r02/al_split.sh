#!/bin/bash
# r02 call AL: speculative split point of the two-segment plan (config-2 shapes, Pr = 26/27/28)
O=gpurun_out/r02al; mkdir -p $O
run() { Z=512 N=2000 M=$1 SDTW_SPEC_SPLIT=$2 CONFIGS='[{}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"M\": $1, \"split\": $2, \"r\": /; s/$/}/" >> $O/split.jsonl 2>&1; }
for s in 0 11 12 13 14 15 16; do run 99840 $s; done
for s in 0 12 13 14 15 16; do run 100000 $s; done
for s in 0 13 15 16 17 18; do run 107520 $s; done
cat $O/split.jsonl
