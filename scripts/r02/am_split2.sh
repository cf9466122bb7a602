#!/bin/bash
# r02 call AM: split point of the two-segment plan, wider (Pr = 25..32)
O=gpurun_out/r02am; mkdir -p $O
run() { Z=512 N=2000 M=$1 SDTW_SPEC_SPLIT=$2 CONFIGS='[{}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"M\": $1, \"split\": $2, \"r\": /; s/$/}/" >> $O/split.jsonl 2>&1; }
for s in 0 13 14 15 16 17; do run 96000 $s; done
for s in 17 18 19; do run 99840 $s; done
for s in 17 18 19; do run 100000 $s; done
for s in 19 20 21; do run 107520 $s; done
for s in 0 15 16 17 18 19 20 21 22; do run 115200 $s; done
cat $O/split.jsonl
