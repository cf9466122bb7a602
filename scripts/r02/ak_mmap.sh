#!/bin/bash
# r02 call AK: config-2 shape at reference lengths around round multiples (3,840 columns per round)
O=gpurun_out/r02ak; mkdir -p $O
for M in 96000 99839 99840 99841 100000 103680 103681 107520 115200; do
  Z=512 N=2000 M=$M CONFIGS='[{}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"M\": $M, \"r\": /; s/$/}/" >> $O/mmap.jsonl 2>&1
done
cat $O/mmap.jsonl
