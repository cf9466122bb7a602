#!/bin/bash
# r02 call BJ: the per-rank shard of config 3 under strong scaling (512 / P queries vs 10M on one GPU)
O=gpurun_out/r02bj; mkdir -p $O
for Z in 64 128 256 512; do
  Z=$Z N=2000 M=10000000 CONFIGS='[{}, {}]' timeout 600 python scripts/sweep.py | sed "s/^/{\"Z\": $Z, \"r\": /; s/$/}/" >> $O/shards.jsonl 2>&1
done
cat $O/shards.jsonl
