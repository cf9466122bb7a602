#!/bin/bash
# r02 call AQ: unit overhead in the speculative list-scheduling model (SDTW_SPEC_OVH) across Pr = 25..30
O=gpurun_out/r02aq; mkdir -p $O
for ov in 0 0.25 0.5 1.0; do
for M in 96000 99840 100000 107520 115200; do
  SDTW_SPEC_OVH=$ov Z=512 N=2000 M=$M CONFIGS='[{}, {}]' timeout 300 python scripts/sweep.py | sed "s/^/{\"ovh\": $ov, \"M\": $M, \"r\": /; s/$/}/" >> $O/ovh.jsonl 2>&1
done; done
cat $O/ovh.jsonl
