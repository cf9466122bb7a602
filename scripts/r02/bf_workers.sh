#!/bin/bash
# r02 call BF: config 3 with 3 vs 4 resident workers per SM
O=gpurun_out/r02bf; mkdir -p $O
Z=512 N=2000 M=10000000 CONFIGS='[{}, {"OPT_WORKERS": 3}, {"OPT_WORKERS": 3, "OPT_SEGMENTS": 8}, {}]' timeout 900 python scripts/sweep.py > $O/workers_c3.jsonl 2>&1
cat $O/workers_c3.jsonl
