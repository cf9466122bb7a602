#!/bin/bash
# r02 call AD: N = 8,000 with global query rows -- can a shallower ring reach 4 CTAs per SM?
O=gpurun_out/r02ad; mkdir -p $O
TRACE=1 Z=512 N=8000 M=1000000 CONFIGS='[{}, {"OPT_CHUNK": 64, "OPT_RING": 256}, {"OPT_CHUNK": 64, "OPT_RING": 512}, {"OPT_CHUNK": 32, "OPT_RING": 128}, {"OPT_CHUNK": 64, "OPT_RING": 256, "OPT_QUERY_ROWS": 2}]' timeout 900 python scripts/sweep.py > $O/sweep_c5_8000.jsonl 2>&1
Z=512 N=8000 M=1000000 CONFIGS='[{}, {"OPT_CHUNK": 64, "OPT_RING": 256}]' timeout 900 python scripts/sweep.py > $O/sweep_n8000.jsonl 2>&1
