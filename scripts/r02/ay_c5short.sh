#!/bin/bash
# r02 call AY: config 5 short queries (N = 500 / 1,000, checkpointed start): ring width and chunk
O=gpurun_out/r02ay; mkdir -p $O
TRACE=1 Z=512 N=500 M=1000000 CONFIGS='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 2, "OPT_CHUNK": 64}, {"OPT_LANES": 8}, {"OPT_CHUNK": 16}, {"OPT_SEGMENTS": 3}, {"OPT_SEGMENTS": 10}, {}]' timeout 900 python scripts/sweep.py > $O/c5_500.jsonl 2>&1
TRACE=1 Z=512 N=1000 M=1000000 CONFIGS='[{}, {"OPT_LANES": 2}, {"OPT_LANES": 2, "OPT_CHUNK": 128}, {"OPT_CHUNK": 128}, {"OPT_SEGMENTS": 3}, {}]' timeout 900 python scripts/sweep.py > $O/c5_1000.jsonl 2>&1
SDTW_DEBUG_PLAN=1 TRACE=1 Z=512 N=500 M=1000000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py 2>&1 | grep plan | head -2 > $O/plan.txt
SDTW_DEBUG_PLAN=1 TRACE=1 Z=512 N=1000 M=1000000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py 2>&1 | grep plan | head -2 >> $O/plan.txt
cat $O/*.jsonl $O/plan.txt
