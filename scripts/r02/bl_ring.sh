#!/bin/bash
# r02 call BL: config 5 short queries on 2-warp rings -- shallower inter-warp rings for an 8th resident CTA
O=gpurun_out/r02bl; mkdir -p $O
TRACE=1 Z=512 N=1000 M=1000000 CONFIGS='[{}, {"OPT_RING": 512}, {"OPT_CHUNK": 64}, {"OPT_CHUNK": 64, "OPT_RING": 256}, {}]' timeout 900 python scripts/sweep.py > $O/c5_1000.jsonl 2>&1
TRACE=1 Z=512 N=500 M=1000000 CONFIGS='[{}, {"OPT_RING": 256}, {"OPT_CHUNK": 32}, {}]' timeout 900 python scripts/sweep.py > $O/c5_500.jsonl 2>&1
for cfg in '{}' '{"OPT_RING": 512}'; do SDTW_DEBUG_PLAN=1 TRACE=1 Z=512 N=1000 M=1000000 CONFIGS="[$cfg]" timeout 600 python scripts/sweep.py 2>&1 | grep plan | head -1 >> $O/plans.txt; done
cat $O/*.jsonl $O/plans.txt
