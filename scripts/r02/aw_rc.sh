#!/bin/bash
# r02 call AW: correction length (OPT_SPEC_ROUNDS) vs the auto 3N rule at config 2 and config 5 N = 4,000 / 8,000
O=gpurun_out/r02aw; mkdir -p $O
Z=512 N=2000 M=100000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 1}, {}, {"OPT_SPEC_ROUNDS": 1}]' timeout 600 python scripts/sweep.py > $O/rc_c2.jsonl 2>&1
TRACE=1 Z=512 N=4000 M=1000000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 2}, {"OPT_SPEC_ROUNDS": 3}, {}]' timeout 900 python scripts/sweep.py > $O/rc_c5_4000.jsonl 2>&1
TRACE=1 Z=512 N=8000 M=1000000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 3}, {"OPT_SPEC_ROUNDS": 4}, {"OPT_SPEC_ROUNDS": 5}, {}]' timeout 900 python scripts/sweep.py > $O/rc_c5_8000.jsonl 2>&1
TRACE=1 Z=512 N=1000 M=1000000 CONFIGS='[{}, {"OPT_SEGMENTS": 4}, {"OPT_SEGMENTS": 8}, {}]' timeout 900 python scripts/sweep.py > $O/seg_c5_1000.jsonl 2>&1
SDTW_DEBUG_PLAN=1 TRACE=1 Z=512 N=8000 M=1000000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py > $O/plan_c5_8000.txt 2>&1
cat $O/*.jsonl; grep plan $O/plan_c5_8000.txt | head -3
