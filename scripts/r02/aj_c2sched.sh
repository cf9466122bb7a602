#!/bin/bash
# r02 call AJ: config-2 schedule knobs with the tail skip (segments x correction rounds x workers)
O=gpurun_out/r02aj; mkdir -p $O
Z=512 N=2000 M=100000 CONFIGS='[{}, {"OPT_SEGMENTS": 2, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 3, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 4, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 3}, {"OPT_SEGMENTS": 4}, {"OPT_SCHED": 2, "OPT_SEGMENTS": 1, "OPT_WORKERS": 4}, {"OPT_SCHED": 2, "OPT_SEGMENTS": 2}, {}]' timeout 600 python scripts/sweep.py > $O/sweep_c2.jsonl 2>&1
Z=512 N=2000 M=99840 CONFIGS='[{}, {"OPT_SEGMENTS": 2, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 3}, {}]' timeout 600 python scripts/sweep.py > $O/sweep_c2_99840.jsonl 2>&1
SDTW_DEBUG_PLAN=1 Z=512 N=2000 M=99840 CONFIGS='[{}]' timeout 600 python scripts/sweep.py > $O/plan_99840.txt 2>&1
SDTW_DEBUG_PLAN=1 Z=512 N=2000 M=100000 CONFIGS='[{}]' timeout 600 python scripts/sweep.py > $O/plan_100000.txt 2>&1
cat $O/sweep_c2.jsonl $O/sweep_c2_99840.jsonl
