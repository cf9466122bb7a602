#!/bin/bash
# r02 call W: where config 2 loses against config 3 -- correction length, segments, one unit per query
O=gpurun_out/r02w; mkdir -p $O
Z=512 N=2000 M=100000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 1}, {"OPT_SCHED": 2, "OPT_SEGMENTS": 1}, {"OPT_SCHED": 2, "OPT_SEGMENTS": 2}, {"OPT_SCHED": 1}, {"OPT_SEGMENTS": 3}, {"OPT_SEGMENTS": 4, "OPT_SPEC_ROUNDS": 1}, {"OPT_WORKERS": 4, "OPT_SCHED": 2, "OPT_SEGMENTS": 1}]' timeout 900 python scripts/sweep.py > $O/sweep_c2.jsonl 2>&1
Z=512 N=2000 M=99840 CONFIGS='[{}]' timeout 900 python scripts/sweep.py > $O/sweep_c2_whole_rounds.jsonl 2>&1
