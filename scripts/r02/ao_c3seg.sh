#!/bin/bash
# r02 call AO: config-3 segment count / correction length with the final library (tail of late B units)
O=gpurun_out/r02ao; mkdir -p $O
Z=512 N=2000 M=10000000 CONFIGS='[{}, {"OPT_SEGMENTS": 5}, {"OPT_SEGMENTS": 7}, {"OPT_SEGMENTS": 8}, {"OPT_SEGMENTS": 10}, {"OPT_SEGMENTS": 12}, {"OPT_SEGMENTS": 6, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 8, "OPT_SPEC_ROUNDS": 1}, {}]' timeout 900 python scripts/sweep.py > $O/sweep_c3.jsonl 2>&1
SDTW_UNIT_LOG=$O/log_c3_s8.txt Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_SEGMENTS": 8}]' timeout 300 python scripts/sweep.py > /dev/null 2>&1; python scripts/unit_timeline.py $O/log_c3_s8.txt > $O/sum_c3_s8.txt 2>&1
cat $O/sweep_c3.jsonl $O/sum_c3_s8.txt
