#!/bin/bash
# r02 call AN: per-unit timelines of the speculative schedule (good and bad split points)
O=gpurun_out/r02an; mkdir -p $O
run() { SDTW_UNIT_LOG=$O/log_$1_$2.txt Z=512 N=2000 M=$1 SDTW_SPEC_SPLIT=$2 CONFIGS='[{}]' timeout 300 python scripts/sweep.py > /dev/null 2>&1; python scripts/unit_timeline.py $O/log_$1_$2.txt > $O/sum_$1_$2.txt 2>&1; }
run 115200 17; run 115200 19; run 100000 0; run 99840 0; run 99840 14
Z=512 N=2000 M=10000000 SDTW_UNIT_LOG=$O/log_c3.txt CONFIGS='[{}]' timeout 300 python scripts/sweep.py > /dev/null 2>&1; python scripts/unit_timeline.py $O/log_c3.txt > $O/sum_c3.txt 2>&1
head -c 1000000 $O/log_115200_17.txt > /dev/null
cat $O/sum_*.txt
