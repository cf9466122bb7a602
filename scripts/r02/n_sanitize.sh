#!/bin/bash
# r02 call N: compute-sanitizer on the final library (incl. uint8, checkpointed start, split
# calls); row-pair tile microbenchmark
O=gpurun_out/r02n; mkdir -p $O
(cd scripts && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tilebench tilebench.cu && ./tilebench) > $O/tilebench.txt 2>&1
bash scripts/sanitize.sh $O > /dev/null 2>&1
grep -h "SUMMARY" $O/sanitize_*.log >> $O/sanitize_summary.txt
