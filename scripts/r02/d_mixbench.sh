#!/bin/bash
O=gpurun_out/r02d; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mixbench scripts/mixbench.cu && /tmp/mixbench > $O/mixbench.txt 2>&1
