#!/bin/bash
# r02 call P: the fixed-slot row-pair tile loop vs the kernel's strip-pair mix (mixbench)
O=gpurun_out/r02p; mkdir -p $O
cd scripts
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tilebench2 tilebench2.cu && ./tilebench2 > ../$O/tilebench2.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o mixbench mixbench.cu && ./mixbench > ../$O/mixbench.txt 2>&1
