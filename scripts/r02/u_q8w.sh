#!/bin/bash
# r02 call U: uint8 kernel at W = 14 vs 30 (instruction-footprint vs per-step overhead)
O=gpurun_out/r02u; mkdir -p $O
SDTW_LIB=$PWD/variants/q8w14.so Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_PRECISION": 8}, {"OPT_PRECISION": 8, "OPT_SEGMENT_W": 14}, {"OPT_PRECISION": 8, "OPT_SEGMENT_W": 14, "OPT_LANES": 8}, {"OPT_PRECISION": 8, "OPT_Q8_PRUNE": 96}, {"OPT_PRECISION": 8, "OPT_Q8_PRUNE": 96, "OPT_SEGMENT_W": 14}]' timeout 1200 python scripts/sweep.py > $O/sweep_q8w.jsonl 2>&1
