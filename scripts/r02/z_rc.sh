#!/bin/bash
O=gpurun_out/r02z; mkdir -p $O
Z=512 N=2000 M=100000 CONFIGS='[{}, {"OPT_SEGMENTS": 2, "OPT_SPEC_ROUNDS": 1}, {"OPT_SEGMENTS": 2}, {"OPT_SEGMENTS": 2, "OPT_SPEC_ROUNDS": 1, "OPT_CHUNK": 64}]' timeout 900 python scripts/sweep.py > $O/sweep_c2_rc.jsonl 2>&1
Z=512 N=1000 M=1000000 CONFIGS='[{}, {"OPT_SPEC_ROUNDS": 1}]' timeout 900 python scripts/sweep.py > $O/sweep_c5_1000_rc.jsonl 2>&1
