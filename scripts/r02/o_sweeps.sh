#!/bin/bash
# r02 call O: packed-half and uint8 schedule sweeps at config 3 (W, lanes, chunk)
O=gpurun_out/r02o; mkdir -p $O
Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_PRECISION": 16}, {"OPT_PRECISION": 16, "OPT_SEGMENT_W": 62}, {"OPT_PRECISION": 16, "OPT_SEGMENT_W": 62, "OPT_LANES": 2}, {"OPT_PRECISION": 16, "OPT_LANES": 8}, {"OPT_PRECISION": 16, "OPT_CHUNK": 64}, {"OPT_PRECISION": 16, "OPT_SEGMENT_W": 62, "OPT_CHUNK": 128}]' timeout 1200 python scripts/sweep.py > $O/sweep_half.jsonl 2>&1
Z=512 N=2000 M=10000000 CONFIGS='[{"OPT_PRECISION": 8}, {"OPT_PRECISION": 8, "OPT_LANES": 2}, {"OPT_PRECISION": 8, "OPT_LANES": 8}, {"OPT_PRECISION": 8, "OPT_CHUNK": 64}, {"OPT_PRECISION": 8, "OPT_CHUNK": 32}]' timeout 1200 python scripts/sweep.py > $O/sweep_q8.jsonl 2>&1
