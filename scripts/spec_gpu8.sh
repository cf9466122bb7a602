#!/bin/bash
mkdir -p gpurun_out
C="512:2000:10000000:"
for o in OPT_CHUNK=64 OPT_CHUNK=96 OPT_CHUNK=160 OPT_RING=512 OPT_RING=2048 OPT_SEGMENTS=7 OPT_WORKERS=3 OPT_LANES=3 OPT_LANES=5 OPT_SPEC_ROUNDS=1; do C="$C;512:2000:10000000:$o"; done
CASES="$C" timeout 1500 python scripts/spec_sweep.py > gpurun_out/spec_tune.jsonl 2>&1
cat gpurun_out/spec_tune.jsonl | cut -c1-160
