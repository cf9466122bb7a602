#!/bin/bash
mkdir -p gpurun_out
CASES="OPT_LANES=2;OPT_LANES=6;OPT_LANES=8;OPT_LANES=8,OPT_CHUNK=64;OPT_LANES=8,OPT_CHUNK=128;OPT_LANES=8,OPT_WORKERS=1;OPT_LANES=8,OPT_SEGMENTS=4;OPT_LANES=8,OPT_SEGMENTS=16;OPT_LANES=8,OPT_PAD=256" timeout 900 python scripts/ragged_sweep.py > gpurun_out/ragged_sweep2.jsonl 2>&1
LMIN=500 LMAX=2000 CASES="OPT_LANES=2;OPT_LANES=8;OPT_LANES=8,OPT_CHUNK=64" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_sweep2.jsonl 2>&1
LMIN=2000 LMAX=8000 CASES="OPT_LANES=8;OPT_LANES=8,OPT_CHUNK=128" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_sweep2.jsonl 2>&1
CASES="512:2000:100000:;512:2000:100000:OPT_LANES=8;512:2000:100000:OPT_LANES=6;512:2000:100000:OPT_LANES=8,OPT_CHUNK=64" timeout 300 python scripts/spec_sweep.py >> gpurun_out/ragged_sweep2.jsonl 2>&1
cat gpurun_out/ragged_sweep2.jsonl | cut -c1-200
