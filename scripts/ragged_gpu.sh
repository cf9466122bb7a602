#!/bin/bash
mkdir -p gpurun_out
CASES=";OPT_CHUNK=64;OPT_CHUNK=128;OPT_WORKERS=1;OPT_WORKERS=2;OPT_SEGMENTS=8;OPT_SEGMENTS=32;OPT_LANES=8;OPT_CHUNK=64,OPT_SEGMENTS=16" timeout 900 python scripts/ragged_sweep.py > gpurun_out/ragged_sweep.jsonl 2>&1
LMIN=500 LMAX=2000 CASES=";OPT_CHUNK=64" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_sweep.jsonl 2>&1
LMIN=2000 LMAX=8000 CASES=";OPT_CHUNK=128" timeout 300 python scripts/ragged_sweep.py >> gpurun_out/ragged_sweep.jsonl 2>&1
CASES="512:2000:10000000:OPT_SCHED=3;512:2000:10000000:" timeout 300 python scripts/spec_sweep.py >> gpurun_out/ragged_sweep.jsonl 2>&1
cat gpurun_out/ragged_sweep.jsonl
