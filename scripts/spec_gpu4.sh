#!/bin/bash
mkdir -p gpurun_out
C=""
for S in 5 6 8 10 12; do C="$C;512:2000:10000000:OPT_SCHED=3,OPT_SEGMENTS=$S"; done
for S in 40 65 90; do C="$C;64:2000:10000000:OPT_SCHED=3,OPT_SEGMENTS=$S"; done
for S in 10 16 24; do C="$C;200:2000:10000000:OPT_SCHED=3,OPT_SEGMENTS=$S"; done
C="$C;512:2000:10000000:OPT_SCHED=3,OPT_SEGMENTS=8,OPT_WORKERS=3;512:2000:1000000:;512:2000:1000000:OPT_SCHED=3;512:2000:1000000:OPT_SCHED=3,OPT_SEGMENTS=2"
CASES="${C#;}" timeout 1200 python scripts/spec_sweep.py > gpurun_out/spec_segs.jsonl 2>&1
cat gpurun_out/spec_segs.jsonl | cut -c1-200
