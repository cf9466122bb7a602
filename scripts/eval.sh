#!/bin/bash
# One GPU-box evaluation of the current build: sweep (CONFIGS env), GPU parity tests,
# one ncu --set full capture of the DP kernel on prof_one.py.  Usage: scripts/eval.sh TAG [notest] [noprof]
cd "$(dirname "$0")/.."
TAG=${1:-x}
mkdir -p gpurun_out
timeout 400 python scripts/sweep.py > gpurun_out/${TAG}_sweep.jsonl 2>&1
if [[ "$*" != *notest* ]]; then
  timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/${TAG}_pytest.log 2>&1
fi
if [[ "$*" != *noprof* ]]; then
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 1 -c 1 \
     -o gpurun_out/${TAG}_dp python scripts/prof_one.py > gpurun_out/${TAG}_ncu.log 2>&1
fi
cat gpurun_out/${TAG}_sweep.jsonl; tail -2 gpurun_out/${TAG}_pytest.log 2>/dev/null; tail -1 gpurun_out/${TAG}_ncu.log 2>/dev/null
