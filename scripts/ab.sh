#!/bin/bash
# A/B of library variants on one GPU box: sweep (CONFIGS env) with the in-tree lib and
# with each variants/<name>.so, then GPU tests (+ optional ncu) on the in-tree lib.
# Usage: scripts/ab.sh TAG [variant names...]   (env: NOTEST=1, PROF=1)
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
LIB=paper_2403_06931_b200/libsdtw.so
cp $LIB variants/_main.so
timeout 400 python scripts/sweep.py > gpurun_out/${TAG}_main.jsonl 2>&1
for v in "$@"; do
  cp variants/$v.so $LIB
  timeout 400 python scripts/sweep.py > gpurun_out/${TAG}_$v.jsonl 2>&1
done
cp variants/_main.so $LIB
[ -z "$NOTEST" ] && timeout 900 python -m pytest tests -m gpu -x -q --timeout 400 > gpurun_out/${TAG}_pytest.log 2>&1
[ -n "$PROF" ] && timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 1 -c 1 \
     -o gpurun_out/${TAG}_dp python scripts/prof_one.py > gpurun_out/${TAG}_ncu.log 2>&1
for f in gpurun_out/${TAG}_*.jsonl; do echo "== $f"; cat $f; done
tail -2 gpurun_out/${TAG}_pytest.log 2>/dev/null
