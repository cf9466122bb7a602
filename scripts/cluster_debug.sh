#!/bin/bash
mkdir -p gpurun_out
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/clspec.so paper_2403_06931_b200/libsdtw.so
{
python scripts/cluster_case.py
W=30 L=1 CL=4 python scripts/cluster_case.py
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in initcheck racecheck synccheck memcheck; do
  echo "== $tool"; timeout 600 $CS --tool $tool --print-limit 10 python scripts/cluster_case.py 2>&1 | tail -25
done
} > gpurun_out/cluster_debug.log 2>&1
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
python scripts/cluster_case.py >> gpurun_out/cluster_debug.log 2>&1
cat gpurun_out/cluster_debug.log | cut -c1-300
