#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
for v in o1_nomov; do
  cp variants/$v.so paper_2403_06931_b200/libsdtw.so
  echo "== $v"; timeout 600 python scripts/o1_probe.py 2>&1 | head -6
done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
