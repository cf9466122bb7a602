#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
for v in cur_o1 bdptrace_o1; do
  cp variants/$v.so paper_2403_06931_b200/libsdtw.so
  echo "== $v"; timeout 900 python -m pytest tests/test_gpu_parity.py -q --tb=no -rf 2>&1 | grep "FAILED\|passed\|failed" | cut -c1-120 | tail -12
done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
