#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
for v in bdptrace bdptrace_o1 bdptrace_nofma; do
  cp variants/$v.so paper_2403_06931_b200/libsdtw.so
  echo "== $v"; timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "test_ragged_shapes_bit_exact" --tb=no 2>&1 | tail -1
done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
