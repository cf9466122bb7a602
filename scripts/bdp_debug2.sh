#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -3
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/bdptrace.so paper_2403_06931_b200/libsdtw.so
echo "== bdptrace (with early-clobber fix)"; timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "test_ragged_shapes_bit_exact" --tb=short 2>&1 | grep "AssertionError\|passed\|failed" | cut -c1-250 | tail -5
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
