#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/cur_o1.so paper_2403_06931_b200/libsdtw.so
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do echo "== $tool"; timeout 600 $CS --tool $tool --print-limit 5 python scripts/o1_probe.py 2>&1 | grep -v "^{" | tail -12; done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
