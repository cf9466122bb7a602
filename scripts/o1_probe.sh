#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/cur_o1.so paper_2403_06931_b200/libsdtw.so
timeout 600 python scripts/o1_probe.py 2>&1 | tail -8
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
