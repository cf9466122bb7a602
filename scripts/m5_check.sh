#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/m5.so paper_2403_06931_b200/libsdtw.so
timeout 600 python bench.py --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH m5', d['value'])"
cp variants/m5_o1.so paper_2403_06931_b200/libsdtw.so
echo "== m5_o1"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
