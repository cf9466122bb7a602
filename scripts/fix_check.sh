#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH c3', d['value'])"
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -2
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/fix_bdptrace.so paper_2403_06931_b200/libsdtw.so
echo "== fix_bdptrace"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1
cp variants/fix_clspec2.so paper_2403_06931_b200/libsdtw.so
echo "== fix_clspec2"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1
cp variants/fix_o1.so paper_2403_06931_b200/libsdtw.so
echo "== fix_o1"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
