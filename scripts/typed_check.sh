#!/bin/bash
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/typed.so paper_2403_06931_b200/libsdtw.so
timeout 600 python bench.py --steps 3 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('BENCH typed c3', d['value'])"
echo "== typed"; timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_spec.py -q --tb=no 2>&1 | tail -1
for v in typed_o1 typed_bdp; do
  cp variants/$v.so paper_2403_06931_b200/libsdtw.so
  echo "== $v"; timeout 600 python -m pytest tests/test_gpu_parity.py -q --tb=no 2>&1 | tail -1
done
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
