#!/bin/bash
mkdir -p gpurun_out
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/clspec2.so paper_2403_06931_b200/libsdtw.so
{ echo "== variant2, pytest config1"; timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "test_config1_bit_exact_all_schedules" --tb=no -rf 2>&1 | tail -9
  echo "== variant2, cluster only"; HIST=6,7 python scripts/cluster_hist.py
  echo "== variant2, full history"; python scripts/cluster_hist.py
  CS=/usr/local/cuda/bin/compute-sanitizer
  for tool in memcheck synccheck initcheck; do echo "== $tool"; HIST=6 timeout 600 $CS --tool $tool --print-limit 10 python scripts/cluster_hist.py 2>&1 | tail -12; done
} > gpurun_out/cluster_debug3.log 2>&1
cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
cat gpurun_out/cluster_debug3.log | cut -c1-250
