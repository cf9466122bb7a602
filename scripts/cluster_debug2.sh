#!/bin/bash
mkdir -p gpurun_out
cp paper_2403_06931_b200/libsdtw.so /tmp/cur.so
cp variants/clspec.so paper_2403_06931_b200/libsdtw.so
{ echo "== variant, full history"; python scripts/cluster_hist.py
  echo "== variant, cluster only"; HIST=6,7 python scripts/cluster_hist.py
  echo "== variant, 1 then cluster"; HIST=1,6 python scripts/cluster_hist.py
  echo "== variant, 4 then cluster"; HIST=4,6 python scripts/cluster_hist.py
  echo "== variant, 0 then cluster"; HIST=0,6 python scripts/cluster_hist.py
  cp /tmp/cur.so paper_2403_06931_b200/libsdtw.so
  echo "== current, full history"; python scripts/cluster_hist.py
} > gpurun_out/cluster_debug2.log 2>&1
cat gpurun_out/cluster_debug2.log | cut -c1-200
