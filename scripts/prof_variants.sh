#!/bin/bash
# ncu --set full of the DP kernel for two schedules on the c2 workload.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for v in "c2:1:30:4" "c4:2:28:4"; do
  IFS=: read name pk w gw <<< "$v"
  cat > /tmp/one.py <<PY
import sys, torch; sys.path.insert(0, ".")
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference
dev = torch.device("cuda", 0)
Y = torch.from_numpy(nanopore_reference(100000, 2)).to(dev); Q = torch.from_numpy(nanopore_queries(512, 2000, 100000, 2)).to(dev)
with sd.options(OPT_PACKED=$pk, OPT_SEGMENT_W=$w, OPT_LANES=$gw):
    sd.set_reference(Y)
    for _ in range(3): sd.batch(Q)
torch.cuda.synchronize()
PY
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sdtw_dp -s 2 -c 1 -o gpurun_out/pv_$name python /tmp/one.py > gpurun_out/pv_$name.log 2>&1
done
echo done
