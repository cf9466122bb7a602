"""Small workloads for compute-sanitizer (scripts/sanitize.sh): every kernel family once."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

dev = torch.device("cuda", 0)
Y = nanopore_reference(20_000, 1)
Q = nanopore_queries(8, 300, 20_000, 1)
sd.set_reference(torch.as_tensor(Y, device=dev))
Qt = torch.as_tensor(Q, device=dev)
runs = [dict(), dict(OPT_PACKED=0, OPT_SEGMENT_W=15, OPT_LANES=2), dict(OPT_PACKED=2, OPT_SEGMENT_W=28),
        dict(OPT_CLUSTER=2, OPT_LANES=2), dict(OPT_SCHED=2, OPT_SEGMENTS=3), dict(OPT_PACKED=3),
        dict(OPT_SCHED=3, OPT_LANES=1), dict(OPT_SCHED=3, OPT_LANES=1, OPT_SPEC_ROUNDS=1, OPT_SEGMENTS=8)]
for cfg in runs:
    with sd.options(**cfg):
        sd.batch(Qt)
        sd.traceback(Qt)
sd.path(Qt[:4])
off = np.array([0, 100, 350, 360, 900], np.int64)
sd.batch_ragged(Qt.reshape(-1)[:900], off, start=True)
with sd.options(OPT_SCHED=3, OPT_LANES=1):
    sd.batch_ragged(Qt.reshape(-1)[:900], off, start=True)
with sd.options(OPT_PRECISION=16, OPT_SCHED=3, OPT_LANES=1):
    sd.batch(Qt)
torch.cuda.synchronize()
print("sanitize cases done")
