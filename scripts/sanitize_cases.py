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
# round 2: uint8 codebook (radix-select codebook, quantiser, integer DP with / without pruning),
# checkpointed start index (the traceback default) and its forced form, the reference-split calls
for tau in (-1, 40):
    with sd.options(OPT_Q8_PRUNE=tau, OPT_SCHED=3, OPT_LANES=1):
        sd.batch_q8(Qt)
    with sd.options(OPT_Q8_PRUNE=tau):
        sd.batch_q8(Qt)
sd.quantize(Qt)
with sd.options(OPT_START=2):
    sd.traceback(Qt)
    sd.path(Qt[:2])
with sd.options(OPT_LANES=1):
    c, e, ck, cl, n = sd.batch_columns(Qt, last=False)
    sd.boundary_dp(Qt, ck, False, n)
    sd.columns_dominate(ck, ck)
torch.cuda.synchronize()
print("sanitize cases done")
