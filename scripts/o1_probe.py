"""Probe of the -Xptxas -O1 build: the same small batch several times and per schedule;
reports mismatches against the oracle and run-to-run differences."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference
Y = oracle.znorm(nanopore_reference(100_000, 4)[None])[0]
Q = oracle.znorm(nanopore_queries(64, 500, 100_000, 4))
ref = oracle.sdtw(Q, Y)
sd.set_reference(torch.as_tensor(Y, device="cuda"))
Qt = torch.as_tensor(Q, device="cuda")
for opts in [dict(OPT_SCHED=1), dict(OPT_SCHED=2), dict(OPT_SCHED=3), dict(OPT_SCHED=1, OPT_LANES=1),
             dict(OPT_SCHED=1, OPT_PACKED=0), dict(OPT_SCHED=1, OPT_LANES=2, OPT_CHUNK=16)]:
    outs = []
    for rep in range(3):
        with sd.options(OPT_NORMALIZE=0, **opts):
            c, e = sd.batch(Qt)
        outs.append(c.cpu().numpy())
    bad = [int(np.sum(o != ref["cost"])) for o in outs]
    lower = [int(np.sum(o < ref["cost"])) for o in outs]
    same = all(np.array_equal(outs[0], o) for o in outs)
    print(opts, "mismatches per rep", bad, "lower", lower, "reps identical", same, flush=True)
