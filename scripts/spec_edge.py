"""Edge shapes of the speculative schedule vs sequential segments (bit-identical results)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

dev = torch.device("cuda", 0)
for Z, N, M, trace in [(1, 2000, 10_000_000, False), (1, 500, 2_000_000, True), (2048, 300, 1_000_000, False),
                       (3, 8000, 3_000_000, False), (700, 64, 500_000, True)]:
    Y = torch.from_numpy(nanopore_reference(M, 5)).to(dev)
    Q = torch.from_numpy(nanopore_queries(Z, N, M, 5)).to(dev)
    sd.set_reference(Y)
    run = sd.traceback if trace else sd.batch
    with sd.options(OPT_SCHED=3):
        a = [t.cpu() for t in run(Q)]
        fixed = sd.spec_recomputed()
    with sd.options(OPT_SCHED=2):
        b = [t.cpu() for t in run(Q)]
    same = all(torch.equal(x, y) for x, y in zip(a, b))
    print(Z, N, M, trace, "identical" if same else "DIFFERENT", "recomputed", fixed, flush=True)
