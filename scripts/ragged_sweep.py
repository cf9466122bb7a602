"""Ragged-batch schedules on one GPU (c6-like: reads log-uniform in [LMIN, LMAX] vs an
M-sample reference): TCUPS of sd.batch_ragged with device inputs, best of REPS.
CASES env: "opt=v,opt=v;..." (empty = defaults)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_ragged, nanopore_reference

dev = torch.device("cuda", 0)
Z = int(os.environ.get("Z", 512)); M = int(os.environ.get("M", 1_000_000))
LMIN = int(os.environ.get("LMIN", 500)); LMAX = int(os.environ.get("LMAX", 8000))
REPS = int(os.environ.get("REPS", 3))
Q, off = nanopore_ragged(Z, M, 6, LMIN, LMAX)
Qt = torch.from_numpy(Q).to(dev); offt = torch.from_numpy(off).to(dev)
sd.set_reference(torch.from_numpy(nanopore_reference(M, 6)).to(dev))
cells = float(off[-1]) * M
for case in os.environ.get("CASES", "").split(";"):
    opts = {k: int(v) for k, v in (kv.split("=") for kv in case.split(",") if kv)}
    with sd.options(**opts):
        sd.batch_ragged(Qt, offt)
        best = 1e30
        for _ in range(REPS):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(); a.record()
            c, e = sd.batch_ragged(Qt, offt)
            b.record(); torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
    print(json.dumps({"Z": Z, "M": M, "lens": [LMIN, LMAX], "opts": opts, "ms": round(best, 3),
                      "tcups": round(cells / best / 1e9, 3), "cost0": float(c[0])}), flush=True)
