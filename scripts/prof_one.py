"""One workload for ncu captures: Z x N queries vs an M-sample reference, default
schedule (override with OPT_* env vars), 2 launches (the second one is profiled)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

Z = int(os.environ.get("Z", 512)); N = int(os.environ.get("N", 2000)); M = int(os.environ.get("M", 1_000_000))
dev = torch.device("cuda", 0)
Y = torch.from_numpy(nanopore_reference(M, 3)).to(dev)
Q = torch.from_numpy(nanopore_queries(Z, N, M, 3)).to(dev)
opts = {k: int(v) for k, v in os.environ.items() if k.startswith("OPT_")}
with sd.options(**opts):
    sd.set_reference(Y)
    for _ in range(int(os.environ.get("REPS", 2))):
        sd.traceback(Q) if os.environ.get("TRACE") else sd.batch(Q)
torch.cuda.synchronize()
print("done", opts)
