"""Config-1 inputs on a two-chain cluster schedule (debugging aid for compute-sanitizer)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

Y = oracle.znorm(nanopore_reference(4096, 1)[None])[0]
Q = oracle.znorm(nanopore_queries(8, 64, 4096, 1))
ref = oracle.sdtw(Q, Y)
dev = torch.device("cuda", 0)
cfg = dict(OPT_NORMALIZE=0, OPT_PACKED=1, OPT_SEGMENT_W=int(os.environ.get("W", 14)),
           OPT_LANES=int(os.environ.get("L", 2)), OPT_CLUSTER=int(os.environ.get("CL", 2)))
with sd.options(**cfg):
    sd.set_reference(torch.as_tensor(Y, device=dev))
    c, e = sd.batch(torch.as_tensor(Q, device=dev))
c = c.cpu().numpy()
print(cfg, "bad queries:", np.nonzero(c != ref["cost"])[0].tolist(), "got", c[:6], "want", ref["cost"][:6])
