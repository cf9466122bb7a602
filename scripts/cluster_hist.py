"""Config-1 schedules in sequence (as tests/test_gpu_parity.py runs them), reporting which
cluster runs go wrong; HIST env selects the schedules run before the cluster one."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import oracle
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference
from test_gpu_parity import SCHEDULES

Y = oracle.znorm(nanopore_reference(4096, 1)[None])[0]
Q = oracle.znorm(nanopore_queries(8, 64, 4096, 1))
ref = oracle.sdtw(Q, Y)
dev = torch.device("cuda", 0)
Yt, Qt = torch.as_tensor(Y, device=dev), torch.as_tensor(Q, device=dev)
order = [int(x) for x in os.environ.get("HIST", "0,1,2,3,4,5,6,7,8,10").split(",")]
for k in order:
    for fma in (1, 0):
        with sd.options(OPT_NORMALIZE=0, OPT_FMA=fma, **SCHEDULES[k]):
            sd.set_reference(Yt)
            c, e = sd.batch(Qt)
            sd.traceback(Qt)
        r = oracle.sdtw(Q, Y, fma=bool(fma))
        bad = np.nonzero(c.cpu().numpy() != r["cost"])[0].tolist()
        print(k, fma, SCHEDULES[k], "bad", bad, flush=True)
