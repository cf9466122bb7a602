import numpy as np, torch, sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference
M = 200_000
Y = oracle.znorm(nanopore_reference(M, 71)[None])[0]
per = -(-(-(-M // 2)) // 960) * 960
Q = np.stack([Y[per - 200:per + 1300], oracle.znorm(nanopore_queries(1, 1500, M, 72))[0]]).astype(np.float32)
Qt = torch.as_tensor(Q, device="cuda")
with sd.options(OPT_NORMALIZE=0, OPT_LANES=1, OPT_SPEC_ROUNDS=1):
    print("round cols", sd.round_columns(1500))
    sd.set_reference(torch.as_tensor(Y[:per], device="cuda"))
    c0, e0, ck0, cl0, n0 = sd.batch_columns(Qt)
    print("rank0 free", c0, e0, "check", n0, "last col min/max/inf", cl0.min().item(), cl0.max().item(), torch.isinf(cl0).sum().item())
    sd.set_reference(torch.as_tensor(Y[per:], device="cuda"))
    c1, e1, ck1, cl1, n1 = sd.batch_columns(Qt, last=False)
    print("rank1 free", c1, e1, "check", n1, "ck min", ck1.min().item())
    c2, e2, B = sd.boundary_dp(Qt, cl0, free_start=False, n_cols=n1)
    print("corr", c2, e2, "B min/inf", B.min().item(), torch.isinf(B).sum().item(), "dom", (B >= ck1).all(dim=1))
    c3, e3, C3 = sd.boundary_dp(Qt, cl0, free_start=True, n_cols=0)
    print("full", c3, e3)
    c4, e4, _ = sd.boundary_dp(Qt, None, free_start=True, n_cols=0)
    print("full inf bnd", c4, e4)
