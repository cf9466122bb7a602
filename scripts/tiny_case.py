import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_2403_06931_b200 as sd, oracle
Z, N, M, trace = [int(a) for a in sys.argv[1:5]]
opts = eval(sys.argv[5]) if len(sys.argv) > 5 else {}
rng = np.random.default_rng(1)
Q = rng.standard_normal((Z, N)).astype(np.float32); Y = rng.standard_normal(M).astype(np.float32)
dev = torch.device("cuda", 0)
with sd.options(OPT_NORMALIZE=0, **opts):
    sd.set_reference(torch.as_tensor(Y, device=dev))
    out = (sd.traceback if trace else sd.batch)(torch.as_tensor(Q, device=dev))
ref = oracle.sdtw(Q, Y, start=bool(trace))
c = out[0].cpu().numpy(); e = out[1].cpu().numpy()
print(sys.argv[1:], "EXACT" if np.array_equal(c, ref["cost"]) and np.array_equal(e, ref["end"]) else "MISMATCH", c[:3], ref["cost"][:3], e[:3], ref["end"][:3], flush=True)
