"""Run small configurations one by one (each in a subprocess with a timeout)."""
import json, os, subprocess, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import sys, time, numpy as np, torch
sys.path.insert(0, %r)
import paper_2403_06931_b200 as sd, oracle
opts = %s
Z, N, M, trace = %d, %d, %d, %d
rng = np.random.default_rng(1)
Q = rng.standard_normal((Z, N)).astype(np.float32); Y = rng.standard_normal(M).astype(np.float32)
dev = torch.device("cuda", 0)
t0 = time.time()
with sd.options(OPT_NORMALIZE=0, **opts):
    sd.set_reference(torch.as_tensor(Y, device=dev))
    print("ref ok", time.time() - t0, flush=True)
    out = (sd.traceback if trace else sd.batch)(torch.as_tensor(Q, device=dev))
    torch.cuda.synchronize()
print("gpu ok", time.time() - t0, flush=True)
ref = oracle.sdtw(Q, Y, start=bool(trace))
c = out[0].cpu().numpy(); e = out[1].cpu().numpy()
print("EXACT" if np.array_equal(c, ref["cost"]) and np.array_equal(e, ref["end"]) else "MISMATCH", c[:3], ref["cost"][:3], e[:3], ref["end"][:3], flush=True)
'''
cases = [
    (dict(OPT_PACKED=0, OPT_SEGMENT_W=8, OPT_LANES=1), 1, 64, 300, 0),
    (dict(OPT_PACKED=0, OPT_SEGMENT_W=8, OPT_LANES=1), 2, 64, 5000, 0),
    (dict(OPT_PACKED=0, OPT_SEGMENT_W=16, OPT_LANES=2), 2, 300, 5000, 0),
    (dict(OPT_PACKED=1, OPT_SEGMENT_W=16, OPT_LANES=1), 2, 300, 5000, 0),
    (dict(OPT_PACKED=1, OPT_SEGMENT_W=32, OPT_LANES=4), 2, 300, 20000, 0),
    (dict(OPT_PACKED=1, OPT_SEGMENT_W=32, OPT_LANES=2, OPT_CLUSTER=2), 2, 300, 20000, 0),
    (dict(), 8, 300, 20000, 1),
]
for opts, Z, N, M, tr in cases:
    src = CHILD % (ROOT, repr(opts), Z, N, M, tr)
    t = time.time()
    try:
        r = subprocess.run([sys.executable, "-c", src], capture_output=True, text=True, timeout=int(os.environ.get("CASE_TIMEOUT", "60")))
        print(opts, Z, N, M, tr, "rc", r.returncode, "%.1fs" % (time.time() - t), r.stdout.strip().replace("\n", " | "), r.stderr.strip()[-400:], flush=True)
    except subprocess.TimeoutExpired as ex:
        print(opts, Z, N, M, tr, "TIMEOUT", (ex.stdout or b"")[-300:], flush=True)
