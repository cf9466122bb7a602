"""Small-batch schedules on one GPU: TCUPS of sd.batch (device inputs, CUDA events, best of
REPS) for the sequential and the speculative schedules, and how many queries the
speculative run recomputed.  CASES env: "Z:N:M:opt=v,opt=v;..." """
import json, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

dev = torch.device("cuda", 0)
REPS = int(os.environ.get("REPS", 3))
cases = os.environ.get("CASES", "64:2000:10000000:OPT_SCHED=1;64:2000:10000000:OPT_SCHED=3")
refs = {}
for case in cases.split(";"):
    f = case.split(":")
    Z, N, M = int(f[0]), int(f[1]), int(f[2])
    opts = dict(kv.split("=") for kv in f[3].split(",") if kv) if len(f) > 3 else {}
    opts = {k: int(v) for k, v in opts.items()}
    if M not in refs:
        refs[M] = torch.from_numpy(nanopore_reference(M, 3)).to(dev)
    Q = torch.from_numpy(nanopore_queries(Z, N, M, 3)).to(dev)
    with sd.options(**opts):
        sd.set_reference(refs[M])
        run = sd.traceback if os.environ.get("TRACE") else sd.batch
        run(Q)
        best = 1e30
        for _ in range(REPS):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            c, e = run(Q)[:2]
            b.record()
            torch.cuda.synchronize()
            best = min(best, a.elapsed_time(b))
        fixed = sd.spec_recomputed()
    print(json.dumps({"Z": Z, "N": N, "M": M, "opts": opts, "ms": round(best, 3),
                      "tcups": round(Z * N * M / best / 1e9, 3), "recomputed": fixed,
                      "cost0": float(c[0]), "end0": int(e[0])}), flush=True)
