"""Schedule sweep (the paper's segment-width experiment, re-run on B200):
GCUPS of the DP path for several (W, warps/CTA, cluster) settings; results must be
bit-identical across settings (checked)."""
import itertools, json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

TRACE = bool(int(os.environ.get("TRACE", "0")))
Z = int(os.environ.get("Z", 512)); N = int(os.environ.get("N", 2000)); M = int(os.environ.get("M", 1_000_000))
dev = torch.device("cuda", 0)
Y = torch.from_numpy(nanopore_reference(M, 3)).to(dev)
Q = torch.from_numpy(nanopore_queries(Z, N, M, 3)).to(dev)
sd.set_reference(Y)
configs = json.loads(os.environ.get("CONFIGS", "[]")) or [
    dict(OPT_PACKED=p, OPT_SEGMENT_W=w, OPT_LANES=g, OPT_CLUSTER=c)
    for (p, w) in [(1, 6), (1, 14), (1, 30), (1, 62), (0, 15), (0, 31)] for g in (2, 4, 8) for c in (1, 2)]
ref = None
for cfg in configs:
    try:
        with sd.options(**cfg):
            for _ in range(2):
                c, e = (sd.traceback(Q)[:2] if TRACE else sd.batch(Q))
            torch.cuda.synchronize()
            t = time.perf_counter()
            reps = 3
            for _ in range(reps):
                c, e = (sd.traceback(Q)[:2] if TRACE else sd.batch(Q))
            torch.cuda.synchronize()
            dt = (time.perf_counter() - t) / reps
        same = None
        if ref is None:
            ref = (c.clone(), e.clone())
        else:
            same = bool(torch.equal(c, ref[0]) and torch.equal(e, ref[1]))
        print(json.dumps(dict(cfg=cfg, ms=dt * 1e3, gcups=Z * N * M / dt / 1e9, identical=same,
                              recomputed=sd.spec_recomputed())), flush=True)
    except Exception as ex:
        print(json.dumps(dict(cfg=cfg, error=str(ex)[:200])), flush=True)
