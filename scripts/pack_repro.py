"""Reproducer of the float-pair pack defect: BASELINE config 1 (8 x 64 vs
4,096, seed 1, raw normalised inputs) through the four-chain kernel (OPT_PACKED=2, W=28,
4 warps) -- the case that fails at ptxas -O3 with the inline-PTX pack -- printed against the
oracle.  Run with SDTW_LIB=variants/<build>.so (ptx_o3 / ptx_o1 / ptx_o0 / the default C++ pack)."""
import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference

Y = oracle.znorm(nanopore_reference(4096, 1)[None])[0]
Q = oracle.znorm(nanopore_queries(8, 64, 4096, 1))
ref = oracle.sdtw(Q, Y, fma=True, start=True)
bad = 0
for name, opts, trace in [("C=4 W=28 lanes=4 cost/end", dict(OPT_PACKED=2, OPT_SEGMENT_W=28, OPT_LANES=4), False),
                          ("C=4 W=28 lanes=4 forward start", dict(OPT_PACKED=2, OPT_SEGMENT_W=28, OPT_LANES=4,
                                                                  OPT_START=1), True),
                          ("C=2 W=30 (default)", dict(), False)]:
    with sd.options(OPT_NORMALIZE=0, **opts):
        sd.set_reference(torch.as_tensor(Y, device="cuda"))
        out = (sd.traceback if trace else sd.batch)(torch.as_tensor(Q, device="cuda"))
    c = out[0].cpu().numpy()
    wrong = np.nonzero(c.view(np.uint32) != ref["cost"].view(np.uint32))[0]
    bad += len(wrong)
    print("%-32s wrong costs: %s" % (name, ", ".join("q%d %.6g (oracle %.6g)" % (q, c[q], ref["cost"][q])
                                                      for q in wrong) or "none"))
print("library:", os.environ.get("SDTW_LIB", "in-tree"), sd.build_info(), "->", "FAIL" if bad else "OK")
