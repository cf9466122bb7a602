import sys, torch; sys.path.insert(0, ".")
import paper_2403_06931_b200 as sd
from datagen import nanopore_queries, nanopore_reference
dev = torch.device("cuda", 0)
Y = torch.from_numpy(nanopore_reference(200000, 2)).to(dev); Q = torch.from_numpy(nanopore_queries(512, 2000, 200000, 2)).to(dev)
pk, w, gw = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
with sd.options(OPT_PACKED=pk, OPT_SEGMENT_W=w, OPT_LANES=gw):
    sd.set_reference(Y)
    for _ in range(3): sd.batch(Q)
torch.cuda.synchronize()
