"""The query-sharded multi-GPU path on the one GPU available.

* NCCL at world size 1: process-group init, sharding, the record and path all-gathers and
  unpacking run for real on NCCL; results are compared with the ORACLE (raw mode, cost bit
  for bit, end exact or tied, start exact), not with the library's own single call.
* 2 and 3 ranks sharing the GPU (gloo moves the records; NCCL refuses two ranks on one
  device): every rank runs the CUDA library on its shard -- including Z not divisible by
  the world size and an empty last shard -- and every rank's gathered result must equal the
  oracle on the whole batch.  (tests/test_distributed_gloo.py covers world sizes 2-4 on CPU
  with an injected DP.)"""
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r'''
import os, sys, numpy as np, torch, torch.distributed as dist
sys.path.insert(0, %(root)r)
import paper_2403_06931_b200 as sd
from paper_2403_06931_b200.distributed import distributed_batch
from datagen import nanopore_queries, nanopore_reference
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
dist.init_process_group("nccl", init_method="tcp://127.0.0.1:%(port)d", rank=0, world_size=1, device_id=dev)
import oracle
Yn = oracle.znorm(nanopore_reference(50_000, 3)[None])[0]
Qn = oracle.znorm(nanopore_queries(40, 400, 50_000, 3))
ref = oracle.sdtw(Qn, Yn, fma=True, start=True)
Q = torch.as_tensor(Qn, device=dev)
with sd.options(OPT_NORMALIZE=0):
    sd.set_reference(torch.as_tensor(Yn, device=dev))
    c, e, s = distributed_batch(Q, traceback=True, device=dev)
    assert c.device.type == "cuda"          # records stay on the NCCL device
    c, e, s = c.cpu().numpy(), e.cpu().numpy(), s.cpu().numpy()
    assert np.array_equal(c.view(np.uint32), ref["cost"].view(np.uint32)), (c, ref["cost"])
    assert np.array_equal(e, ref["end"]) and np.array_equal(s, ref["start"])
    c, e, s, lo, hi = distributed_batch(Q[:6], path=True, device=dev)
    lo, hi = lo.cpu().numpy(), hi.cpu().numpy()
    for q in range(6):
        rc, re_, rs, rlo, rhi = oracle.sdtw_path(Qn[q], Yn, fma=True)
        assert rc == c[q].item() and re_ == e[q].item() and rs == s[q].item()
        assert np.array_equal(lo[q], rlo) and np.array_equal(hi[q], rhi), q
dist.destroy_process_group()
print("nccl world-1 OK")
'''


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_distributed_batch_over_nccl_world1():
    code = SCRIPT % dict(root=ROOT, port=_free_port())
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "nccl world-1 OK" in r.stdout


def _shared_worker(rank, world, port, Z, out_q):
    import numpy as np
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        sys.path.insert(0, ROOT)
        import oracle
        import paper_2403_06931_b200 as sd
        from paper_2403_06931_b200.distributed import distributed_batch
        from datagen import nanopore_queries, nanopore_reference
        Yn = oracle.znorm(nanopore_reference(30_000, 9)[None])[0]
        Qn = oracle.znorm(nanopore_queries(Z, 350, 30_000, 9))
        with sd.options(OPT_NORMALIZE=0):
            sd.set_reference(torch.as_tensor(Yn, device="cuda"))
            c, e, s = distributed_batch(torch.as_tensor(Qn, device="cuda"), traceback=True)
        out_q.put((rank, np.asarray(c), np.asarray(e), np.asarray(s)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,Z", [(2, 7), (3, 7), (3, 4)])
def test_query_shards_share_gpu_vs_oracle(world, Z):
    """Z=7 over 2 or 3 ranks: uneven shards; Z=4 over 3 ranks: shard sizes 2, 2, 0."""
    import numpy as np
    import torch.multiprocessing as mp
    import oracle
    from datagen import nanopore_queries, nanopore_reference
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shared_worker, args=(r, world, port, Z, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=300))
        except Exception:
            break
    for p in procs:
        p.join(timeout=30)
        if p.exitcode is None:
            p.kill()
    assert len(res) == world and all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    Yn = oracle.znorm(nanopore_reference(30_000, 9)[None])[0]
    Qn = oracle.znorm(nanopore_queries(Z, 350, 30_000, 9))
    ref = oracle.sdtw(Qn, Yn, fma=True, start=True)
    for rank, c, e, s in res:
        assert np.array_equal(c.view(np.uint32), ref["cost"].view(np.uint32)), (rank, c, ref["cost"])
        assert np.array_equal(e, ref["end"]) and np.array_equal(s, ref["start"]), rank
