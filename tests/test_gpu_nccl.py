"""The multi-GPU code path over NCCL on the one GPU available (world size 1): process-group
init, sharding, the record and path all-gathers and unpacking run for real on NCCL; results
must equal the single-call results bit for bit.  (World sizes >= 2 are covered on CPU by
tests/test_distributed_gloo.py; the round-end box has one GPU.)"""
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
Y = nanopore_reference(50_000, 3)
Q = torch.as_tensor(nanopore_queries(40, 400, 50_000, 3), device=dev)
sd.set_reference(torch.as_tensor(Y, device=dev))
c, e, s = distributed_batch(Q, traceback=True, device=dev)
c0, e0, s0 = sd.traceback(Q)
assert np.array_equal(c, c0.cpu().numpy()) and np.array_equal(e, e0.cpu().numpy()) and np.array_equal(s, s0.cpu().numpy())
c, e, s, lo, hi = distributed_batch(Q[:6], path=True, device=dev)
r = sd.path(Q[:6])
assert np.array_equal(lo, r[3].cpu().numpy()) and np.array_equal(hi, r[4].cpu().numpy())
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
