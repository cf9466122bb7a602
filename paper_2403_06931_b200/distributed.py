"""Query-sharded multi-GPU sDTW (BASELINE.json north_star "Multi-GPU").

One process per GPU.  The reference is replicated (every rank calls
``set_reference``); queries are independent, so rank r takes the contiguous
shard [r*ceil(Z/P), min(Z, (r+1)*ceil(Z/P))), runs the CUDA path on it, and
the per-query records are exchanged with ONE all-gather (NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests).  The reference is never split:
a warp path may span any length of it.

Record layout (int64 x 3 per query): [fp32 cost bits, end, start-or--1]; with the full
warp path (sdtw_path) a second all-gather moves the per-row column ranges (int32 x 2 x N).
"""
from __future__ import annotations

from typing import Callable, Optional

import numpy as np
import torch
import torch.distributed as dist


def shard_bounds(Z: int, world: int, rank: int):
    """Contiguous shard of rank `rank`: (lo, hi, per_rank) with per_rank = ceil(Z/world)."""
    per = -(-Z // world) if world > 0 else 0
    lo = min(Z, rank * per)
    hi = min(Z, lo + per)
    return lo, hi, per


def _pack(cost, end, start, per: int, device) -> torch.Tensor:
    cost = torch.as_tensor(np.asarray(cost.cpu() if isinstance(cost, torch.Tensor) else cost, np.float32))
    end = torch.as_tensor(np.asarray(end.cpu() if isinstance(end, torch.Tensor) else end, np.int64))
    n = cost.shape[0]
    rec = torch.full((per, 3), -1, dtype=torch.int64)
    if n:
        rec[:n, 0] = cost.view(torch.int32).to(torch.int64)
        rec[:n, 1] = end
        if start is not None:
            st = torch.as_tensor(np.asarray(start.cpu() if isinstance(start, torch.Tensor) else start, np.int64))
            rec[:n, 2] = st
    return rec.to(device)


def _unpack(rec: torch.Tensor, Z: int, want_start: bool):
    rec = rec[:Z].cpu()
    cost = rec[:, 0].to(torch.int32).view(torch.float32).numpy().copy()
    end = rec[:, 1].numpy().copy()
    start = rec[:, 2].numpy().copy() if want_start else None
    return cost, end, start


def _gather(t: torch.Tensor, world: int, group):
    full = torch.empty((t.shape[0] * world, *t.shape[1:]), dtype=t.dtype, device=t.device)
    try:
        dist.all_gather_into_tensor(full, t, group=group)
    except (RuntimeError, NotImplementedError, AttributeError):
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t, group=group)
        full = torch.cat(parts, 0)
    return full


def distributed_batch(Q, group=None, traceback: bool = False,
                      fn: Optional[Callable] = None, device=None, pre_sharded: bool = False,
                      path: bool = False):
    """Shard Q [Z, N] over the ranks of `group`, compute locally, all-gather results.

    fn(Q_shard) -> (cost, end[, start[, path_lo, path_hi]]); default: this package's CUDA
    ``batch`` / ``traceback`` / ``path``.  With pre_sharded=True, Q is already this rank's
    shard and every rank holds the same number of queries (global Z = world *
    Q.shape[0]).  Returns numpy (cost[Z], end[Z], start[Z] | None) on every rank, plus
    (path_lo[Z, N], path_hi[Z, N]) int32 when path=True (a second all-gather)."""
    traceback = traceback or path
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    if pre_sharded:
        per = int(Q.shape[0])
        Z = per * world
        lo, hi = 0, per
    else:
        Z = int(Q.shape[0])
        lo, hi, per = shard_bounds(Z, world, rank)
    if fn is None:
        import paper_2403_06931_b200 as sd
        fn = sd.path if path else (sd.traceback if traceback else sd.batch)
    if device is None:
        device = Q.device if isinstance(Q, torch.Tensor) else torch.device("cpu")
    if dist.get_backend(group) == "nccl" and device.type != "cuda":
        device = torch.device("cuda", torch.cuda.current_device())
    N = int(Q.shape[1]) if len(Q.shape) > 1 else 1
    if hi > lo:
        out = fn(Q[lo:hi])
    else:
        out = (np.empty(0, np.float32), np.empty(0, np.int64), np.empty(0, np.int64),
               np.empty((0, N), np.int32), np.empty((0, N), np.int32))
    start = out[2] if traceback else None
    rec = _pack(out[0], out[1], start, per, device)
    res = _unpack(_gather(rec, world, group), Z, traceback)
    if not path:
        return res
    pth = torch.full((per, N, 2), -1, dtype=torch.int32)
    n = hi - lo
    if n:
        for k, a in ((0, out[3]), (1, out[4])):
            pth[:n, :, k] = torch.as_tensor(np.asarray(a.cpu() if isinstance(a, torch.Tensor) else a, np.int32))
    full = _gather(pth.to(device), world, group)[:Z].cpu().numpy()
    return res + (full[:, :, 0].copy(), full[:, :, 1].copy())
