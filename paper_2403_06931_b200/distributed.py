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


# --------------------------------------------------------------------------------------
# Reference split: for batches too small to fill
# P GPUs by query sharding, rank r takes the reference slice [r*L, (r+1)*L) (L a multiple
# of the DP round width) and ALL queries.  Exactness follows the speculative segments of
# DESIGN.md §13 with one segment per rank: the free DP of each slice (start anywhere in
# it, +inf boundary) runs everywhere at once; one all-gather moves every rank's last DP
# column (Z x N fp32) to its successor, which runs a short correction DP from it (no free
# start) over the first check_cols columns of its slice; where that correction is
# overtaken by the free DP on every row the result is lexmin(free, correction); queries
# with a correction not overtaken are recomputed exactly by a rank-ordered chain of full
# boundary DPs (point-to-point column hand-offs).  The ops object supplies the DP calls
# (the CUDA library on GPUs; a plain DP in the CPU tests).


class CudaSplitOps:
    """The DP calls of the reference split on the CUDA library (current device)."""

    def __init__(self, sd):
        self.sd = sd

    def round_columns(self, N: int) -> int:
        return self.sd.round_columns(N)

    def set_reference(self, Yslice):
        with self.sd.options(OPT_NORMALIZE=0):              # the slice is globally normalised
            self.sd.set_reference(Yslice)

    def batch_columns(self, Q, last: bool):
        with self.sd.options(OPT_NORMALIZE=0):
            return self.sd.batch_columns(Q, last=last)

    def boundary_dp(self, Q, boundary, free_start: bool, n_cols: int):
        with self.sd.options(OPT_NORMALIZE=0):
            return self.sd.boundary_dp(Q, boundary, free_start=free_start, n_cols=n_cols)

    def normalize(self, Q, Y):
        """Per-query and whole-reference z-normalisation on the GPU (sdtw_znormalize):
        the slices must share the global statistics of the reference."""
        Yd = torch.as_tensor(np.asarray(Y, np.float32), device=Q.device)
        return self.sd.znormalize(Q), self.sd.znormalize(Yd).cpu().numpy()


def split_bounds(M: int, world: int, cols: int):
    """Slice [lo, hi) of every rank: equal multiples of the round width, the last takes the rest."""
    per = -(-(-(-M // world)) // cols) * cols
    return [(min(M, r * per), min(M, (r + 1) * per)) for r in range(world)]


def _lexmin(c1, e1, c2, e2):
    """Element-wise lexicographic min of (cost, end) pairs (numpy)."""
    take = (c2 < c1) | ((c2 == c1) & (e2 < e1))
    return np.where(take, c2, c1), np.where(take, e2, e1)


def _comm_device(group, dev):
    """gloo moves host tensors (CPU tests, or several ranks sharing one GPU); NCCL device ones."""
    if dist.is_initialized() and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return dev


def reference_split_batch(Q: torch.Tensor, Y, ops=None, group=None, normalize: bool = False):
    """Exact sDTW of all queries Q [Z, N] against the reference Y (length M), the reference
    split over the ranks of `group`.  Inputs are taken as already z-normalised unless
    `normalize` (then each query and the whole reference are normalised first, on the GPU).
    Returns (cost fp32 [Z], end int64 [Z]) as numpy on every rank, plus the number of
    queries that needed the exact fallback chain."""
    if ops is None:
        import paper_2403_06931_b200 as sd
        ops = CudaSplitOps(sd)
    if normalize:
        Q, Y = ops.normalize(Q, Y)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    Z, N = Q.shape
    Yn = np.asarray(Y.cpu() if isinstance(Y, torch.Tensor) else Y, np.float32)
    M = Yn.shape[0]
    cols = ops.round_columns(N)
    bounds = split_bounds(M, world, cols)
    lo, hi = bounds[rank]
    if any(b[1] <= b[0] for b in bounds):
        raise ValueError("reference too short for %d slices of %d-column rounds" % (world, cols))
    dev = Q.device
    cdev = _comm_device(group, dev)
    ops.set_reference(torch.as_tensor(Yn[lo:hi], device=dev) if dev.type == "cuda" else Yn[lo:hi])
    last = rank < world - 1
    cf, ef, col_check, col_last, check_cols = ops.batch_columns(Q, last)
    cf = np.asarray(cf.cpu() if isinstance(cf, torch.Tensor) else cf, np.float32)
    ef = np.asarray(ef.cpu() if isinstance(ef, torch.Tensor) else ef, np.int64) + lo
    # 1) every rank's last column -> its successor (one all-gather, Z x N fp32 per rank)
    mine = col_last if col_last is not None else torch.full((Z, N), float("inf"), device=dev)
    mine = torch.as_tensor(mine, dtype=torch.float32, device=cdev).reshape(Z, N)
    cols_all = _gather(mine.contiguous(), world, group).reshape(world, Z, N) if world > 1 else mine[None]
    cols_all = cols_all.to(dev)
    # 2) correction of this slice from the predecessor's last column
    cc = np.full(Z, np.inf, np.float32)
    ec = np.zeros(Z, np.int64)
    dom = np.ones(Z, bool)
    if rank > 0:
        c2, e2, colB = ops.boundary_dp(Q, cols_all[rank - 1], False, check_cols)
        cc = np.asarray(c2.cpu() if isinstance(c2, torch.Tensor) else c2, np.float32)
        ec = np.asarray(e2.cpu() if isinstance(e2, torch.Tensor) else e2, np.int64) + lo
        B = torch.as_tensor(colB, device=dev).reshape(Z, N)
        F = torch.as_tensor(col_check, device=dev).reshape(Z, N)
        dom = (B >= F).all(dim=1).cpu().numpy()
    # 3) per-query records of every rank (one all-gather)
    rec = torch.zeros((Z, 5), dtype=torch.int64)
    rec[:, 0] = torch.from_numpy(cf.view(np.int32).astype(np.int64))
    rec[:, 1] = torch.from_numpy(ef)
    rec[:, 2] = torch.from_numpy(cc.view(np.int32).astype(np.int64))
    rec[:, 3] = torch.from_numpy(ec)
    rec[:, 4] = torch.from_numpy(dom.astype(np.int64))
    recs = (_gather(rec.to(cdev), world, group).reshape(world, Z, 5) if world > 1 else rec[None]).cpu().numpy()
    cost = recs[0, :, 0].astype(np.int32).view(np.float32).copy()
    end = recs[0, :, 1].copy()
    bad = np.zeros(Z, bool)
    for r in range(1, world):
        cost, end = _lexmin(cost, end, recs[r, :, 0].astype(np.int32).view(np.float32), recs[r, :, 1])
        ok = recs[r, :, 4] != 0
        cr = np.where(ok, recs[r, :, 2].astype(np.int32).view(np.float32), np.inf).astype(np.float32)
        cost, end = _lexmin(cost, end, cr, np.where(ok, recs[r, :, 3], 0))
        bad |= ~ok
    idx = np.nonzero(bad)[0]
    if idx.size:
        # 4) exact fallback for those queries: rank-ordered chain of full boundary DPs
        Qf = Q[torch.as_tensor(idx, device=dev)].contiguous()
        F_ = len(idx)
        if rank == 0:
            tin = None
            cfl, efl = cf[idx], ef[idx]
            tout = torch.as_tensor(col_last, device=dev).reshape(Z, N)[torch.as_tensor(idx, device=dev)]
        else:
            tin = torch.empty((F_, N), dtype=torch.float32, device=cdev)
            dist.recv(tin, src=_global(group, rank - 1), group=group)
            c3, e3, tout = ops.boundary_dp(Qf, tin.to(dev), True, 0)
            cfl = np.asarray(c3.cpu() if isinstance(c3, torch.Tensor) else c3, np.float32)
            efl = np.asarray(e3.cpu() if isinstance(e3, torch.Tensor) else e3, np.int64) + lo
        if rank < world - 1:
            dist.send(torch.as_tensor(tout, dtype=torch.float32, device=cdev).reshape(F_, N).contiguous(),
                      dst=_global(group, rank + 1), group=group)
        rf = torch.zeros((F_, 2), dtype=torch.int64)
        rf[:, 0] = torch.from_numpy(np.asarray(cfl, np.float32).view(np.int32).astype(np.int64))
        rf[:, 1] = torch.from_numpy(np.asarray(efl, np.int64))
        rfs = _gather(rf.to(cdev), world, group).reshape(world, F_, 2).cpu().numpy()
        c_, e_ = rfs[0, :, 0].astype(np.int32).view(np.float32), rfs[0, :, 1]
        for r in range(1, world):
            c_, e_ = _lexmin(c_, e_, rfs[r, :, 0].astype(np.int32).view(np.float32), rfs[r, :, 1])
        cost[idx], end[idx] = c_, e_
    end = np.where(np.isinf(cost), 0, end)
    return cost.astype(np.float32), end.astype(np.int64), int(idx.size)


def _global(group, r: int) -> int:
    return dist.get_global_rank(group, r) if group is not None else r
