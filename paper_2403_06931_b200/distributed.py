"""Query-sharded multi-GPU sDTW (BASELINE.json north_star "Multi-GPU").

One process per GPU.  The reference is replicated (every rank calls
``set_reference``); queries are independent, so rank r takes the contiguous
shard [r*ceil(Z/P), min(Z, (r+1)*ceil(Z/P))), runs the CUDA path on it, and
the per-query records are exchanged with ONE all-gather (NCCL over
NVLink/NVSwitch on GPUs, gloo in the CPU tests).  The reference is never split:
a warp path may span any length of it.

Records stay on the communication device: they are packed with tensor views on the GPU
(no host round trip), gathered, and returned as torch tensors on that device.
Record layout (int64 x 3 per query): [fp32 cost bits, end, start-or--1]; with the full
warp path (sdtw_path) a second all-gather moves the per-row column ranges (int32 x 2 x N).
This module does no arithmetic of the method: the DP, the overtaking test and the
(cost, end) merges of the reference split all run in the library's kernels.
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


def _on(x, dtype, device) -> torch.Tensor:
    """x (torch tensor or array) as a tensor of `dtype` on `device` (no copy when it is already there)."""
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=dtype)
    return torch.as_tensor(np.asarray(x), device=device).to(dtype)


def _pack(cost, end, start, per: int, device) -> torch.Tensor:
    """[per, 3] int64 records on `device`: fp32 cost bits, end, start (-1 without start)."""
    rec = torch.full((per, 3), -1, dtype=torch.int64, device=device)
    n = int(cost.shape[0])
    if n:
        rec[:n, 0] = _on(cost, torch.float32, device).view(torch.int32).to(torch.int64)
        rec[:n, 1] = _on(end, torch.int64, device)
        if start is not None:
            rec[:n, 2] = _on(start, torch.int64, device)
    return rec


def _unpack(rec: torch.Tensor, Z: int, want_start: bool):
    rec = rec[:Z]
    cost = rec[:, 0].to(torch.int32).view(torch.float32)
    end = rec[:, 1].clone()
    start = rec[:, 2].clone() if want_start else None
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


def comm_device(group=None, device=None):
    """Where the collectives run: the CUDA device for NCCL, the host for gloo."""
    if dist.get_backend(group) == "nccl":
        if device is not None and torch.device(device).type == "cuda":
            return torch.device(device)
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def distributed_batch(Q, group=None, traceback: bool = False,
                      fn: Optional[Callable] = None, device=None, pre_sharded: bool = False,
                      path: bool = False):
    """Shard Q [Z, N] over the ranks of `group`, compute locally, all-gather results.

    fn(Q_shard) -> (cost, end[, start[, path_lo, path_hi]]); default: this package's CUDA
    ``batch`` / ``traceback`` / ``path``.  With pre_sharded=True, Q is already this rank's
    shard and every rank holds the same number of queries (global Z = world *
    Q.shape[0]).  Returns torch tensors on the communication device (the GPU under NCCL,
    the host under gloo) on every rank: (cost[Z] fp32, end[Z] int64, start[Z] int64 |
    None), plus (path_lo[Z, N], path_hi[Z, N]) int32 when path=True (a second all-gather)."""
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
    cdev = comm_device(group, device)
    N = int(Q.shape[1]) if len(Q.shape) > 1 else 1
    if hi > lo:
        out = fn(Q[lo:hi])
    else:
        out = (np.empty(0, np.float32), np.empty(0, np.int64), np.empty(0, np.int64),
               np.empty((0, N), np.int32), np.empty((0, N), np.int32))
    start = out[2] if traceback else None
    rec = _pack(out[0], out[1], start, per, cdev)
    res = _unpack(_gather(rec, world, group), Z, traceback)
    if not path:
        return res
    pth = torch.full((per, N, 2), -1, dtype=torch.int32, device=cdev)
    n = hi - lo
    if n:
        pth[:n, :, 0] = _on(out[3], torch.int32, cdev)
        pth[:n, :, 1] = _on(out[4], torch.int32, cdev)
    full = _gather(pth, world, group)[:Z]
    return res + (full[:, :, 0].contiguous(), full[:, :, 1].contiguous())


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
# boundary DPs (point-to-point column hand-offs).  The ops object supplies the DP calls and
# the two decisions (overtaking test, lexicographic merge): the CUDA library on GPUs, plain
# numpy in the CPU tests.


class CudaSplitOps:
    """The DP calls and decisions of the reference split on the CUDA library (current device).

    NOTE: set_reference REPLACES this device's library reference with the rank's slice; a
    later sdtw_batch on this device runs against that slice until set_reference is called
    again (the library keeps one reference per device)."""

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

    def columns_dominate(self, B, F):
        return self.sd.columns_dominate(B, F)

    def merge_candidates(self, cost, end, valid):
        return self.sd.merge_candidates(cost, end, valid)

    def normalize(self, Q, Y):
        """Per-query and whole-reference z-normalisation on the GPU (sdtw_znormalize):
        the slices share the global statistics of the reference.  Exact sums (reading G8) make
        this bit-identical to set_reference's own grid-reduction normalisation."""
        Yd = Y.to(device=Q.device, dtype=torch.float32) if isinstance(Y, torch.Tensor) else \
            torch.as_tensor(np.asarray(Y, np.float32), device=Q.device)
        return self.sd.znormalize(Q), self.sd.znormalize(Yd)


def split_bounds(M: int, world: int, cols: int):
    """Slice [lo, hi) of every rank: equal multiples of the round width, the last takes the rest."""
    per = -(-(-(-M // world)) // cols) * cols
    return [(min(M, r * per), min(M, (r + 1) * per)) for r in range(world)]


def _comm_device(group, dev):
    """gloo moves host tensors (CPU tests, or several ranks sharing one GPU); NCCL device ones."""
    if dist.is_initialized() and dist.get_backend(group) == "gloo":
        return torch.device("cpu")
    return dev


def _bits(c) -> torch.Tensor:
    return c.view(torch.int32).to(torch.int64)


def _float(b: torch.Tensor) -> torch.Tensor:
    return b.to(torch.int32).view(torch.float32)


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
    dev = Q.device
    Yt = _on(Y, torch.float32, dev)
    M = int(Yt.shape[0])
    cols = ops.round_columns(N)
    bounds = split_bounds(M, world, cols)
    lo, hi = bounds[rank]
    if any(b[1] <= b[0] for b in bounds):
        raise ValueError("reference too short for %d slices of %d-column rounds" % (world, cols))
    cdev = _comm_device(group, dev)
    ops.set_reference(Yt[lo:hi].contiguous())
    last = rank < world - 1
    cf, ef, col_check, col_last, check_cols = ops.batch_columns(Q, last)
    cf = _on(cf, torch.float32, cdev)
    ef = _on(ef, torch.int64, cdev) + lo
    # 1) every rank's last column -> its successor (one all-gather, Z x N fp32 per rank)
    mine = col_last if col_last is not None else torch.full((Z, N), float("inf"), device=dev)
    mine = _on(mine, torch.float32, cdev).reshape(Z, N).contiguous()
    cols_all = (_gather(mine, world, group) if world > 1 else mine).reshape(world, Z, N)
    # 2) correction of this slice from the predecessor's last column (no free start); it is
    #    usable iff overtaken: its column >= the free DP's column at check_cols - 1, every row
    cc = torch.full((Z,), float("inf"), dtype=torch.float32, device=cdev)
    ec = torch.zeros(Z, dtype=torch.int64, device=cdev)
    dom = torch.ones(Z, dtype=torch.int64, device=cdev)
    if rank > 0:
        c2, e2, colB = ops.boundary_dp(Q, _on(cols_all[rank - 1], torch.float32, dev), False, check_cols)
        cc = _on(c2, torch.float32, cdev)
        ec = _on(e2, torch.int64, cdev) + lo
        dom = _on(ops.columns_dominate(_on(colB, torch.float32, dev).reshape(Z, N),
                                       _on(col_check, torch.float32, dev).reshape(Z, N)), torch.int64, cdev)
    # 3) per-query records of every rank (one all-gather): free (cost, end), correction
    #    (cost, end), overtaken flag
    rec = torch.stack([_bits(cf), ef, _bits(cc), ec, dom], dim=1)
    recs = (_gather(rec, world, group) if world > 1 else rec).reshape(world, Z, 5)
    # lexmin over 2*world candidate sets: every free candidate, every overtaken correction
    cand_c = torch.cat([_float(recs[:, :, 0]), _float(recs[:, :, 2])], 0)
    cand_e = torch.cat([recs[:, :, 1], recs[:, :, 3]], 0)
    valid = torch.cat([torch.ones((world, Z), dtype=torch.int32, device=cdev), recs[:, :, 4].to(torch.int32)], 0)
    cost, end, bad = ops.merge_candidates(_on(cand_c, torch.float32, dev), _on(cand_e, torch.int64, dev),
                                          _on(valid, torch.int32, dev))
    cost = _on(cost, torch.float32, "cpu").numpy().copy()
    end = _on(end, torch.int64, "cpu").numpy().copy()
    idx = np.nonzero(_on(bad, torch.int32, "cpu").numpy())[0]
    if idx.size:
        # 4) exact fallback for those queries: rank-ordered chain of full boundary DPs
        it = torch.as_tensor(idx, device=dev)
        Qf = Q[it].contiguous()
        F_ = len(idx)
        if rank == 0:
            cfl, efl = cf[torch.as_tensor(idx, device=cdev)], ef[torch.as_tensor(idx, device=cdev)]
            tout = _on(col_last, torch.float32, dev).reshape(Z, N)[it]
        else:
            tin = torch.empty((F_, N), dtype=torch.float32, device=cdev)
            dist.recv(tin, src=_global(group, rank - 1), group=group)
            c3, e3, tout = ops.boundary_dp(Qf, _on(tin, torch.float32, dev), True, 0)
            cfl = _on(c3, torch.float32, cdev)
            efl = _on(e3, torch.int64, cdev) + lo
        if rank < world - 1:
            dist.send(_on(tout, torch.float32, cdev).reshape(F_, N).contiguous(),
                      dst=_global(group, rank + 1), group=group)
        rf = torch.stack([_bits(cfl), efl], dim=1)
        rfs = (_gather(rf, world, group) if world > 1 else rf).reshape(world, F_, 2)
        c_, e_, _ = ops.merge_candidates(_on(_float(rfs[:, :, 0]), torch.float32, dev),
                                         _on(rfs[:, :, 1], torch.int64, dev), None)
        cost[idx] = _on(c_, torch.float32, "cpu").numpy()
        end[idx] = _on(e_, torch.int64, "cpu").numpy()
    return cost.astype(np.float32), end.astype(np.int64), int(idx.size)


def _global(group, r: int) -> int:
    return dist.get_global_rank(group, r) if group is not None else r
