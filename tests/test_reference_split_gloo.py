"""World-size-2/3 gloo tests of the reference-split host logic on CPU.

The DP calls are injected: a plain float32 column-by-column DP written here (the oracle's
non-FMA cell, fl(fl(x-y)^2 + m)), so the slicing, the last-column all-gather, the
correction / overtaking test, the record all-gather and the rank-ordered exact fallback
(point-to-point hand-offs) run without a GPU.  Results must equal the oracle on the whole
reference bit for bit, for random queries (corrections overtaken) and for queries that copy
the reference across a slice boundary (corrections not overtaken -> fallback chain)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

F32 = np.float32
INF = F32(np.inf)
COLS = 8          # "round width" of the injected DP
RC = 2            # correction rounds


def _dp_cols(x, y, T, zrow):
    N = len(x)
    prev = np.asarray(T, F32).copy()
    top = F32(zrow)
    cols = np.empty((len(y), N), F32)
    for j, yj in enumerate(np.asarray(y, F32)):
        up = F32(zrow)
        for i in range(N):
            m = min(prev[i], up, prev[i - 1] if i > 0 else top)
            t = F32(x[i] - yj)
            cols[j, i] = F32(F32(t * t) + F32(m))
            up = cols[j, i]
        prev = cols[j]
        top = F32(zrow)
    return cols


def _best(cols):
    last = cols[:, -1]
    j = int(np.argmin(last))
    return F32(last[j]), j


class NumpyOps:
    def round_columns(self, N):
        return COLS

    def set_reference(self, Y):
        self.Y = np.asarray(Y, F32)

    def batch_columns(self, Q, last):
        Q = np.asarray(Q)
        c, e, ck, cl = [], [], [], []
        for x in Q:
            cols = _dp_cols(x, self.Y, np.full(len(x), INF, F32), 0.0)
            b = _best(cols)
            c.append(b[0]); e.append(b[1])
            ck.append(cols[RC * COLS - 1]); cl.append(cols[-1])
        return (np.array(c, F32), np.array(e, np.int64), torch.tensor(np.array(ck)),
                torch.tensor(np.array(cl)) if last else None, RC * COLS)

    def boundary_dp(self, Q, boundary, free_start, n_cols):
        Q = np.asarray(Q)
        B = np.asarray(boundary, F32)
        Y = self.Y if n_cols == 0 else self.Y[:n_cols]
        c, e, col = [], [], []
        for q, x in enumerate(Q):
            cols = _dp_cols(x, Y, B[q], 0.0 if free_start else INF)
            b = _best(cols)
            c.append(b[0]); e.append(b[1]); col.append(cols[-1])
        return np.array(c, F32), np.array(e, np.int64), torch.tensor(np.array(col))

    # the two decisions (the CUDA library's sdtw_columns_dominate / sdtw_merge_candidates)
    def columns_dominate(self, B, F):
        return torch.tensor((np.asarray(B) >= np.asarray(F)).all(axis=1).astype(np.int32))

    def merge_candidates(self, cost, end, valid):
        c, e = np.asarray(cost), np.asarray(end)
        v = np.ones(c.shape, bool) if valid is None else np.asarray(valid) != 0
        bc = np.full(c.shape[1], INF)
        be = np.zeros(c.shape[1], np.int64)
        for k in range(c.shape[0]):
            take = v[k] & ((c[k] < bc) | ((c[k] == bc) & (e[k] < be)))
            bc = np.where(take, c[k], bc)
            be = np.where(take, e[k], be)
        be = np.where(np.isinf(bc), 0, be)
        return torch.tensor(bc), torch.tensor(be), torch.tensor((~v).any(axis=0).astype(np.int32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(kind, world):
    rng = np.random.default_rng(31)
    Y = rng.standard_normal(100).astype(F32)
    if kind == "random":
        Q = rng.standard_normal((4, 6)).astype(F32)
    else:   # copies of Y across the slice boundaries (56 for 2 ranks; 40, 80 for 3) that run on
            # past the correction's last column (boundary + 15): the corrections are not overtaken
        starts = [50, 54] if world == 2 else [36, 76]
        Q = np.stack([Y[a:a + 24] for a in starts] + [rng.standard_normal(24).astype(F32)]).astype(F32)
    return Q, Y


def _worker(rank, world, port, kind, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2403_06931_b200.distributed import reference_split_batch
        Q, Y = _inputs(kind, world)
        cost, end, fb = reference_split_batch(torch.from_numpy(Q), Y, ops=NumpyOps())
        out_q.put((rank, cost, end, fb))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "random"), (3, "random"), (2, "straddle"), (3, "straddle")])
def test_reference_split_matches_single_process(world, kind):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    Q, Y = _inputs(kind, world)
    ref = oracle.sdtw(Q, Y, fma=False)
    for rank, cost, end, fb in res:
        assert np.array_equal(cost.view(np.uint32), ref["cost"].view(np.uint32)), (rank, cost, ref["cost"])
        assert np.array_equal(end, ref["end"]), (rank, end, ref["end"])
        if kind == "straddle":
            assert fb >= 2                 # both copies go through the exact fallback chain
            assert np.all(cost[:2] == 0)


def test_split_bounds_are_round_multiples():
    from paper_2403_06931_b200.distributed import split_bounds
    b = split_bounds(10_000_000, 8, 7680)
    assert b[0] == (0, 1_251_840) and all((hi - lo) % 7680 == 0 for lo, hi in b[:-1]) and b[-1][1] == 10_000_000
    assert all(b[r][1] == b[r + 1][0] for r in range(7))
