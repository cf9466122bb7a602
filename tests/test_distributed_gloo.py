"""World-size-2 gloo test of the query-sharded multi-GPU host logic on CPU.

The per-rank compute is injected (the CPU oracle -- tests may call it) so that the
sharding, padding, record packing and the one all-gather are exercised without
a GPU; results must equal the single-process oracle bit for bit, including a
batch size not divisible by the world size and an empty shard."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, Z, traceback, out_q):  # noqa: C901
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2403_06931_b200.distributed import distributed_batch
        rng = np.random.default_rng(5)
        Y = rng.standard_normal(700).astype(np.float32)
        Q = rng.standard_normal((Z, 24)).astype(np.float32)

        def fn(Qs):
            r = oracle.sdtw(np.asarray(Qs), Y, start=traceback, threads=1)
            return (r["cost"], r["end"], r["start"]) if traceback else (r["cost"], r["end"])

        cost, end, start = distributed_batch(Q, traceback=traceback, fn=fn)
        out_q.put((rank, cost.numpy(), end.numpy(), None if start is None else start.numpy()))
    finally:
        dist.destroy_process_group()


def _path_worker(rank, world, port, Z, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2403_06931_b200.distributed import distributed_batch
        rng = np.random.default_rng(9)
        Y = rng.standard_normal(300).astype(np.float32)
        Q = rng.standard_normal((Z, 12)).astype(np.float32)

        def fn(Qs):
            rs = [oracle.sdtw_path(q, Y) for q in np.asarray(Qs)]
            return (np.array([r[0] for r in rs], np.float32), np.array([r[1] for r in rs], np.int64),
                    np.array([r[2] for r in rs], np.int64), np.array([r[3] for r in rs], np.int32),
                    np.array([r[4] for r in rs], np.int32))

        out_q.put((rank,) + tuple(t.numpy() for t in distributed_batch(Q, path=True, fn=fn)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("Z", [5, 1])
def test_gloo_world2_path_matches_single_process(Z):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_path_worker, args=(r, 2, port, Z, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(9)
    Y = rng.standard_normal(300).astype(np.float32)
    Q = rng.standard_normal((Z, 12)).astype(np.float32)
    for _, cost, end, start, lo, hi in res:
        for k in range(Z):
            rc, re, rs, rlo, rhi = oracle.sdtw_path(Q[k], Y)
            assert cost[k] == rc and end[k] == re and start[k] == rs
            assert np.array_equal(lo[k], rlo) and np.array_equal(hi[k], rhi)


@pytest.mark.parametrize("world,Z,traceback", [(2, 7, False), (2, 8, True), (2, 1, True),
                                               (3, 7, True), (3, 2, False), (4, 9, True), (4, 3, True)])
def test_gloo_world_n_matches_single_process(world, Z, traceback):
    """World sizes 2-4, Z not divisible by the world size, empty shards (Z < world)."""
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, Z, traceback, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(5)
    Y = rng.standard_normal(700).astype(np.float32)
    Q = rng.standard_normal((Z, 24)).astype(np.float32)
    ref = oracle.sdtw(Q, Y, start=True)
    for _, cost, end, start in res:
        assert np.array_equal(cost, ref["cost"])
        assert np.array_equal(end, ref["end"])
        if traceback:
            assert np.array_equal(start, ref["start"])


def test_shard_bounds_cover_everything_once():
    from paper_2403_06931_b200.distributed import shard_bounds
    for Z in (0, 1, 7, 8, 512, 513):
        for world in (1, 2, 3, 8):
            seen = []
            for r in range(world):
                lo, hi, per = shard_bounds(Z, world, r)
                assert 0 <= hi - lo <= per
                seen.extend(range(lo, hi))
            assert seen == list(range(Z))
