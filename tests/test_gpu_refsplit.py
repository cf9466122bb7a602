"""GPU parity of the reference split: 2 and 3 ranks sharing the test GPU
(gloo for the exchanges; NCCL on a multi-GPU node), every rank holding one slice of the
reference, results bit-exact against the oracle on the whole reference -- random queries
(corrections overtaken) and queries copying the reference across a slice boundary past the
correction (exact fallback chain)."""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(kind, world):
    import oracle
    from datagen import nanopore_queries, nanopore_reference
    M = 200_000
    Y = oracle.znorm(nanopore_reference(M, 71)[None])[0]
    if kind == "random":
        return oracle.znorm(nanopore_queries(8, 300, M, 71)), Y, {}
    per = -(-(-(-M // world)) // 960) * 960          # slice length, one-warp rings (960 columns per round)
    Q = np.stack([Y[r * per - 200:r * per + 1300] for r in range(1, world)] +
                 [oracle.znorm(nanopore_queries(1, 1500, M, 72))[0]]).astype(np.float32)
    return Q, Y, dict(OPT_LANES=1, OPT_SPEC_ROUNDS=1)


def _worker(rank, world, port, kind, out_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        import paper_2403_06931_b200 as sd
        from paper_2403_06931_b200.distributed import reference_split_batch
        Q, Y, opts = _inputs(kind, world)
        with sd.options(**opts):
            cost, end, fb = reference_split_batch(torch.as_tensor(Q, device="cuda"), Y)
        out_q.put((rank, cost, end, fb))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,kind", [(2, "random"), (3, "random"), (2, "straddle"), (3, "straddle")])
def test_reference_split_bit_exact(world, kind):
    import oracle
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    for _ in range(world):
        try:
            res.append(q.get(timeout=180))
        except Exception:                            # a rank died: do not wait for the rest
            break
    for p in procs:
        p.join(timeout=30)
        if p.exitcode is None:
            p.kill()
    assert len(res) == world and all(p.exitcode == 0 for p in procs), [p.exitcode for p in procs]
    Q, Y, _ = _inputs(kind, world)
    ref = oracle.sdtw(Q, Y, last_rows=True)
    for rank, cost, end, fb in res:
        assert np.array_equal(cost.view(np.uint32), ref["cost"].view(np.uint32)), (rank, cost[:4], ref["cost"][:4])
        for k in np.nonzero(end != ref["end"])[0]:
            assert ref["last_rows"][k, end[k]] == ref["cost"][k], (rank, k)
        if kind == "straddle":
            assert fb >= world - 1 and np.all(cost[:world - 1] == 0)


def test_boundary_dp_pieces_match_oracle():
    """The two library calls alone: the free DP of the whole reference equals the batch, and
    a boundary DP over a prefix from +inf with the free start equals the batch on that prefix."""
    import oracle
    import paper_2403_06931_b200 as sd
    from datagen import nanopore_queries, nanopore_reference
    M = 3840 * 30
    Y = oracle.znorm(nanopore_reference(M, 73)[None])[0]
    Q = oracle.znorm(nanopore_queries(5, 400, M, 73))
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device="cuda"))
        Qt = torch.as_tensor(Q, device="cuda")
        cw = sd.round_columns(400)
        c0, e0 = sd.batch(Qt)
        c1, e1, ck, cl, n = sd.batch_columns(Qt)
        assert torch.equal(c0, c1) and torch.equal(e0, e1) and n % cw == 0
        c2, e2, col = sd.boundary_dp(Qt, None, True, 10 * cw)
    ref = oracle.sdtw(Q, Y[:10 * cw])
    assert np.array_equal(c2.cpu().numpy(), ref["cost"]) and np.array_equal(e2.cpu().numpy(), ref["end"])


def test_reference_split_calls_reject_bad_arguments():
    import oracle
    import paper_2403_06931_b200 as sd
    from datagen import nanopore_queries, nanopore_reference
    M = 3840 * 20
    Y = oracle.znorm(nanopore_reference(M, 74)[None])[0]
    Q = torch.as_tensor(oracle.znorm(nanopore_queries(3, 200, M, 74)), device="cuda")
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device="cuda"))
        cw = sd.round_columns(200)
        with pytest.raises(sd.SdtwError) as ei:
            sd.boundary_dp(Q, None, True, cw + 1)                   # not a multiple of the round width
        assert ei.value.status == sd.E_ARG
        with pytest.raises(sd.SdtwError):
            sd.boundary_dp(Q, None, True, M + cw)                   # past the reference
        with sd.options(OPT_CLUSTER=2):
            with pytest.raises(sd.SdtwError):
                sd.batch_columns(Q)                                  # clusters keep sequential segments
        sd.set_reference(torch.as_tensor(Y[:M - 5], device="cuda"))
        with pytest.raises(sd.SdtwError):
            sd.batch_columns(Q)                                      # last column needs whole rounds
        c, e, ck, cl, n = sd.batch_columns(Q, last=False)
        assert cl is None and torch.isfinite(ck).all()


def test_reference_split_normalises_raw_inputs():
    """normalize=True on raw inputs equals the whole-reference batch with OPT_NORMALIZE=1
    (world size 1: one slice, no exchange)."""
    import paper_2403_06931_b200 as sd
    from datagen import nanopore_queries, nanopore_reference
    from paper_2403_06931_b200.distributed import reference_split_batch
    M = 3840 * 40
    Y = nanopore_reference(M, 75)
    Q = torch.as_tensor(nanopore_queries(6, 500, M, 75), device="cuda")
    cost, end, fb = reference_split_batch(Q, Y, normalize=True)
    sd.set_reference(torch.as_tensor(Y, device="cuda"))
    c, e = sd.batch(Q)
    assert np.array_equal(cost, c.cpu().numpy()) and np.array_equal(end, e.cpu().numpy()) and fb == 0


def test_column_calls_write_nothing_on_nonfinite_input():
    """ABI: no partial results on error -- a NaN query sample makes
    sdtw_batch_columns / sdtw_boundary_dp return SDTW_E_NONFINITE with every output buffer
    (cost, end, both columns / col_out) untouched."""
    import ctypes
    import oracle
    import paper_2403_06931_b200 as sd
    from datagen import nanopore_queries, nanopore_reference
    M = 3840 * 20
    Y = oracle.znorm(nanopore_reference(M, 75)[None])[0]
    Q = torch.as_tensor(oracle.znorm(nanopore_queries(4, 300, M, 75)), device="cuda")
    Q[2, 5] = float("nan")
    with sd.options(OPT_NORMALIZE=0):
        sd.set_reference(torch.as_tensor(Y, device="cuda"))
        outs = [torch.full((4,), 7.0, device="cuda"), torch.full((4,), -3, dtype=torch.int64, device="cuda"),
                torch.full((4, 300), 7.0, device="cuda"), torch.full((4, 300), 7.0, device="cuda")]
        before = [o.clone() for o in outs]
        n = ctypes.c_int64(0)
        rc = sd._lib.sdtw_batch_columns(ctypes.c_void_p(Q.data_ptr()), 4, 300, ctypes.c_void_p(outs[0].data_ptr()),
                                        ctypes.c_void_p(outs[1].data_ptr()), ctypes.c_void_p(outs[2].data_ptr()),
                                        ctypes.c_void_p(outs[3].data_ptr()), ctypes.byref(n))
        assert rc == sd.E_NONFINITE
        bnd = torch.zeros((4, 300), device="cuda")
        rc = sd._lib.sdtw_boundary_dp(ctypes.c_void_p(Q.data_ptr()), 4, 300, ctypes.c_void_p(bnd.data_ptr()), 0, 0,
                                      ctypes.c_void_p(outs[0].data_ptr()), ctypes.c_void_p(outs[1].data_ptr()),
                                      ctypes.c_void_p(outs[2].data_ptr()))
        assert rc == sd.E_NONFINITE
        torch.cuda.synchronize()
    for a, b in zip(outs, before):
        assert torch.equal(a, b)
