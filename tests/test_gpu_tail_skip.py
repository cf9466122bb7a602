"""GPU parity of the tail skip: in the partial last round of the reference the
warps whose strips all lie beyond M stop one round early.  For every fill level of that
round (1, 2, 3 or 4 warps of the ring still holding columns) and every schedule (one CTA
per query, sequential persistent segments, speculative segments, a 2-CTA cluster ring, four
and one chains per lane), cost/end must be what the
oracle gives and bit-identical to the run without the skip (SDTW_NO_TAIL_SKIP, read per
call).  Query 0 is cut verbatim from the last N samples of the reference, so its optimum
(cost 0) sits in the partial round itself."""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import oracle  # noqa: E402
import paper_2403_06931_b200 as sd  # noqa: E402
from datagen import nanopore_queries, nanopore_reference  # noqa: E402

DEV = torch.device("cuda", 0)


def _batch(Q, Y, opts, skip):
    if skip:
        os.environ.pop("SDTW_NO_TAIL_SKIP", None)
    else:
        os.environ["SDTW_NO_TAIL_SKIP"] = "1"
    try:
        with sd.options(OPT_NORMALIZE=0, **opts):
            sd.set_reference(torch.as_tensor(Y, device=DEV))
            c, e = sd.batch(torch.as_tensor(np.ascontiguousarray(Q), device=DEV))
            torch.cuda.synchronize()
    finally:
        os.environ.pop("SDTW_NO_TAIL_SKIP", None)
    return c.cpu().numpy(), e.cpu().numpy()


@pytest.mark.parametrize("fill", [1, 961, 1921, 2881, 0])
@pytest.mark.parametrize("sched", [dict(), dict(OPT_SCHED=2, OPT_SEGMENTS=3), dict(OPT_SCHED=3),
                                   dict(OPT_CLUSTER=2, OPT_LANES=2), dict(OPT_PACKED=2), dict(OPT_PACKED=0)])
def test_tail_skip_matches_oracle_and_no_skip(fill, sched):
    N, Z = 200, 6
    with sd.options(**sched):
        cols = sd.round_columns(N)                  # 3840 with the default 4-warp rings
    M = cols * 12 + (fill if fill <= 1 else fill * cols // 3840)   # last round: `fill` (scaled) columns
    Y = oracle.znorm(nanopore_reference(M, 71)[None])[0]
    Q = oracle.znorm(nanopore_queries(Z, N, M, 71))
    Q[0] = Y[M - N:]                                # exact cut at the very end: cost 0, end M-1
    c, e = _batch(Q, Y, sched, skip=True)
    c0, e0 = _batch(Q, Y, sched, skip=False)
    assert np.array_equal(c.view(np.uint32), c0.view(np.uint32)) and np.array_equal(e, e0)
    ref = oracle.sdtw(Q, Y, fma=True, last_rows=True)
    assert np.array_equal(c.view(np.uint32), ref["cost"].view(np.uint32)), (c, ref["cost"])
    for k in np.nonzero(e != ref["end"])[0]:
        assert ref["last_rows"][k, e[k]] == ref["cost"][k], (k, e[k], ref["end"][k])
    assert c[0] == 0.0 and e[0] == M - 1


def _batch_kind(kind, Q, Y, skip):
    if skip:
        os.environ.pop("SDTW_NO_TAIL_SKIP", None)
    else:
        os.environ["SDTW_NO_TAIL_SKIP"] = "1"
    try:
        opts = dict(OPT_NORMALIZE=0, OPT_PRECISION=16) if kind == "half" else dict(OPT_NORMALIZE=0)
        with sd.options(**opts):
            sd.set_reference(torch.as_tensor(Y, device=DEV))
            Qt = torch.as_tensor(np.ascontiguousarray(Q), device=DEV)
            c, e = sd.batch_q8(Qt) if kind == "q8" else sd.batch(Qt)
            torch.cuda.synchronize()
    finally:
        os.environ.pop("SDTW_NO_TAIL_SKIP", None)
    return c.cpu().numpy(), e.cpu().numpy()


@pytest.mark.parametrize("kind", ["half", "q8"])
def test_tail_skip_reduced_precision_kernels(kind):
    """The packed-half and uint8-codebook kernels (sdtw_dp2.cuh) skip the same way: over
    reference lengths that leave their last round filled to different depths, the results are
    bit-identical to the run without the skip, and the verbatim copy of the reference's last
    N samples is found at cost 0, end M-1; parity against the reduced-precision oracles is
    in test_gpu_half.py / test_gpu_q8.py."""
    N, Z = 200, 4
    for M in range(30_000, 30_000 + 6 * 1_283, 1_283):
        Y = oracle.znorm(nanopore_reference(M, 73)[None])[0]
        Q = oracle.znorm(nanopore_queries(Z, N, M, 73))
        Q[0] = Y[M - N:]
        c, e = _batch_kind(kind, Q, Y, True)
        c0, e0 = _batch_kind(kind, Q, Y, False)
        assert np.array_equal(c.view(np.uint32), c0.view(np.uint32)) and np.array_equal(e, e0), M
        assert c[0] == 0.0 and e[0] == M - 1, (M, c[0], e[0])
