"""B200-native batched subsequence DTW (arXiv 2403.06931) -- Python binding.

Argument marshalling only: every step of the hot path (z-normalisation, the
wavefront DP, the min/argmin epilogue) runs in the sm_100a kernels of
``libsdtw.so`` behind the C ABI of ``include/sdtw.h``.  There is no CPU
fallback: importing this package fails loudly when the library is missing, and
every call raises when the CUDA path fails.

Functions mirror the ABI names (minus the ``sdtw_`` prefix):
``set_reference``, ``batch``, ``batch_ragged``, ``traceback``, ``path``, ``znormalize``, ``batch_q8``,
``q8_codebook``, ``quantize``, ``set_option``,
``get_option``, ``profile``, ``launch_count``, ``release``.
Inputs may be torch tensors (CUDA or CPU) or numpy arrays.  torch supplies
device memory and the current stream (passed as SDTW_OPT_STREAM).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# SDTW_LIB: load an experimental build of the same library from its own path (A/B and
# alternate-layout parity runs) instead of overwriting the in-tree libsdtw.so
LIB_PATH = os.environ.get("SDTW_LIB") or os.path.join(_HERE, "libsdtw.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        "paper_2403_06931_b200: CUDA library %s is missing -- run "
        "`python __graft_entry__.py` (or `python paper_2403_06931_b200/build.py`); "
        "there is no CPU fallback" % LIB_PATH)

_lib = ctypes.CDLL(LIB_PATH)
_f32p = ctypes.c_void_p
_i64 = ctypes.c_int64
_lib.sdtw_set_reference.argtypes = [ctypes.c_void_p, _i64]
_lib.sdtw_batch.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_traceback.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_batch_ragged.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p]
_lib.sdtw_path.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                           ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_znormalize.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p]
_lib.sdtw_set_option.argtypes = [ctypes.c_int, _i64]
_lib.sdtw_get_option.argtypes = [ctypes.c_int, ctypes.POINTER(_i64)]
_lib.sdtw_profile.argtypes = [ctypes.POINTER(ctypes.c_double), ctypes.POINTER(_i64)]
_lib.sdtw_spec_recomputed.argtypes = [ctypes.POINTER(_i64)]
_lib.sdtw_round_columns.argtypes = [_i64, ctypes.POINTER(_i64)]
_lib.sdtw_batch_columns.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                    ctypes.c_void_p, ctypes.POINTER(_i64)]
_lib.sdtw_boundary_dp.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_int, _i64, ctypes.c_void_p,
                                  ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_columns_dominate.argtypes = [ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_void_p]
_lib.sdtw_merge_candidates.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, _i64, _i64, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_batch_q8.argtypes = [ctypes.c_void_p, _i64, _i64, ctypes.c_void_p, ctypes.c_void_p]
_lib.sdtw_q8_codebook.argtypes = [ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_float)]
_lib.sdtw_quantize.argtypes = [ctypes.c_void_p, _i64, ctypes.c_void_p]
_lib.sdtw_launch_count.restype = _i64
_lib.sdtw_last_error.restype = ctypes.c_char_p
_lib.sdtw_version.restype = ctypes.c_int
_lib.sdtw_build_info.restype = ctypes.c_char_p
for _n in ("sdtw_set_reference", "sdtw_batch", "sdtw_batch_ragged", "sdtw_traceback", "sdtw_path", "sdtw_znormalize",
           "sdtw_set_option", "sdtw_get_option", "sdtw_profile", "sdtw_spec_recomputed", "sdtw_round_columns",
           "sdtw_batch_columns", "sdtw_boundary_dp", "sdtw_columns_dominate", "sdtw_merge_candidates",
           "sdtw_batch_q8", "sdtw_q8_codebook", "sdtw_quantize"):
    getattr(_lib, _n).restype = ctypes.c_int

# ABI constants (include/sdtw.h)
OK, E_ARG, E_NOREF, E_CUDA, E_NOMEM, E_NONFINITE = range(6)
OPT_NORMALIZE, OPT_FMA, OPT_SEGMENT_W, OPT_LANES, OPT_CLUSTER, OPT_STREAM, OPT_PACKED, OPT_CHUNK, \
    OPT_PROFILE, OPT_RING, OPT_SCHED, OPT_SEGMENTS, OPT_WORKERS, OPT_PRECISION, OPT_PAD, \
    OPT_SPEC_ROUNDS, OPT_START, OPT_Q8_PRUNE, OPT_Q8_CLIP, OPT_STAT_FIXUP_DEPTH, OPT_QUERY_ROWS = range(1, 22)
_STATUS = {0: "SDTW_OK", 1: "SDTW_E_ARG", 2: "SDTW_E_NOREF", 3: "SDTW_E_CUDA", 4: "SDTW_E_NOMEM",
           5: "SDTW_E_NONFINITE"}

EXPORTED_SYMBOLS = ("sdtw_set_reference", "sdtw_batch", "sdtw_batch_ragged", "sdtw_traceback", "sdtw_path", "sdtw_znormalize",
                    "sdtw_set_option", "sdtw_get_option", "sdtw_profile", "sdtw_spec_recomputed", "sdtw_launch_count",
                    "sdtw_round_columns", "sdtw_batch_columns", "sdtw_boundary_dp",
                    "sdtw_columns_dominate", "sdtw_merge_candidates",
                    "sdtw_batch_q8", "sdtw_q8_codebook", "sdtw_quantize",
                    "sdtw_last_error", "sdtw_release", "sdtw_version", "sdtw_build_info")


class SdtwError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__("%s: %s" % (_STATUS.get(status, status), msg))
        self.status = status


def _check(rc: int):
    if rc != OK:
        raise SdtwError(rc, _lib.sdtw_last_error().decode(errors="replace"))


def _torch():
    try:
        import torch
        return torch
    except ImportError:  # pragma: no cover
        return None


def _bind_stream(t):
    """Route the library onto torch's current stream of the tensor's device."""
    torch = _torch()
    if torch is not None and isinstance(t, torch.Tensor) and t.is_cuda:
        _check(_lib.sdtw_set_option(OPT_STREAM, torch.cuda.current_stream(t.device).cuda_stream))
    else:
        _check(_lib.sdtw_set_option(OPT_STREAM, 0))


def _as_f32(x):
    """(keepalive, pointer, shape) for a torch tensor or array-like, contiguous fp32."""
    torch = _torch()
    if torch is not None and isinstance(x, torch.Tensor):
        t = x.detach()
        if t.dtype != torch.float32:
            t = t.float()
        t = t.contiguous()
        return t, t.data_ptr(), tuple(t.shape)
    a = np.ascontiguousarray(np.asarray(x, dtype=np.float32))
    return a, a.ctypes.data, a.shape


def version() -> int:
    return int(_lib.sdtw_version())


def build_info() -> str:
    """sdtw_build_info: the nvcc/ptxas version the library was compiled with, and its pack mode."""
    return _lib.sdtw_build_info().decode()


def set_option(key: int, value: int):
    _check(_lib.sdtw_set_option(int(key), int(value)))


def get_option(key: int) -> int:
    v = _i64()
    _check(_lib.sdtw_get_option(int(key), ctypes.byref(v)))
    return int(v.value)


def set_reference(Y):
    """sdtw_set_reference(Y, M): install the reference on the current device."""
    keep, ptr, shape = _as_f32(Y)
    if len(shape) != 1:
        raise ValueError("reference must be 1-D")
    _bind_stream(keep)
    _check(_lib.sdtw_set_reference(ctypes.c_void_p(ptr), shape[0]))


def _outputs(keep, Z, trace):
    torch = _torch()
    if torch is not None and isinstance(keep, torch.Tensor) and keep.is_cuda:
        dev = keep.device
        cost = torch.empty(Z, dtype=torch.float32, device=dev)
        end = torch.empty(Z, dtype=torch.int64, device=dev)
        start = torch.empty(Z, dtype=torch.int64, device=dev) if trace else None
        ptrs = (cost.data_ptr(), end.data_ptr(), start.data_ptr() if trace else 0)
    else:
        cost = np.empty(Z, np.float32)
        end = np.empty(Z, np.int64)
        start = np.empty(Z, np.int64) if trace else None
        ptrs = (cost.ctypes.data, end.ctypes.data, start.ctypes.data if trace else 0)
    return cost, end, start, ptrs


def batch(Q):
    """sdtw_batch: Q [Z, N] -> (cost[Z] fp32, end[Z] int64) on Q's device (numpy if host)."""
    keep, ptr, shape = _as_f32(Q)
    if len(shape) == 1:
        shape = (1, shape[0])
    Z, N = shape
    cost, end, _, (pc, pe, _) = _outputs(keep, Z, False)
    _bind_stream(keep)
    _check(_lib.sdtw_batch(ctypes.c_void_p(ptr), Z, N, ctypes.c_void_p(pc), ctypes.c_void_p(pe)))
    return cost, end


def batch_q8(Q):
    """sdtw_batch_q8 (uint8 codebook): Q [Z, N] -> (cost[Z] int32, the exact
    integer cost; end[Z] int64) on Q's device (numpy if host).  Pruning: OPT_Q8_PRUNE."""
    keep, ptr, shape = _as_f32(Q)
    if len(shape) == 1:
        shape = (1, shape[0])
    Z, N = shape
    cost, end, _, (pc, pe, _) = _outputs(keep, Z, False)
    torch = _torch()
    cost = cost.view(torch.int32) if torch is not None and isinstance(cost, torch.Tensor) else cost.view(np.int32)
    _bind_stream(keep)
    _check(_lib.sdtw_batch_q8(ctypes.c_void_p(ptr), Z, N, ctypes.c_void_p(pc), ctypes.c_void_p(pe)))
    return cost, end


def q8_codebook():
    """sdtw_q8_codebook: (lo, hi) of the current reference's uint8 codebook."""
    lo, hi = ctypes.c_float(), ctypes.c_float()
    _check(_lib.sdtw_q8_codebook(ctypes.byref(lo), ctypes.byref(hi)))
    return np.float32(lo.value), np.float32(hi.value)


def quantize(X):
    """sdtw_quantize: uint8 codes of X under the current codebook (same device as X)."""
    keep, ptr, shape = _as_f32(X)
    n = int(np.prod(shape)) if len(shape) else 1
    torch = _torch()
    if torch is not None and isinstance(keep, torch.Tensor) and keep.is_cuda:
        out = torch.empty(shape, dtype=torch.uint8, device=keep.device)
        po = out.data_ptr()
    else:
        out = np.empty(shape, np.uint8)
        po = out.ctypes.data
    _bind_stream(keep)
    _check(_lib.sdtw_quantize(ctypes.c_void_p(ptr), n, ctypes.c_void_p(po)))
    return out


def round_columns(N: int) -> int:
    """sdtw_round_columns: reference columns per DP round for queries of length N."""
    n = _i64()
    _check(_lib.sdtw_round_columns(int(N), ctypes.byref(n)))
    return int(n.value)


def batch_columns(Q, last: bool = True):
    """sdtw_batch_columns (device tensors only): Q [Z, N] -> (cost, end, col_check [Z, N],
    col_last [Z, N], check_cols): the free DP's column at reference column check_cols - 1
    and at the last column."""
    torch = _torch()
    Z, N = Q.shape
    col_check = torch.empty((Z, N), dtype=torch.float32, device=Q.device)
    col_last = torch.empty((Z, N), dtype=torch.float32, device=Q.device) if last else None
    keep, ptr, _ = _as_f32(Q)
    cost, end, _, (pc, pe, _) = _outputs(keep, Z, False)
    n = _i64()
    _bind_stream(keep)
    _check(_lib.sdtw_batch_columns(ctypes.c_void_p(ptr), Z, N, ctypes.c_void_p(pc), ctypes.c_void_p(pe),
                                   ctypes.c_void_p(col_check.data_ptr()),
                                   ctypes.c_void_p(None if col_last is None else col_last.data_ptr()),
                                   ctypes.byref(n)))
    return cost, end, col_check, col_last, int(n.value)


def boundary_dp(Q, boundary=None, free_start: bool = True, n_cols: int = 0, column: bool = True):
    """sdtw_boundary_dp (device tensors only): the DP over reference columns [0, n_cols)
    from the left boundary column `boundary` [Z, N] (None = +inf), with or without the free
    start -> (cost, end, column n_cols-1 [Z, N] or None)."""
    torch = _torch()
    Z, N = Q.shape
    keep, ptr, _ = _as_f32(Q)
    bkeep = None if boundary is None else boundary.to(torch.float32).contiguous()
    col = torch.empty((Z, N), dtype=torch.float32, device=Q.device) if column else None
    cost, end, _, (pc, pe, _) = _outputs(keep, Z, False)
    _bind_stream(keep)
    _check(_lib.sdtw_boundary_dp(ctypes.c_void_p(ptr), Z, N,
                                 ctypes.c_void_p(None if bkeep is None else bkeep.data_ptr()),
                                 1 if free_start else 0, int(n_cols), ctypes.c_void_p(pc), ctypes.c_void_p(pe),
                                 ctypes.c_void_p(None if col is None else col.data_ptr())))
    return cost, end, col


def columns_dominate(B, F):
    """sdtw_columns_dominate (device tensors [Z, N]): int32 [Z], 1 iff B >= F on every row."""
    torch = _torch()
    Bk = B.to(torch.float32).contiguous()
    Fk = F.to(torch.float32).contiguous()
    Z, N = Bk.shape
    out = torch.empty(Z, dtype=torch.int32, device=Bk.device)
    _bind_stream(Bk)
    _check(_lib.sdtw_columns_dominate(ctypes.c_void_p(Bk.data_ptr()), ctypes.c_void_p(Fk.data_ptr()), Z, N,
                                      ctypes.c_void_p(out.data_ptr())))
    return out


def merge_candidates(cost, end, valid=None):
    """sdtw_merge_candidates (device tensors [n_sets, Z]): per query the lexicographic
    (cost, end) minimum over the valid sets -> (cost [Z], end [Z], invalid [Z] int32)."""
    torch = _torch()
    ck = cost.to(torch.float32).contiguous()
    ek = end.to(torch.int64).contiguous()
    vk = None if valid is None else valid.to(torch.int32).contiguous()
    S, Z = ck.shape
    oc = torch.empty(Z, dtype=torch.float32, device=ck.device)
    oe = torch.empty(Z, dtype=torch.int64, device=ck.device)
    oi = torch.empty(Z, dtype=torch.int32, device=ck.device)
    _bind_stream(ck)
    _check(_lib.sdtw_merge_candidates(ctypes.c_void_p(ck.data_ptr()), ctypes.c_void_p(ek.data_ptr()),
                                      ctypes.c_void_p(None if vk is None else vk.data_ptr()), S, Z,
                                      ctypes.c_void_p(oc.data_ptr()), ctypes.c_void_p(oe.data_ptr()),
                                      ctypes.c_void_p(oi.data_ptr())))
    return oc, oe, oi


def traceback(Q):
    """sdtw_traceback: Q [Z, N] -> (cost, end, start)."""
    keep, ptr, shape = _as_f32(Q)
    if len(shape) == 1:
        shape = (1, shape[0])
    Z, N = shape
    cost, end, start, (pc, pe, ps) = _outputs(keep, Z, True)
    _bind_stream(keep)
    _check(_lib.sdtw_traceback(ctypes.c_void_p(ptr), Z, N, ctypes.c_void_p(pc), ctypes.c_void_p(pe),
                               ctypes.c_void_p(ps)))
    return cost, end, start


def batch_ragged(Q, offsets, start: bool = False):
    """sdtw_batch_ragged: Q = queries back to back (1-D), query q = Q[offsets[q]:offsets[q+1]]
    -> (cost, end) or (cost, end, start), each exactly the single-query result."""
    keep, ptr, shape = _as_f32(Q)
    torch = _torch()
    if torch is not None and isinstance(offsets, torch.Tensor):
        okeep = offsets.to(torch.int64).contiguous()
        optr = okeep.data_ptr()
        Z = okeep.numel() - 1
    else:
        okeep = np.ascontiguousarray(np.asarray(offsets, dtype=np.int64))
        optr = okeep.ctypes.data
        Z = okeep.shape[0] - 1
    if Z < 0:
        raise ValueError("offsets needs n_queries + 1 entries")
    cost, end, st, (pc, pe, ps) = _outputs(keep, Z, start)
    _bind_stream(keep)
    _check(_lib.sdtw_batch_ragged(ctypes.c_void_p(ptr), ctypes.c_void_p(optr), Z, ctypes.c_void_p(pc),
                                  ctypes.c_void_p(pe), ctypes.c_void_p(ps if start else 0)))
    return (cost, end, st) if start else (cost, end)


def path(Q):
    """sdtw_path: Q [Z, N] -> (cost, end, start, path_lo [Z, N] int32, path_hi [Z, N] int32):
    row i of query q's optimal warp path covers reference columns path_lo[q, i]..path_hi[q, i]."""
    keep, ptr, shape = _as_f32(Q)
    if len(shape) == 1:
        shape = (1, shape[0])
    Z, N = shape
    cost, end, start, (pc, pe, ps) = _outputs(keep, Z, True)
    torch = _torch()
    if torch is not None and isinstance(keep, torch.Tensor) and keep.is_cuda:
        lo = torch.empty((Z, N), dtype=torch.int32, device=keep.device)
        hi = torch.empty((Z, N), dtype=torch.int32, device=keep.device)
        pl, ph = lo.data_ptr(), hi.data_ptr()
    else:
        lo = np.empty((Z, N), np.int32)
        hi = np.empty((Z, N), np.int32)
        pl, ph = lo.ctypes.data, hi.ctypes.data
    _bind_stream(keep)
    _check(_lib.sdtw_path(ctypes.c_void_p(ptr), Z, N, ctypes.c_void_p(pc), ctypes.c_void_p(pe),
                          ctypes.c_void_p(ps), ctypes.c_void_p(pl), ctypes.c_void_p(ph)))
    return cost, end, start, lo, hi


def znormalize(X):
    """sdtw_znormalize (the paper's runNormalizer): per-series z-normalisation on the GPU."""
    keep, ptr, shape = _as_f32(X)
    rows = 1 if len(shape) == 1 else shape[0]
    L = shape[-1]
    torch = _torch()
    if torch is not None and isinstance(keep, torch.Tensor) and keep.is_cuda:
        out = torch.empty_like(keep)
        po = out.data_ptr()
    else:
        out = np.empty(shape, np.float32)
        po = out.ctypes.data
    _bind_stream(keep)
    _check(_lib.sdtw_znormalize(ctypes.c_void_p(ptr), rows, L, ctypes.c_void_p(po)))
    return out


def profile():
    """(dp_ms, launches) of the last batch/traceback call (dp_ms needs OPT_PROFILE=1)."""
    ms = ctypes.c_double()
    n = _i64()
    _check(_lib.sdtw_profile(ctypes.byref(ms), ctypes.byref(n)))
    return float(ms.value), int(n.value)


def spec_recomputed() -> int:
    """Queries of the last batch call recomputed after a failed speculative correction."""
    n = _i64()
    _check(_lib.sdtw_spec_recomputed(ctypes.byref(n)))
    return int(n.value)


def launch_count() -> int:
    return int(_lib.sdtw_launch_count())


def release():
    _lib.sdtw_release()


class options:
    """Context manager: temporarily set ABI options, e.g. ``with options(OPT_FMA=0): ...``."""

    def __init__(self, **kw):
        self.kw = {globals()[k] if isinstance(k, str) else k: v for k, v in kw.items()}
        self.old = {}

    def __enter__(self):
        for k, v in self.kw.items():
            self.old[k] = get_option(k)
            set_option(k, v)
        return self

    def __exit__(self, *exc):
        for k, v in self.old.items():
            set_option(k, v)
        return False
