"""ctypes binding of the CPU oracle (oracle/sdtw_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / ``--impl reference`` legs of bench.py -- never by the product
package ``paper_2403_06931_b200``. It shares no code with the CUDA path.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "sdtw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
CFLAGS = ["-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-pthread"]

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (no FP contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + ".tmp%d" % os.getpid()
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        f32p = ctypes.POINTER(ctypes.c_float)
        i64p = ctypes.POINTER(ctypes.c_int64)
        i64 = ctypes.c_int64
        L.oracle_sdtw.argtypes = [f32p, i64, i64, f32p, i64, ctypes.c_int, f32p, i64p, i64p, f32p, ctypes.c_int]
        L.oracle_sdtw.restype = ctypes.c_int
        L.oracle_sdtw_full.argtypes = [f32p, i64, f32p, i64, ctypes.c_int, f32p, i64p]
        L.oracle_sdtw_full.restype = ctypes.c_int
        L.oracle_walkback.argtypes = [f32p, i64, i64, i64]
        L.oracle_walkback.restype = i64
        L.oracle_walkback_path.argtypes = [f32p, i64, i64, i64, i64p, i64p]
        L.oracle_walkback_path.restype = ctypes.c_int
        u8p = ctypes.POINTER(ctypes.c_uint8)
        L.oracle_sdtw_q8.argtypes = [u8p, i64, i64, u8p, i64, ctypes.c_int, i64p, i64p]
        L.oracle_sdtw_q8.restype = ctypes.c_int
        L.oracle_round_half.argtypes = [ctypes.c_double, ctypes.c_double]
        L.oracle_round_half.restype = ctypes.c_float
        _lib = L
    return _lib


def _f32(a):
    a = np.ascontiguousarray(a, dtype=np.float32)
    return a, a.ctypes.data_as(ctypes.POINTER(ctypes.c_float))


def _i64(a):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))


def sdtw(Q, Y, fma: bool = True, start: bool = False, last_rows: bool = False,
         threads: int | None = None, half: bool = False):
    """Batched sDTW on raw inputs (no normalisation). Q: [Z,N] or [N]; Y: [M].
    half=True: the packed-half recurrence (inputs rounded to binary16, every op rounded).

    Returns dict(cost[Z] f32, end[Z] i64, start[Z] i64 | None, last_rows[Z,M] | None)."""
    Q = np.asarray(Q, dtype=np.float32)
    if Q.ndim == 1:
        Q = Q[None, :]
    Z, N = Q.shape
    Qc, qp = _f32(Q)
    Yc, yp = _f32(Y)
    M = Yc.shape[0]
    cost = np.empty(Z, np.float32)
    end = np.empty(Z, np.int64)
    st = np.empty(Z, np.int64) if start else None
    lr = np.empty((Z, M), np.float32) if last_rows else None
    if threads is None:
        threads = os.cpu_count() or 1
    rc = lib().oracle_sdtw(qp, Z, N, yp, M, 2 if half else int(bool(fma)),
                           cost.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), _i64(end),
                           _i64(st) if st is not None else None,
                           lr.ctypes.data_as(ctypes.POINTER(ctypes.c_float)) if lr is not None else None,
                           int(threads))
    if rc != 0:
        raise ValueError("oracle_sdtw: bad arguments")
    return dict(cost=cost, end=end, start=st, last_rows=lr)


def sdtw_full(x, Y, fma: bool = True):
    """Full D and S matrices (N x M) for one query -- small instances only."""
    xc, xp = _f32(x)
    Yc, yp = _f32(Y)
    N, M = xc.shape[0], Yc.shape[0]
    D = np.empty((N, M), np.float32)
    S = np.empty((N, M), np.int64)
    rc = lib().oracle_sdtw_full(xp, N, yp, M, int(bool(fma)),
                                D.ctypes.data_as(ctypes.POINTER(ctypes.c_float)), _i64(S))
    if rc != 0:
        raise ValueError("oracle_sdtw_full: bad arguments")
    return D, S


def walkback(D, end: int) -> int:
    Dc, dp = _f32(D)
    N, M = Dc.shape
    return int(lib().oracle_walkback(dp, N, M, int(end)))


def round_half(v: float, err: float = 0.0) -> float:
    """binary16 round-to-nearest-even of v (+ an exact residual err), as a float."""
    return float(lib().oracle_round_half(float(v), float(err)))


def walkback_path(D, end: int):
    """Full warp path of the walk-back from (N-1, end): per row i the first and last
    column visited, (lo[N], hi[N]) int64."""
    Dc, dp = _f32(D)
    N, M = Dc.shape
    lo = np.empty(N, np.int64)
    hi = np.empty(N, np.int64)
    if lib().oracle_walkback_path(dp, N, M, int(end), _i64(lo), _i64(hi)) != 0:
        raise ValueError("oracle_walkback_path: bad arguments")
    return lo, hi


def sdtw_path(x, Y, fma: bool = True):
    """(cost, end, start, lo, hi) of one query from the full matrices -- small instances."""
    D, S = sdtw_full(x, Y, fma)
    last = D[-1]
    cost = last.min()
    end = int(np.flatnonzero(last == cost)[0])
    lo, hi = walkback_path(D, end)
    return np.float32(cost), end, int(S[-1, end]), lo, hi


def znorm(X):
    """Per-series z-normalisation, §5.1 Eq. 2 with the statistics of the
    quoted code: mean = sum/n, var = sumSq/n - mean^2 (population, reading
    G7), S = sqrt(var), z = (x - mean)/S rounded once to fp32.  Reading G8: sum and sumSq
    are the EXACT sums of the fp32 samples, each rounded once to fp64 (math.fsum is the
    library's exactly rounded sum; x*x is exact in fp64 for an fp32 x), so the result does
    not depend on any summation order.  Reading G9: var <= 1e-12*E[x^2] or sumSq == 0 ->
    all zeros.  Every fp64 operation below is one IEEE-rounded numpy/Python operation."""
    X = np.asarray(X, dtype=np.float32)
    shape = X.shape
    if X.ndim == 1:
        X = X[None, :]
    n_series, n = X.shape
    if n < 1:
        raise ValueError("znorm: series length must be >= 1")
    out = np.empty((n_series, n), np.float32)
    for q in range(n_series):
        x = X[q].astype(np.float64)
        s = math.fsum(x)
        sumsq = math.fsum(x * x)
        mean = s / n
        ex2 = sumsq / n
        var = ex2 - mean * mean
        if sumsq == 0.0 or var <= 1e-12 * ex2:
            out[q] = 0.0
            continue
        sd = math.sqrt(var)
        out[q] = ((x - mean) / sd).astype(np.float32)
    return out.reshape(shape)


def sdtw_normalized(Q, Y, fma: bool = True, start: bool = False, threads: int | None = None):
    """End-to-end oracle: z-normalise reference (globally) and each query, then sDTW
    (§5: runSDTW normalises both the reference and the batch)."""
    Yn = znorm(np.asarray(Y, np.float32)[None, :])[0]
    Qn = znorm(Q)
    return sdtw(Qn, Yn, fma=fma, start=start, threads=threads)


# ----------------------------------------------------------------------------------------
# uint8 codebook (§Discussion)
Q8_INF = 1 << 30


def codebook(Y, clip_ppm: int = 1000):
    """The reference codebook: "get the distribution of floating point values and
    then evenly divide the bulk of the distribution across uint8 values clamping any
    outliers to the extreme values".  Reading G18: the bulk is [lo, hi] with lo / hi the
    order statistics (0-based ranks in the sorted samples) k and M-1-k,
    k = floor(clip_ppm * (M-1) / 10^6) (integer arithmetic).  Returns (lo, hi) as fp32."""
    y = np.sort(np.asarray(Y, np.float32).ravel(), kind="stable")
    M = y.shape[0]
    k = (int(clip_ppm) * (M - 1)) // 1_000_000
    return np.float32(y[k]), np.float32(y[M - 1 - k])


def quantize(v, lo, hi):
    """uint8 codes (reading G19): "evenly divide" = 256 equal-width levels over [lo, hi],
    code = clamp(floor((v - lo) * (255 / (hi - lo)) + 0.5), 0, 255) with every operation
    one IEEE fp64 rounding (numpy evaluates the expression one operation at a time, no
    contraction); hi == lo -> all codes 0."""
    v = np.asarray(v, np.float32)
    lo64, hi64 = np.float64(np.float32(lo)), np.float64(np.float32(hi))
    if not hi64 > lo64:
        return np.zeros(v.shape, np.uint8)
    s = np.float64(255.0) / (hi64 - lo64)
    u = (v.astype(np.float64) - lo64) * s + np.float64(0.5)
    return np.clip(np.floor(u), 0.0, 255.0).astype(np.uint8)


def sdtw_q8(Qc, Yc, tau: int = -1):
    """Batched sDTW over uint8 codes (oracle_sdtw_q8 in sdtw_oracle.c): exact integer costs
    (int64; Q8_INF = every path pruned) and the smallest argmin end.  tau < 0: no pruning."""
    Qc = np.ascontiguousarray(Qc, dtype=np.uint8)
    if Qc.ndim == 1:
        Qc = Qc[None, :]
    Yc = np.ascontiguousarray(Yc, dtype=np.uint8)
    Z, N = Qc.shape
    M = Yc.shape[0]
    cost = np.empty(Z, np.int64)
    end = np.empty(Z, np.int64)
    u8p = ctypes.POINTER(ctypes.c_uint8)
    rc = lib().oracle_sdtw_q8(Qc.ctypes.data_as(u8p), Z, N, Yc.ctypes.data_as(u8p), M, int(tau), _i64(cost), _i64(end))
    if rc != 0:
        raise ValueError("oracle_sdtw_q8: bad arguments")
    return dict(cost=cost, end=end)


def sdtw_q8_normalized(Q, Y, tau: int = -1, clip_ppm: int = 1000, normalize: bool = True):
    """End-to-end uint8 oracle: z-normalise (as sdtw_normalized), codebook of the reference,
    code both sides, integer DP.  Returns dict(cost, end, lo, hi, Qc, Yc)."""
    Yn = znorm(np.asarray(Y, np.float32)[None, :])[0] if normalize else np.asarray(Y, np.float32)
    Qn = znorm(Q) if normalize else np.asarray(Q, np.float32)
    lo, hi = codebook(Yn, clip_ppm)
    Yc = quantize(Yn, lo, hi)
    Qc = quantize(Qn, lo, hi)
    r = sdtw_q8(Qc, Yc, tau)
    r.update(lo=lo, hi=hi, Qc=Qc, Yc=Yc)
    return r
