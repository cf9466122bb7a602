// sdtw_path.cuh -- full warp path of each query's optimal match (SURVEY.md §8(f)
// NEXT-2; the paper's walk-back), on top of sdtw_traceback's
// (cost, end, start).
//
// Reduction (pinned on the oracle by tests/test_path_oracle.py::test_path_window_reduction):
// the path of the argmin chain lies in reference columns [start, end]; the DP restricted
// to that window (free start in row 0, +inf left edge) gives every neighbour of a path
// cell a value >= its full-DP value, with equality along the chain, so the tie rule
// (diag > up > left) picks the same predecessor at every path cell.  Two kernels:
//
//  * path_dp_kernel  -- one CTA per query: the window DP, T = blockDim threads own T
//    consecutive query rows (a band), an anti-diagonal sweep over the window columns
//    with one barrier per step; each cell's predecessor code (0 diag, 1 up, 2 left) is
//    packed 16 per 32-bit word.  Bands run top to bottom; the last row of a band is
//    handed to the next through a global row buffer.  The cell arithmetic is the DP
//    kernel's (t = x - y, fma(t,t,m) or fl(fl(t*t)+m)), so D(N-1, end) must reproduce
//    the batch cost bit for bit -- checked, a mismatch raises the error flag.
//  * path_walk_kernel -- one thread per query walks the codes back from (N-1, end) and
//    writes, per row i, the first and last column the path visits (path_lo, path_hi).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {

struct PathParams {
    const float* X;          // [Zc][N] queries of this chunk (same values the DP used)
    const float* Y;          // reference (normalised), Malloc floats
    const float* cost;       // [Zc] batch costs
    const int64_t* start;    // [Zc]
    const int64_t* end;      // [Zc]
    int N;
    int W;                   // code words per row = ceil(Lmax / 16)
    int Lmax;
    uint32_t* codes;         // [Zc][N][W]
    float* rowbuf;           // [Zc][Lmax] last row of the previous band
    int32_t* path_lo;        // [Zc][N]
    int32_t* path_hi;        // [Zc][N]
    int* err_flag;           // set to 2 on a recomputation mismatch
};

template <bool FMA>
__device__ __forceinline__ float path_cell(float x, float y, float m) {
    const float t = __fsub_rn(x, y);
    if (FMA) return __fmaf_rn(t, t, m);
    return __fadd_rn(__fmul_rn(t, t), m);
}

template <bool FMA>
__global__ void __launch_bounds__(256) path_dp_kernel(const PathParams P) {
    extern __shared__ float pvals[];                 // [2][T]: each thread's value of the last two steps
    const int q = blockIdx.x;
    const int T = blockDim.x, k = threadIdx.x;
    const float c = P.cost[q];
    if (!(c < INFINITY)) return;                     // no path (raw-mode overflow)
    const int64_t j0 = P.start[q];
    const int L = (int)(P.end[q] - j0 + 1);
    const int N = P.N;
    const float* xq = P.X + (int64_t)q * N;
    const float* yw = P.Y + j0;
    uint32_t* cq = P.codes + (int64_t)q * N * P.W;
    float* rb = P.rowbuf + (int64_t)q * P.Lmax;
    const float INF = INFINITY;

    for (int band = 0; band * T < N; ++band) {
        const int i = band * T + k;
        const bool live = i < N;
        const float x = live ? xq[i] : 0.0f;
        float up_prev = (i == 0) ? 0.0f : INF;       // D(i-1, j-1) for j = 0: virtual row / +inf edge
        float left = INF;                            // D(i, -1) = +inf
        uint32_t word = 0;
        const int steps = L + T - 1;
        for (int s = 0; s < steps; ++s) {
            const int j = s - k;
            float v = INF;
            if (live && j >= 0 && j < L) {
                float up;
                if (k == 0) up = (band == 0) ? 0.0f : rb[j];      // row above the band
                else up = pvals[((s - 1) & 1) * T + k - 1];        // thread k-1, step s-1
                const float diag = up_prev;
                const float m = fminf(fminf(diag, up), left);
                v = path_cell<FMA>(x, yw[j], m);
                const uint32_t code = (diag == m) ? 0u : ((up == m) ? 1u : 2u);
                word |= code << (2 * (j & 15));
                if ((j & 15) == 15 || j == L - 1) {
                    cq[(int64_t)i * P.W + (j >> 4)] = word;
                    word = 0;
                }
                up_prev = up;
                left = v;
                if (i == N - 1 && j == L - 1 && v != c) atomicExch(P.err_flag, 2);
            }
            pvals[(s & 1) * T + k] = v;
            if (k == T - 1 && live && j >= 0 && j < L) rb[j] = v;   // for the next band (read later)
            __syncthreads();
        }
        __syncthreads();
    }
}

__global__ void path_walk_kernel(const PathParams P, int Zc) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Zc) return;
    const int N = P.N;
    int32_t* lo = P.path_lo + (int64_t)q * N;
    int32_t* hi = P.path_hi + (int64_t)q * N;
    if (!(P.cost[q] < INFINITY)) {
        for (int i = 0; i < N; ++i) lo[i] = hi[i] = -1;
        return;
    }
    const int64_t j0 = P.start[q];
    const uint32_t* cq = P.codes + (int64_t)q * N * P.W;
    int i = N - 1;
    int j = (int)(P.end[q] - j0);
    hi[i] = (int32_t)(j0 + j);
    int wi = -1;
    uint32_t w = 0;
    while (i > 0) {
        if ((i * P.W + (j >> 4)) != wi) { wi = i * P.W + (j >> 4); w = cq[wi]; }
        const uint32_t code = (w >> (2 * (j & 15))) & 3u;
        if (code == 0) {                  // diag
            lo[i] = (int32_t)(j0 + j);
            --i; --j;
            hi[i] = (int32_t)(j0 + j);
        } else if (code == 1) {           // up
            lo[i] = (int32_t)(j0 + j);
            --i;
            hi[i] = (int32_t)(j0 + j);
        } else {                          // left
            --j;
        }
        if (j < 0) { atomicExch(P.err_flag, 2); return; }
    }
    lo[0] = (int32_t)(j0 + j);
    if (j != 0) atomicExch(P.err_flag, 2);        // the chain must start at the window's first column
}

}  // namespace sdtw
