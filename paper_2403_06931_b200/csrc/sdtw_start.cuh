// sdtw_start.cuh -- the start index by round checkpoints and a windowed walk-back
// (VERDICT r01 item 4).
//
// The start column of reading G6 (forward propagation with priority diag > up > left) is
// the column where the paper's walk-back from (N-1, end) reaches row 0, provided
// the walk compares the EXACT D values (pinned: tests/test_oracle_pins.py
// test_walkback_equals_forward_start).  The cost/end DP already computes every exact D;
// the CKPT kernels additionally store the last column of every round (cpr = 32*C*G*WC
// reference columns).  So for a query with end e in round k:
//
//  1. window [j0, e] with j0 = k' * cpr for some k' <= k; its left boundary column
//     D(., j0 - 1) is the stored checkpoint of round k'-1 (exact), or +inf for j0 = 0;
//  2. window_dp_kernel recomputes the window from that boundary with the free start in
//     row 0 -- the DP kernel's cell arithmetic, so every window cell equals the full
//     DP's cell bit for bit (checked at (N-1, e) against the batch cost) -- and records
//     each cell's argmin predecessor (0 diag, 1 up, 2 left, priority in that order) as a
//     2-bit code, 16 per word;
//  3. window_walk_kernel walks the codes back from (N-1, e).  Reaching row 0 inside the
//     window gives the start column (identical to forward propagation, since the codes
//     come from the exact D values).  Leaving the window through its left boundary means
//     the chain starts further left: the host moves j0 back (doubling the window) and
//     repeats for those queries only.
//
// merge_ckpt_kernel first turns the speculative schedule's checkpoints into exact
// columns: inside the correction rounds of segment s the exact column is the cell-wise
// min of the free DP (A_s) and the correction (C_s) columns; after them it
// is the free column itself (the correction was overtaken).  Queries whose correction was
// not overtaken are recomputed by spec_fixup with one CTA per ring, which stores exact
// columns directly.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {

// ck[q][a_s + j][r] = min(ck[q][a_s + j][r], ckc[q][s-1][j][r]) for s >= 1, j < Rc, r < N,
// skipping queries marked for recomputation (fix[q] != 0).  grid (Sg-1, Z), block over rows.
static __global__ void merge_ckpt_kernel(float* ck, const float* __restrict__ ckc, const int* __restrict__ fix,
                                         int Pr, int Pd, int N, int Sg, int Rc) {
    const int s = blockIdx.x + 1, q = blockIdx.y;
    if (fix && fix[q]) return;
    const int a = (int)((int64_t)s * Pr / Sg);
    for (int j = 0; j < Rc; ++j) {
        float* dst = ck + ((int64_t)q * Pr + a + j) * Pd;
        const float* src = ckc + (((int64_t)q * (Sg - 1) + s - 1) * Rc + j) * Pd;
        for (int r = threadIdx.x; r < N; r += blockDim.x) dst[r] = fminf(dst[r], src[r]);
    }
}

struct WinParams {
    const float* X;          // [Z][N] normalised queries (the values the DP used)
    const float* Y;          // library reference (normalised), Malloc floats
    const float* cost;       // [Z] batch costs
    const int64_t* end;      // [Z] batch ends
    const float* ck;         // [Z][Pr][Pd] exact round checkpoints
    const int* qidx;         // [Zc] queries of this launch
    const int* k0;           // [Zc] first round of each query's window (j0 = k0 * cpr)
    int64_t cpr;             // reference columns per round
    int Pr, Pd, N;
    int W;                   // code words per row = ceil(Lmax / 16)
    int Lmax;
    uint32_t* codes;         // [Zc][N][W]
    float* rowbuf;           // [Zc][Lmax]
    int64_t* out_start;      // [Z]: the start column, or -1 (window too short)
    int32_t* path_lo;        // [Z][N] or nullptr: the warp path's first column per row
    int32_t* path_hi;        // [Z][N] or nullptr: last column per row
    int* err_flag;           // set to 2 on a recomputation mismatch
};

template <bool FMA>
__device__ __forceinline__ float win_cell(float x, float y, float m) {
    const float t = __fsub_rn(x, y);
    if (FMA) return __fmaf_rn(t, t, m);
    return __fadd_rn(__fmul_rn(t, t), m);
}

// One CTA per window: T threads own T consecutive query rows (a band) and sweep the
// window's anti-diagonals with one barrier per step (the path_dp_kernel scheme, from a
// checkpoint boundary instead of +inf).
template <bool FMA>
__global__ void __launch_bounds__(256) window_dp_kernel(const WinParams P) {
    extern __shared__ float pvals[];                 // [2][T]
    const int z = blockIdx.x;
    const int q = P.qidx[z];
    const int T = blockDim.x, k = threadIdx.x;
    const float c = P.cost[q];
    if (!(c < INFINITY)) return;
    const int64_t j0 = (int64_t)P.k0[z] * P.cpr;
    const int L = (int)(P.end[q] - j0 + 1);
    const int N = P.N;
    const float* xq = P.X + (int64_t)q * N;
    const float* yw = P.Y + j0;
    const float* bnd = P.k0[z] > 0 ? P.ck + ((int64_t)q * P.Pr + P.k0[z] - 1) * P.Pd : nullptr;
    uint32_t* cq = P.codes + (int64_t)z * N * P.W;
    float* rb = P.rowbuf + (int64_t)z * P.Lmax;
    const float INF = INFINITY;

    for (int band = 0; band * T < N; ++band) {
        const int i = band * T + k;
        const bool live = i < N;
        const float x = live ? xq[i] : 0.0f;
        // column j0 - 1: the checkpoint (exact) or +inf; row -1: the free start (0)
        float up_prev = (i == 0) ? 0.0f : (bnd && live ? bnd[i - 1] : INF);   // D(i-1, j0-1)
        float left = (bnd && live) ? bnd[i] : INF;                              // D(i, j0-1)
        uint32_t word = 0;
        const int steps = L + T - 1;
        for (int s = 0; s < steps; ++s) {
            const int j = s - k;
            float v = INF;
            if (live && j >= 0 && j < L) {
                float up;
                if (k == 0) up = (band == 0) ? 0.0f : rb[j];
                else up = pvals[((s - 1) & 1) * T + k - 1];
                const float diag = up_prev;
                const float m = fminf(fminf(diag, up), left);
                v = win_cell<FMA>(x, yw[j], m);
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
            if (k == T - 1 && live && j >= 0 && j < L) rb[j] = v;
            __syncthreads();
        }
        __syncthreads();
    }
}

// One thread per window: walk the codes back from (N-1, end).  Row 0 reached inside the
// window -> out_start[q] = its column (and the path rows, if requested); the left
// boundary crossed -> out_start[q] = -1 (the host widens the window).
__global__ void window_walk_kernel(const WinParams P, int Zc) {
    const int z = blockIdx.x * blockDim.x + threadIdx.x;
    if (z >= Zc) return;
    const int q = P.qidx[z];
    const int N = P.N;
    int32_t* lo = P.path_lo ? P.path_lo + (int64_t)q * N : nullptr;
    int32_t* hi = P.path_hi ? P.path_hi + (int64_t)q * N : nullptr;
    if (!(P.cost[q] < INFINITY)) {
        P.out_start[q] = 0;
        if (lo)
            for (int i = 0; i < N; ++i) lo[i] = hi[i] = -1;
        return;
    }
    const int64_t j0 = (int64_t)P.k0[z] * P.cpr;
    const uint32_t* cq = P.codes + (int64_t)z * N * P.W;
    int i = N - 1;
    int j = (int)(P.end[q] - j0);
    if (hi) hi[i] = (int32_t)(j0 + j);
    int wi = -1;
    uint32_t w = 0;
    while (i > 0) {
        if ((i * P.W + (j >> 4)) != wi) { wi = i * P.W + (j >> 4); w = cq[wi]; }
        const uint32_t code = (w >> (2 * (j & 15))) & 3u;
        if (code != 1u && j == 0) { P.out_start[q] = -1; return; }   // predecessor in column j0 - 1
        if (code == 0) {                  // diag
            if (lo) lo[i] = (int32_t)(j0 + j);
            --i; --j;
            if (hi) hi[i] = (int32_t)(j0 + j);
        } else if (code == 1) {           // up
            if (lo) lo[i] = (int32_t)(j0 + j);
            --i;
            if (hi) hi[i] = (int32_t)(j0 + j);
        } else {                          // left
            --j;
        }
    }
    // row 0: the free start (virtual row -1 = 0 is always the minimum, code diag)
    if (lo) lo[0] = (int32_t)(j0 + j);
    P.out_start[q] = j0 + j;
}

}  // namespace sdtw
