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

// First round a_s of speculative segment s of Sg (host plan spec_table() and this merge).
// Equal segments, except the two-segment plan: there the first segment takes 16/25 of the
// rounds.  Its chain A_0 -> B_0 -> C_1 carries the correction and should be the longer one;
// measured at the config-2 shape (512 x 2,000, Pr = 25..30 rounds, profiles/r02al-r02am, r02ar)
// the midpoint split ran at 6.7-7.4 TCUPS depending on Pr (equal B units leave a tail of
// late long units) and a 0.64 split at 7.3-7.6 everywhere.
__host__ __device__ inline int spec_seg_start(int s, int Pr, int Sg) {
    if (Sg == 2 && s == 1) return (int)((int64_t)Pr * 16 / 25);
    return (int)((int64_t)s * Pr / Sg);
}

// ck[q][a_s + j][r] = min(ck[q][a_s + j][r], ckc[q][s-1][j][r]) for s >= 1, j < Rc, r < N,
// skipping queries marked for recomputation (fix[q] != 0).  grid (Sg-1, Z), block over rows.
static __global__ void merge_ckpt_kernel(float* ck, const float* __restrict__ ckc, const int* __restrict__ fix,
                                         int Pr, int Pd, int N, int Sg, int Rc) {
    const int s = blockIdx.x + 1, q = blockIdx.y;
    if (fix && fix[q]) return;
    const int a = spec_seg_start(s, Pr, Sg);
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

// One CTA per window: T threads own T consecutive query rows (a band) and sweep the window
// in strips of WS columns: at step s thread k computes its row's columns [WS(s-k), WS(s-k)+WS)
// -- a strip whose up inputs thread k-1 produced at step s-1 (shared memory) -- so one
// barrier covers WS cells per thread (the path_dp_kernel scheme with WS = 1 needed one barrier
// and ~60 instructions per cell; ncu r02, config 5 N = 8,000).  Every cell is the DP kernel's
// cell from the checkpoint boundary (exact), and records its argmin predecessor as a 2-bit
// code (0 diag, 1 up, 2 left, priority in that order), 16 codes per word.
constexpr int kWinStrip = 8;
template <bool FMA>
__global__ void __launch_bounds__(256) window_dp_kernel(const WinParams P) {
    constexpr int WS = kWinStrip;
    extern __shared__ __align__(16) float pvals[];   // [2][T][WS]: the strips of the last two steps
    const int z = blockIdx.x;
    const int q = P.qidx[z];
    const int T = blockDim.x, k = threadIdx.x;
    const float c = P.cost[q];
    if (!(c < INFINITY)) return;
    const int64_t j0 = (int64_t)P.k0[z] * P.cpr;
    const int L = (int)(P.end[q] - j0 + 1);
    const int nst = (L + WS - 1) / WS;               // strips in the window
    const int N = P.N;
    const float* xq = P.X + (int64_t)q * N;
    const float* yw = P.Y + j0;
    const float* bnd = P.k0[z] > 0 ? P.ck + ((int64_t)q * P.Pr + P.k0[z] - 1) * P.Pd : nullptr;
    uint32_t* cq = P.codes + (int64_t)z * N * P.W;
    float* rb = P.rowbuf + (int64_t)z * P.Lmax;
    const float INF = INFINITY;

    // Rows wrap around the T threads: thread k owns rows k, k+T, k+2T, ... and spends P =
    // max(nst, T) steps per row (nst of them computing), so row k+T*r, strip js runs at step
    // k + r*P + js: its up strip (row - 1) was computed one step earlier by thread k-1 (shared
    // memory), or -- thread 0 -- at least one step earlier by thread T-1 of the previous cycle
    // (rb).  The threads stay busy across rows instead of draining after each band of T rows.
    const int Pp = max(nst, T);
    const int cycles = (N + T - 1) / T;
    const int steps = (T - 1) + cycles * Pp;
    int r = 0, js = -k;                              // this thread's cycle and strip at step s
    float up_prev = 0.0f, left = INF, x = 0.0f;
    uint32_t word = 0;
    for (int s = 0; s < steps; ++s) {
        const int i = r * T + k;
        float v[WS];
#pragma unroll
        for (int e = 0; e < WS; ++e) v[e] = INF;
        if (i < N && js >= 0 && js < nst) {
            if (js == 0) {                           // a new row: its sample and left boundary
                x = xq[i];
                // column j0 - 1: the checkpoint (exact) or +inf; row -1: the free start (0)
                up_prev = (i == 0) ? 0.0f : (bnd ? bnd[i - 1] : INF);   // D(i-1, j0-1)
                left = bnd ? bnd[i] : INF;                              // D(i, j0-1)
                word = 0;
            }
            const int jb = js * WS;
            float up[WS];
            if (k == 0) {
#pragma unroll
                for (int e = 0; e < WS; ++e) up[e] = (i == 0) ? 0.0f : (jb + e < L ? rb[jb + e] : INF);
            } else {
                const float4* pv = reinterpret_cast<const float4*>(pvals + (((s - 1) & 1) * T + k - 1) * WS);
#pragma unroll
                for (int e = 0; e < WS / 4; ++e) {
                    const float4 t4 = pv[e];
                    up[4 * e] = t4.x; up[4 * e + 1] = t4.y; up[4 * e + 2] = t4.z; up[4 * e + 3] = t4.w;
                }
            }
            const bool full = jb + WS <= L;          // every strip but possibly the last
            float yv[WS];
            if (full) {                              // yw is 16-byte aligned (j0 is a round start)
                const float4* y4 = reinterpret_cast<const float4*>(yw + jb);
#pragma unroll
                for (int e = 0; e < WS / 4; ++e) {
                    const float4 t4 = __ldg(y4 + e);
                    yv[4 * e] = t4.x; yv[4 * e + 1] = t4.y; yv[4 * e + 2] = t4.z; yv[4 * e + 3] = t4.w;
                }
            } else {
#pragma unroll
                for (int e = 0; e < WS; ++e) yv[e] = jb + e < L ? yw[jb + e] : 0.0f;
            }
            uint32_t half = 0;                       // this strip's WS codes (2 bits each)
#pragma unroll
            for (int e = 0; e < WS; ++e) {
                if (full || jb + e < L) {
                    const float diag = (e == 0) ? up_prev : up[e - 1];
                    const float m = fminf(fminf(diag, up[e]), left);
                    v[e] = win_cell<FMA>(x, yv[e], m);
                    const uint32_t code = (diag == m) ? 0u : ((up[e] == m) ? 1u : 2u);
                    half |= code << (2 * e);
                    left = v[e];
                }
            }
            // 16 codes per word = two strips: the even strip starts the word, the odd one
            // completes and stores it (or the last strip stores what it has)
            static_assert(WS == 8, "two strips per 16-code word");
            if ((js & 1) == 0) word = half;
            else word |= half << 16;
            if ((js & 1) == 1 || js == nst - 1) cq[(int64_t)i * P.W + (jb >> 4)] = word;
            if (i == N - 1 && js == nst - 1) {      // the window reproduces the batch cost
#pragma unroll
                for (int e = 0; e < WS; ++e)
                    if (jb + e == L - 1 && v[e] != c) atomicExch(P.err_flag, 2);
            }
            up_prev = up[WS - 1];
            if (k == T - 1) {                        // the next cycle's thread 0 reads this row
#pragma unroll
                for (int e = 0; e < WS; ++e)
                    if (jb + e < L) rb[jb + e] = v[e];
            }
        }
        float* pw = pvals + ((s & 1) * T + k) * WS;
#pragma unroll
        for (int e = 0; e < WS; ++e) pw[e] = v[e];
        __syncthreads();
        if (++js == Pp) { js = 0; ++r; }
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
