// sdtw_dp.cuh -- the anti-diagonal wavefront DP kernel (sm_100a).
//
// Computes, per query, the sDTW recurrence of PAPER.md §2 Eq. 1
//     D(i,j) = (x_i - y_j)^2 + min{D(i-1,j-1), D(i-1,j), D(i,j-1)}
// with virtual row -1 = 0 (free start) and virtual column -1 = +inf, and folds
// the last row into (cost, smallest argmin column) -- P:L35.
//
// Mapping (B200 re-design of the paper's segment-per-thread scheme):
//  * A query is processed by a RING of G = GW*CL warps (GW warps per CTA, CL CTAs
//    in a thread-block cluster).  Each physical lane carries C "chains"; chain c of
//    lane l of ring warp g is virtual lane u = C*(32g+l)+c.  There are V = 32*C*G
//    virtual lanes; virtual lane u owns a strip of WC reference columns per round
//    (the paper's "segment"), round p covering strips p*V .. p*V+V-1.
//  * Virtual lane u processes band b = t-u at global step t (row r = b mod Pd of
//    round p = b div Pd; Pd >= N is the round period, rows >= N are idle).  So
//    each step is one anti-diagonal of virtual lanes.
//  * Strip state lives in registers: D[w] holds the previous row of the strip and
//    is updated in place with a rolling diag (the paper's two row buffers).
//  * Right-edge hand-off: chain c -> chain c+1 in the same lane is a register; the
//    last chain -> next lane by SHFL.UP ("__shfl_up"); lane 31 -> next warp
//    through a shared-memory ring (DSMEM when the next warp is in another CTA of
//    the cluster) with release/acquire progress counters checked every K steps;
//    the last virtual lane -> virtual lane 0 of the next round through the
//    Pd-entry boundary ring (the paper's "shared memory buffer which represents the
//    last segment values").
//  * C == 2 packs the two chains of a lane into f32x2 FADD2/FFMA2 (sm_100a):
//    per 2 cells FADD2 + FFMA2 + 2 FMNMX3 = 2 SASS/cell instead of 3.
//  * TRACE carries, per cell, the start column of its argmin predecessor
//    (priority diag > up > left on equality; reading G6).
#pragma once
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace sdtw {
namespace cg = cooperative_groups;

struct DpParams {
    const float* X;        // [Z][N] query samples (normalised or raw), device
    const float* Y;        // reference, device, Malloc floats (+inf beyond M)
    int Malloc;            // padded reference length (multiple of 4)
    int Z, N, M;
    int Pd;                // round period in steps (>= N)
    int Pr;                // number of rounds
    int K;                 // steps per hand-off chunk (divides 32*C)
    int RS;                // inter-warp ring entries (power of two, >= 4K)
    float* out_cost;
    int64_t* out_end;
    int64_t* out_start;    // TRACE only
    const int* err_flag;   // nonzero -> write no results
};

template <bool TRACE> struct Entry { float d; };
template <> struct Entry<true> { float d; int s; };

__device__ __forceinline__ void st_release_cluster(int* p, int v) {
    asm volatile("st.release.cluster.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
    int v;
    asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
// Wait until *p >= need.  A watchdog turns a protocol bug into a diagnosable trap
// instead of a hung GPU (never reached in a correct run: every wait is bounded by
// the ring's progress).
__device__ __noinline__ void spin_slow(const int* p, int need, int tag) {
    long long n = 0;
    int v;
    while ((v = ld_acquire_cluster(p)) < need) {
        __nanosleep(32);
        if (++n == (1LL << 25)) {
            printf("sdtw watchdog: block %d thread %d tag %d waits *p=%d >= %d\n", (int)blockIdx.x,
                   (int)threadIdx.x, tag, v, need);
            __trap();
        }
    }
}
__device__ __forceinline__ void spin_until_geq(const int* p, int need, int tag = 0) {
    if (ld_acquire_cluster(p) >= need) return;
    spin_slow(p, need, tag);
}

__device__ __forceinline__ unsigned long long pk2(float2 a) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a.x), "f"(a.y));
    return r;
}
__device__ __forceinline__ float2 upk2(unsigned long long r) {
    float2 a;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(r));
    return a;
}
// t = a - b, two lanes, one FADD2 (round-to-nearest, same as two scalar FADD)
__device__ __forceinline__ float2 sub2(float2 a, float2 b) {
    unsigned long long r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)));
    return upk2(r);
}
// a*b + c, two lanes, one FFMA2 (single rounding each, same as fmaf)
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) {
    unsigned long long r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(pk2(a)), "l"(pk2(b)), "l"(pk2(c)));
    return upk2(r);
}

__device__ __forceinline__ float min3f(float a, float b, float c) { return fminf(fminf(a, b), c); }

// fp32 cell value d(x,y) + m (the oracle's `cell`, scalar)
template <bool FMA>
__device__ __forceinline__ float cell1(float x, float y, float m) {
    float t = __fsub_rn(x, y);
    if (FMA) return __fmaf_rn(t, t, m);
    return __fadd_rn(__fmul_rn(t, t), m);
}

// lexicographic (cost, col) "a better than b"
__device__ __forceinline__ bool better(float ca, int ja, float cb, int jb) {
    return ca < cb || (ca == cb && ja < jb);
}

// Load the WC reference samples of strip `strip` (+inf outside [0, Malloc)).
template <int WC>
__device__ __forceinline__ void load_strip(const float* __restrict__ Y, int Malloc, long strip,
                                           float (&y)[WC]) {
    const long col0 = strip * WC;
#pragma unroll
    for (int k = 0; k < WC / 4; ++k) {
        const long c = col0 + 4 * k;
        float4 v;
        if (c + 4 <= (long)Malloc) {
            v = __ldg(reinterpret_cast<const float4*>(Y + c));
        } else {
            v = make_float4(INFINITY, INFINITY, INFINITY, INFINITY);
        }
        y[4 * k + 0] = v.x;
        y[4 * k + 1] = v.y;
        y[4 * k + 2] = v.z;
        y[4 * k + 3] = v.w;
    }
}

// Shared-memory carve-up (dynamic).  Returns total bytes.
struct SmemLayout {
    int off_ctr, off_red, off_x, off_bnd, off_ring, bytes;
};
__host__ __device__ inline SmemLayout smem_layout(int C, bool trace, int GW, int CL, int Pd, int RS) {
    SmemLayout L;
    const int ent = trace ? 8 : 4;
    int o = 0;
    L.off_ctr = o;  o += 2 * 32 * 4;                   // pp[32], cp[32]
    L.off_red = o;  o += 16 * (32 + 16);               // per-warp + per-rank partials
    o = (o + 15) & ~15;
    L.off_x = o;    o += Pd * C * 4;
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * ent;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * ent;
    L.bytes = (o + 15) & ~15;
    (void)CL;
    return L;
}

struct Partial { float cost; int col; int start; int pad; };

// Register strip of one lane: C chains x WC columns of D (previous row) and y.
// C == 2 keeps (chain0, chain1) pairs in aligned 64-bit registers so that FADD2 /
// FFMA2 read and write them in place (no pair-building moves in the hot loop).
template <int C, int WC> struct Strip;
template <int WC> struct Strip<1, WC> {
    float D[WC], Y[WC];
    __device__ __forceinline__ float d(int, int w) const { return D[w]; }
    __device__ __forceinline__ void set_d(int, int w, float v) { D[w] = v; }
    __device__ __forceinline__ void set_y(int, int w, float v) { Y[w] = v; }
};
__device__ __forceinline__ float lo32(unsigned long long r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return a;
}
__device__ __forceinline__ float hi32(unsigned long long r) {
    float a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
    return b;
}
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
template <int WC> struct Strip<2, WC> {
    unsigned long long D[WC], Y[WC];
    __device__ __forceinline__ float d(int c, int w) const { return c ? hi32(D[w]) : lo32(D[w]); }
    __device__ __forceinline__ void set_d(int c, int w, float v) {
        D[w] = c ? pk(lo32(D[w]), v) : pk(v, hi32(D[w]));
    }
    __device__ __forceinline__ void set_y(int c, int w, float v) {
        Y[w] = c ? pk(lo32(Y[w]), v) : pk(v, hi32(Y[w]));
    }
};

// New strip for chain c (round transition): reload y, virtual row -1 = 0.
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void enter_strip(Strip<C, WC>& st, int (&S)[TRACE ? C : 1][TRACE ? WC : 1],
                                            int c, long strip, bool live, const DpParams& P,
                                            float& prevleft, int& prevleft_s) {
    float y[WC];
    if (live) load_strip<WC>(P.Y, P.Malloc, strip, y);
    else {
#pragma unroll
        for (int w = 0; w < WC; ++w) y[w] = INFINITY;
    }
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        st.set_y(c, w, y[w]);
        st.set_d(c, w, 0.0f);
        if constexpr (TRACE) S[c][w] = (int)(strip * WC) + w + 1;   // S(-1, j) = j+1
    }
    prevleft = 0.0f;                    // D(-1, col0-1) = 0
    prevleft_s = (int)(strip * WC);     // so that row 0 gets S = j
}

template <int C, int WC, bool TRACE>
__device__ __forceinline__ void fold_last_row(const Strip<C, WC>& st, const int (&S)[TRACE ? C : 1][TRACE ? WC : 1],
                                              int c, int col0, float& best, int& bestcol, int& beststart) {
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const float v = st.d(c, w);
        if (v < best) {
            best = v;
            bestcol = col0 + w;
            if constexpr (TRACE) beststart = S[c][w];
        }
    }
}

template <int C, int WC, bool FMA, bool TRACE>
__global__ void __launch_bounds__(256) sdtw_dp_kernel(const DpParams P) {
    static_assert(C == 1 || C == 2, "C");
    static_assert(WC % 4 == 0, "WC");
    extern __shared__ __align__(16) unsigned char smem[];
    using E = Entry<TRACE>;

    cg::cluster_group cluster = cg::this_cluster();
    const int CL = (int)cluster.num_blocks();
    const int rank = (int)cluster.block_rank();
    const int q = blockIdx.x / CL;
    const int GW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = GW * CL;
    const int gw = rank * GW + warp;
    const int V = 32 * C * G;
    const int Pd = P.Pd, N = P.N, K = P.K, RS = P.RS;
    const SmemLayout L = smem_layout(C, TRACE, GW, CL, Pd, RS);

    int* pp = reinterpret_cast<int*>(smem + L.off_ctr);        // producer progress seen by warp w
    int* cp = pp + 32;                                          // consumer progress of w's successor
    float* xs = reinterpret_cast<float*>(smem + L.off_x);
    E* bnd = reinterpret_cast<E*>(smem + L.off_bnd);
    E* ring = reinterpret_cast<E*>(smem + L.off_ring);
    Partial* red = reinterpret_cast<Partial*>(smem + L.off_red);

    // ---- prologue: query -> smem (pairs (x_r, x_{r-1 mod Pd}) when C == 2), rings, counters
    const float* xq = P.X + (long)q * N;
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        const float a = (r < N) ? xq[r] : 0.0f;
        if (C == 2) {
            const int rp = (r == 0) ? Pd - 1 : r - 1;
            const float b = (rp < N) ? xq[rp] : 0.0f;
            reinterpret_cast<float2*>(xs)[r] = make_float2(a, b);
        } else {
            xs[r] = a;
        }
        E e;
        e.d = INFINITY;
        if constexpr (TRACE) e.s = 0;
        bnd[r] = e;
    }
    if (threadIdx.x < 32) {
        pp[threadIdx.x] = 0;
        const int g = rank * GW + threadIdx.x;   // successor of local warp threadIdx.x starts at 32C(g+1)
        cp[threadIdx.x] = 32 * C * (g + 1);
    }
    cluster.sync();

    // ---- neighbours in the ring
    const bool has_succ_ring = (gw < G - 1);      // successor is a ring warp (else: the wrap)
    E* succ_ring;
    int* succ_pp;
    if (has_succ_ring) {
        if (warp < GW - 1) {
            succ_ring = ring + (warp + 1) * RS;
            succ_pp = pp + warp + 1;
        } else {
            succ_ring = cluster.map_shared_rank(ring, rank + 1);
            succ_pp = cluster.map_shared_rank(pp, rank + 1);
        }
    } else {
        succ_ring = cluster.map_shared_rank(bnd, 0);         // boundary ring of rank 0
        succ_pp = cluster.map_shared_rank(pp, 0);            // pp[0] of rank 0
    }
    int* pred_cp = nullptr;                                   // where we report consumption
    if (gw > 0) pred_cp = (warp > 0) ? cp + warp - 1 : cluster.map_shared_rank(cp + GW - 1, rank - 1);
    const E* my_in = (gw == 0) ? bnd : ring + warp * RS;
    const int u0 = C * (32 * gw + lane);
    const int u_last = V - 1;
    const int Mtot_bands = P.Pr * Pd;

    // ---- per-lane state
    Strip<C, WC> st;
    int S[TRACE ? C : 1][TRACE ? WC : 1];
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int w = 0; w < WC; ++w) {
            st.set_d(c, w, INFINITY);
            st.set_y(c, w, INFINITY);
            if constexpr (TRACE) S[c][w] = 0;
        }
    float prevleft[C];
    int prevleft_s[C];
    float best[C];
    int bestcol[C], beststart[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        prevleft[c] = INFINITY; prevleft_s[c] = 0;
        best[c] = INFINITY; bestcol[c] = 0x7fffffff; beststart[c] = 0;
    }
    float outv = INFINITY;    // right edge of the lane's last chain (to lane+1 / next warp)
    int outs = 0;
    float right0 = INFINITY;  // C == 2: chain 0 right edge -> chain 1 left at the next step
    int right0_s = 0;

    // band of chain 0 at this warp's first step t = 32*C*gw
    int b0 = -C * lane;
    int p0 = (b0 < 0) ? -1 : 0;
    int r0 = (b0 < 0) ? b0 + Pd : 0;

    // warp g runs steps [32*C*g, 32*C*g + span): its lanes' bands cover [0, Pr*Pd)
    const int span = (32 * C - 1 + Mtot_bands + K - 1) / K * K;
    const int t_begin = 32 * C * gw;
    const int t_end = t_begin + span;
    // a predecessor never publishes past its own end: the successor's trailing
    // (idle-band) chunks must not wait for more
    const int pred_end = t_end - 32 * C;                 // = t_end of warp gw-1
    const int last_end = 32 * C * (G - 1) + span;        // = t_end of warp G-1
    const unsigned FULL = 0xffffffffu;

    for (int t0 = t_begin; t0 < t_end; t0 += K) {
        // ---- chunk-level flow control (one lane each), then converge
        if (lane == 0) {
            if (gw > 0) spin_until_geq(pp + warp, min(t0 + K - 1, pred_end), 1);
            else if (t0 + K - 1 >= Pd) spin_until_geq(pp, min(t0 + K - Pd + u_last, last_end), 2);
        }
        if (lane == 31 && has_succ_ring) spin_until_geq(cp + warp, t0 + K - RS + 1, 3);
        __syncwarp();

#pragma unroll 1
        for (int s = 0; s < K; ++s) {
            const int t = t0 + s;
            // ---- left input of chain 0: previous lane's last chain (SHFL.UP), lane 0: inbox
            float lin = __shfl_up_sync(FULL, outv, 1);
            int lins = 0;
            if constexpr (TRACE) lins = __shfl_up_sync(FULL, outs, 1);
            if (lane == 0) {
                E e;
                if (gw == 0) {
                    if (p0 >= 1) e = my_in[r0];
                    else { e.d = INFINITY; if constexpr (TRACE) e.s = 0; }
                } else {
                    e = my_in[t & (RS - 1)];
                }
                lin = e.d;
                if constexpr (TRACE) lins = e.s;
            }
            const int r1 = (r0 == 0) ? Pd - 1 : r0 - 1;   // chain 1 row
            const int p1 = (r0 == 0) ? p0 - 1 : p0;       // chain 1 round

            // ---- round transitions (new strip: virtual row -1 = 0, reload y)
            if (r0 == 0) {
                const long strip = (long)p0 * V + u0;
                enter_strip<C, WC, TRACE>(st, S, 0, strip, p0 < P.Pr, P, prevleft[0], prevleft_s[0]);
            }
            if (C == 2 && r1 == 0) {
                const long strip = (long)p1 * V + u0 + 1;
                enter_strip<C, WC, TRACE>(st, S, C - 1, strip, p1 < P.Pr, P, prevleft[C - 1], prevleft_s[C - 1]);
            }

            // ---- the cells (Eq. 1)
            if constexpr (C == 1) {
                const float xv = xs[r0];
                float left = lin, diag = prevleft[0];
                int sl = lins, sd = prevleft_s[0];
                prevleft[0] = lin;
                prevleft_s[0] = lins;
#pragma unroll
                for (int w = 0; w < WC; ++w) {
                    const float up = st.D[w];
                    const float m = min3f(diag, up, left);
                    const float v = cell1<FMA>(xv, st.Y[w], m);
                    if constexpr (TRACE) {
                        const int su = S[0][w];
                        const int sv = (diag == m) ? sd : ((up == m) ? su : sl);
                        sd = su; S[0][w] = sv; sl = sv;
                    }
                    diag = up; st.D[w] = v; left = v;
                }
                outv = left;
                outs = sl;
            } else {
                const unsigned long long xx = reinterpret_cast<const unsigned long long*>(xs)[r0];
                float l0 = lin, l1 = right0;
                float d0 = prevleft[0], d1 = prevleft[1];
                int sl0 = lins, sl1 = right0_s, sd0 = prevleft_s[0], sd1 = prevleft_s[1];
                prevleft[0] = l0; prevleft[1] = l1;
                prevleft_s[0] = sl0; prevleft_s[1] = sl1;
#pragma unroll
                for (int w = 0; w < WC; ++w) {
                    const float u0v = lo32(st.D[w]), u1v = hi32(st.D[w]);
                    const float m0 = min3f(d0, u0v, l0);
                    const float m1 = min3f(d1, u1v, l1);
                    unsigned long long tt, vv;
                    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(xx), "l"(st.Y[w]));
                    if (FMA) {
                        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(vv) : "l"(tt), "l"(pk(m0, m1)));
                    } else {
                        const float t0v = lo32(tt), t1v = hi32(tt);
                        vv = pk(__fadd_rn(__fmul_rn(t0v, t0v), m0), __fadd_rn(__fmul_rn(t1v, t1v), m1));
                    }
                    if constexpr (TRACE) {
                        const int su0 = S[0][w], su1 = S[1][w];
                        const int sv0 = (d0 == m0) ? sd0 : ((u0v == m0) ? su0 : sl0);
                        const int sv1 = (d1 == m1) ? sd1 : ((u1v == m1) ? su1 : sl1);
                        sd0 = su0; sd1 = su1; S[0][w] = sv0; S[1][w] = sv1; sl0 = sv0; sl1 = sv1;
                    }
                    st.D[w] = vv;
                    d0 = u0v; d1 = u1v;
                    l0 = lo32(vv); l1 = hi32(vv);
                }
                right0 = l0; right0_s = sl0;
                outv = l1; outs = sl1;
            }

            // ---- last-row fold (minimum extracted as the bottom row is produced)
            if (r0 == N - 1 && p0 >= 0 && p0 < P.Pr)
                fold_last_row<C, WC, TRACE>(st, S, 0, (int)(((long)p0 * V + u0) * WC), best[0], bestcol[0],
                                            beststart[0]);
            if (C == 2 && r1 == N - 1 && p1 >= 0 && p1 < P.Pr)
                fold_last_row<C, WC, TRACE>(st, S, C - 1, (int)(((long)p1 * V + u0 + 1) * WC), best[C - 1],
                                            bestcol[C - 1], beststart[C - 1]);

            // ---- lane 31: right edge to the next warp's inbox (or the boundary ring)
            if (lane == 31) {
                E e;
                e.d = outv;
                if constexpr (TRACE) e.s = outs;
                if (has_succ_ring) {
                    succ_ring[(t + 1) & (RS - 1)] = e;
                } else {
                    const int bl = b0 - (C - 1);               // band of the last chain
                    if (bl >= 0 && bl < Mtot_bands) succ_ring[(C == 2) ? r1 : r0] = e;
                }
            }

            // ---- advance
            ++b0;
            if (++r0 == Pd) { r0 = 0; ++p0; }
        }

        // ---- publish progress
        __syncwarp();
        if (lane == 31) st_release_cluster(succ_pp, t0 + K);
        if (lane == 0 && gw > 0) st_release_cluster(pred_cp, t0 + K);
    }

    // ---- reduction of (cost, col[, start]) over chains, lanes, warps, cluster CTAs
    float bc = best[0];
    int bj = bestcol[0], bs = beststart[0];
#pragma unroll
    for (int c = 1; c < C; ++c)
        if (better(best[c], bestcol[c], bc, bj)) { bc = best[c]; bj = bestcol[c]; bs = beststart[c]; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float oc = __shfl_xor_sync(FULL, bc, o);
        const int oj = __shfl_xor_sync(FULL, bj, o);
        const int os = __shfl_xor_sync(FULL, bs, o);
        if (better(oc, oj, bc, bj)) { bc = oc; bj = oj; bs = os; }
    }
    if (lane == 0) red[warp] = Partial{bc, bj, bs, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < GW; ++w)
            if (better(red[w].cost, red[w].col, bc, bj)) { bc = red[w].cost; bj = red[w].col; bs = red[w].start; }
        Partial* dst = cluster.map_shared_rank(red + 32, 0);
        dst[rank] = Partial{bc, bj, bs, 0};
    }
    cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
        for (int k = 1; k < CL; ++k) {
            const Partial pr = red[32 + k];
            if (better(pr.cost, pr.col, bc, bj)) { bc = pr.cost; bj = pr.col; bs = pr.start; }
        }
        if (*P.err_flag == 0) {
            if (bj == 0x7fffffff) { bj = 0; bs = 0; }   // every cell overflowed (raw mode only)
            P.out_cost[q] = bc;
            P.out_end[q] = bj;
            if (TRACE && P.out_start) P.out_start[q] = bs;
        }
    }
}

}  // namespace sdtw
