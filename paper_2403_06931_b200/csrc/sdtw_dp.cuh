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
#include <type_traits>
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
__device__ __forceinline__ void st_release_cta(int* p, int v) {
    asm volatile("st.release.cta.shared::cta.b32 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(p)), "r"(v)
                 : "memory");
}
__device__ __forceinline__ int ld_acquire_cluster(const int* p) {
    int v;
    asm volatile("ld.acquire.cluster.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ int ld_acquire_cta(const int* p) {
    int v;
    asm volatile("ld.acquire.cta.shared::cta.b32 %0, [%1];"
                 : "=r"(v)
                 : "r"((unsigned)__cvta_generic_to_shared(p))
                 : "memory");
    return v;
}
// Progress counters live in the waiting warp's own CTA.  When the whole ring is
// one CTA (no cluster) every hand-off is CTA-scoped: an LDS-class acquire, no
// L1 invalidation.  Across cluster CTAs the acquire must be cluster-scoped.
template <bool CLUSTER>
__device__ __forceinline__ int ld_acquire(const int* p) {
    return CLUSTER ? ld_acquire_cluster(p) : ld_acquire_cta(p);
}
template <bool CLUSTER>
__device__ __forceinline__ void st_release(int* p, int v, bool local) {
    if (CLUSTER && !local) st_release_cluster(p, v);
    else if (CLUSTER) st_release_cluster(p, v);
    else st_release_cta(p, v);
}
// Wait until *p >= need.  A watchdog turns a protocol bug into a diagnosable trap
// instead of a hung GPU (never reached in a correct run: every wait is bounded by
// the ring's progress).
template <bool CLUSTER>
__device__ __noinline__ void spin_slow(const int* p, int need, int tag) {
    long long n = 0;
    int v;
    while ((v = ld_acquire<CLUSTER>(p)) < need) {
        __nanosleep(128);
        if (++n == (1LL << 24)) {
            printf("sdtw watchdog: block %d thread %d tag %d waits *p=%d >= %d\n", (int)blockIdx.x,
                   (int)threadIdx.x, tag, v, need);
            __trap();
        }
    }
}
template <bool CLUSTER>
__device__ __forceinline__ void spin_until_geq(const int* p, int need, int tag = 0) {
    if (ld_acquire<CLUSTER>(p) >= need) return;
    spin_slow<CLUSTER>(p, need, tag);
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

// Shared-memory carve-up (dynamic).  Returns total bytes.
struct SmemLayout {
    int off_ctr, off_red, off_inf, off_x, off_bnd, off_ring, bytes;
};
__host__ __device__ inline SmemLayout smem_layout(int C, bool trace, int GW, int CL, int Pd, int RS) {
    SmemLayout L;
    const int ent = trace ? 8 : 4;
    int o = 0;
    L.off_ctr = o;  o += 2 * 32 * 4;                   // pp[32], cp[32]
    L.off_red = o;  o += 16 * (32 + 16);               // per-warp + per-rank partials
    L.off_inf = o;  o += 32 * 8;                        // +inf inbox entries (round 0)
    o = (o + 15) & ~15;
    L.off_x = o;    o += (Pd + 1) * C * 4;
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * ent;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * ent;
    L.bytes = (o + 15) & ~15;
    (void)CL;
    return L;
}

struct Partial { float cost; int col; int start; int pad; };

// ----------------------------------------------------------------------------
// Register state of one lane.  C == 2 keeps (chain0, chain1) pairs in aligned
// 64-bit registers so that FADD2 / FFMA2 read and write them in place.
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

// A lane's row state lives in a ROTATING register file of U = WC+1 slots per
// chain (pairs of chains packed in 64-bit registers when C == 2): each cell's new
// value is written into the slot of its diag input, which dies at that cell, so
// the row moves one slot down per step and returns to its origin after U steps.
// The fast loop is unrolled U steps so every slot index is a compile-time
// constant and no register-to-register moves are needed.
template <int C> struct RegT { using T = float; };
template <> struct RegT<2> { using T = unsigned long long; };

template <int C, int WC, bool TRACE> struct RotRow {
    static constexpr int U = WC + 1;
    typename RegT<C>::T D[U];
    int S[TRACE ? C : 1][TRACE ? U : 1];
    // element w of the row when the rotation offset is h (row at slots (w - h) mod U)
    __device__ __forceinline__ static constexpr int slot(int w, int h) { return ((w - h) % U + U) % U; }
    __device__ __forceinline__ float d(int c, int w, int h = 0) const {
        if constexpr (C == 1) return D[slot(w, h)];
        else return c ? hi32(D[slot(w, h)]) : lo32(D[slot(w, h)]);
    }
    __device__ __forceinline__ void set_d(int c, int w, float v, int h = 0) {
        if constexpr (C == 1) D[slot(w, h)] = v;
        else {
            const int k = slot(w, h);
            D[k] = c ? pk(lo32(D[k]), v) : pk(v, hi32(D[k]));
        }
    }
    __device__ __forceinline__ int s(int c, int w, int h = 0) const {
        if constexpr (TRACE) return S[c][slot(w, h)];
        else return 0;
    }
    __device__ __forceinline__ void set_s(int c, int w, int v, int h = 0) {
        if constexpr (TRACE) S[c][slot(w, h)] = v;
    }
};
template <int C, int WC> struct Ys;
template <int WC> struct Ys<1, WC> {
    float Y[WC];
    __device__ __forceinline__ void set(int, int w, float v) { Y[w] = v; }
};
template <int WC> struct Ys<2, WC> {
    unsigned long long Y[WC];
    __device__ __forceinline__ void set(int c, int w, float v) { Y[w] = c ? pk(lo32(Y[w]), v) : pk(v, hi32(Y[w])); }
};

// Per-lane scalars carried from step to step.
template <int C> struct LaneScalars {
    float prevleft[C];   // left input of the previous row (the next row's diag at column 0)
    int prevleft_s[C];
    float right0;        // C == 2: chain 0's right edge -> chain 1's left at the next step
    int right0_s;
    float outv;          // right edge of the last chain (to lane+1 / next warp)
    int outs;
};

// One row of the lane's strips (Eq. 1) at rotation offset H: reads the
// row at offset H, leaves the new row at offset H+1.
// C == 1: per cell FADD, FMNMX3, FFMA (3 SASS).  C == 2: per cell pair FADD2,
// 2x FMNMX3, FFMA2 (2 SASS/cell).  xx: row sample(s); lin: chain 0's left input.
template <int C, int WC, bool FMA, bool TRACE, int H>
__device__ __forceinline__ void row_cells(RotRow<C, WC, TRACE>& R, const Ys<C, WC>& Y, unsigned long long xx,
                                          float lin, int lins, LaneScalars<C>& ls) {
    using RR = RotRow<C, WC, TRACE>;
    if constexpr (C == 1) {
        const float xv = __uint_as_float((unsigned)xx);
        float left = lin, diag = ls.prevleft[0];
        int sl = lins, sd = ls.prevleft_s[0];
        ls.prevleft[0] = lin;
        ls.prevleft_s[0] = lins;
#pragma unroll
        for (int w = 0; w < WC; ++w) {
            const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);   // up slot; diag slot (= output slot)
            const float up = R.D[ku];
            const float dg = (w == 0) ? diag : R.D[kd];
            const float m = min3f(dg, up, left);
            const float v = cell1<FMA>(xv, Y.Y[w], m);
            if constexpr (TRACE) {
                const int su = R.S[0][ku];
                const int sdg = (w == 0) ? sd : R.S[0][kd];
                const int sv = (dg == m) ? sdg : ((up == m) ? su : sl);
                R.S[0][kd] = sv;
                sl = sv;
            }
            R.D[kd] = v;
            left = v;
        }
        ls.outv = left;
        ls.outs = sl;
    } else {
        float l0 = lin, l1 = ls.right0;
        const float pd0 = ls.prevleft[0], pd1 = ls.prevleft[1];
        const int psd0 = ls.prevleft_s[0], psd1 = ls.prevleft_s[1];
        int sl0 = lins, sl1 = ls.right0_s;
        ls.prevleft[0] = l0;
        ls.prevleft[1] = l1;
        ls.prevleft_s[0] = sl0;
        ls.prevleft_s[1] = sl1;
#pragma unroll
        for (int w = 0; w < WC; ++w) {
            const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);
            const float u0v = lo32(R.D[ku]), u1v = hi32(R.D[ku]);
            const float d0 = (w == 0) ? pd0 : lo32(R.D[kd]);
            const float d1 = (w == 0) ? pd1 : hi32(R.D[kd]);
            const float m0 = min3f(d0, u0v, l0);
            const float m1 = min3f(d1, u1v, l1);
            unsigned long long tt, vv;
            asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(xx), "l"(Y.Y[w]));
            if (FMA) {
                asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(vv) : "l"(tt), "l"(pk(m0, m1)));
            } else {
                const float t0v = lo32(tt), t1v = hi32(tt);
                vv = pk(__fadd_rn(__fmul_rn(t0v, t0v), m0), __fadd_rn(__fmul_rn(t1v, t1v), m1));
            }
            if constexpr (TRACE) {
                const int su0 = R.S[0][ku], su1 = R.S[1][ku];
                const int sd0 = (w == 0) ? psd0 : R.S[0][kd];
                const int sd1 = (w == 0) ? psd1 : R.S[1][kd];
                const int sv0 = (d0 == m0) ? sd0 : ((u0v == m0) ? su0 : sl0);
                const int sv1 = (d1 == m1) ? sd1 : ((u1v == m1) ? su1 : sl1);
                R.S[0][kd] = sv0;
                R.S[1][kd] = sv1;
                sl0 = sv0;
                sl1 = sv1;
            }
            R.D[kd] = vv;
            l0 = lo32(vv);
            l1 = hi32(vv);
        }
        ls.right0 = l0;
        ls.right0_s = sl0;
        ls.outv = l1;
        ls.outs = sl1;
    }
}

// Load the WC reference samples of strip `strip` (+inf beyond Malloc).
template <int WC>
__device__ __forceinline__ void load_strip_any(const float* __restrict__ Yg, int Malloc, long strip, float (&y)[WC]) {
    const long col0 = strip * WC;
#pragma unroll
    for (int w = 0; w < WC; ++w) y[w] = (col0 + w < (long)Malloc) ? __ldg(Yg + col0 + w) : INFINITY;
}

// Round transition of chain c at rotation offset 0: new strip (reload y),
// virtual row -1 = 0.
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void enter_strip(RotRow<C, WC, TRACE>& row, Ys<C, WC>& Y, int c, long strip, bool live,
                                            const float* __restrict__ Yg, int Malloc, LaneScalars<C>& ls) {
    float y[WC];
    if (live) load_strip_any<WC>(Yg, Malloc, strip, y);
    else {
#pragma unroll
        for (int w = 0; w < WC; ++w) y[w] = INFINITY;
    }
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        Y.set(c, w, y[w]);
        row.set_d(c, w, 0.0f);
        row.set_s(c, w, (int)(strip * WC) + w + 1);   // S(-1, j) = j+1, so row 0 gets S = j
    }
    ls.prevleft[c] = 0.0f;                // D(-1, col0-1) = 0
    ls.prevleft_s[c] = (int)(strip * WC);
}

// Fold the last row of chain c (rotation offset 0) into (best, bestcol, beststart):
// strict '<' keeps the smallest column on ties (strips are visited in increasing
// column order).
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void fold_last_row(const RotRow<C, WC, TRACE>& row, int c, int col0, float& best,
                                              int& bestcol, int& beststart) {
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const float v = row.d(c, w);
        if (v < best) {
            best = v;
            bestcol = col0 + w;
            beststart = row.s(c, w);
        }
    }
}

// Move the row from rotation offset 1 back to offset 0 (slow path only).
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void unrotate1(RotRow<C, WC, TRACE>& R) {
    using RR = RotRow<C, WC, TRACE>;
    RotRow<C, WC, TRACE> T;
#pragma unroll
    for (int w = 0; w < RR::U; ++w) {
        T.D[w] = R.D[RR::slot(w, 1)];
        if constexpr (TRACE) {
#pragma unroll
            for (int c = 0; c < C; ++c) T.S[c][w] = R.S[c][RR::slot(w, 1)];
        }
    }
    R = T;
}

template <int I, int N_, class F>
__device__ __forceinline__ void static_for(F&& f) {
    if constexpr (I < N_) {
        f(std::integral_constant<int, I>{});
        static_for<I + 1, N_>(f);
    }
}

// index of the (x_r, x_{r-1}) pair of row r in the parity-split layout
__host__ __device__ __forceinline__ int xpair_index(int r, int Pd) { return (r & 1) * ((Pd + 1) >> 1) + (r >> 1); }

// floor-mod
__device__ __forceinline__ int fmod_pos(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }
// does the band interval [blo, blo+len) contain a band whose row (band mod Pd) == row?
__device__ __forceinline__ bool hits_row(int blo, int len, int row, int Pd) {
    return fmod_pos(row - blo, Pd) < len;
}

template <int C, int WC, bool FMA, bool TRACE, bool CLUSTER>
__global__ void __launch_bounds__(256) sdtw_dp_kernel(const DpParams P) {
    static_assert(C == 1 || C == 2, "C");
    static_assert(((WC + 1) & WC) == 0 && (32 * C) % (WC + 1) == 0,
                  "rotation period U = WC+1 must be a power of two dividing 32*C");
    extern __shared__ __align__(16) unsigned char smem[];
    using E = Entry<TRACE>;
    using RowT = RotRow<C, WC, TRACE>;
    constexpr int U = RowT::U;

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
    E* infs = reinterpret_cast<E*>(smem + L.off_inf);

    // ---- prologue: query -> smem (pairs (x_r, x_{r-1 mod Pd}) when C == 2), rings, counters
    const float* xq = P.X + (long)q * N;
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        const float a = (r < N) ? xq[r] : 0.0f;
        if (C == 2) {
            // pairs (x_r, x_{r-1}); even rows then odd rows so that a warp's lanes
            // (rows r, r-2, r-4, ...) read consecutive 8-byte words (no bank conflict)
            const int rp = (r == 0) ? Pd - 1 : r - 1;
            const float b = (rp < N) ? xq[rp] : 0.0f;
            reinterpret_cast<float2*>(xs)[xpair_index(r, Pd)] = make_float2(a, b);
        } else {
            xs[r] = a;
        }
        E e;
        e.d = INFINITY;
        if constexpr (TRACE) e.s = 0;
        bnd[r] = e;
    }
    if (threadIdx.x < 32) {
        E e;
        e.d = INFINITY;
        if constexpr (TRACE) e.s = 0;
        infs[threadIdx.x] = e;
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
    const int u_min = 32 * C * gw;                 // virtual lane of lane 0, chain 0
    const int u_max = u_min + 32 * C - 1;          // virtual lane of lane 31, last chain
    const int u0 = C * (32 * gw + lane);
    const int u_last = V - 1;
    const int Mtot_bands = P.Pr * Pd;

    // ---- per-lane state (the strip's row in a rotating register file)
    RowT R;
    Ys<C, WC> Y;
#pragma unroll
    for (int k = 0; k < U; ++k) {
        if constexpr (C == 1) R.D[k] = INFINITY;
        else R.D[k] = pk(INFINITY, INFINITY);
        if constexpr (TRACE) {
#pragma unroll
            for (int c = 0; c < C; ++c) R.S[c][k] = 0;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c)
#pragma unroll
        for (int w = 0; w < WC; ++w) Y.set(c, w, INFINITY);
    LaneScalars<C> ls;
#pragma unroll
    for (int c = 0; c < C; ++c) { ls.prevleft[c] = INFINITY; ls.prevleft_s[c] = 0; }
    ls.right0 = INFINITY; ls.right0_s = 0; ls.outv = INFINITY; ls.outs = 0;
    float best[C];
    int bestcol[C], beststart[C];
#pragma unroll
    for (int c = 0; c < C; ++c) { best[c] = INFINITY; bestcol[c] = 0x7fffffff; beststart[c] = 0; }

    // band of chain 0 at this warp's first step t = u_min
    int b0 = -C * lane;
    int p0 = (b0 < 0) ? -1 : 0;
    int r0 = (b0 < 0) ? b0 + Pd : 0;

    // warp g runs steps [32*C*g, 32*C*g + span): its lanes' bands cover [0, Pr*Pd)
    const int span = (32 * C - 1 + Mtot_bands + K - 1) / K * K;
    const int t_begin = u_min;
    const int t_end = t_begin + span;
    // a predecessor never publishes past its own end: the successor's trailing
    // (idle-band) chunks must not wait for more
    const int pred_end = t_end - 32 * C;                 // = t_end of warp gw-1
    const int last_end = 32 * C * (G - 1) + span;        // = t_end of warp G-1
    const unsigned FULL = 0xffffffffu;

    // One step on the slow path: per-lane round transitions / last-row folds may occur.
    auto slow_step = [&](int t) {
        float lin = __shfl_up_sync(FULL, ls.outv, 1);
        int lins = 0;
        if constexpr (TRACE) lins = __shfl_up_sync(FULL, ls.outs, 1);
        if (lane == 0) {
            E e;
            if (gw == 0) {
                if (p0 >= 1) e = my_in[r0];
                else { e.d = INFINITY; if constexpr (TRACE) e.s = 0; }
            } else {
                e = my_in[(t - 1) & (RS - 1)];
            }
            lin = e.d;
            if constexpr (TRACE) lins = e.s;
        }
        const int r1 = (r0 == 0) ? Pd - 1 : r0 - 1;   // chain 1 row
        const int p1 = (r0 == 0) ? p0 - 1 : p0;       // chain 1 round
        if (r0 == 0) enter_strip<C, WC, TRACE>(R, Y, 0, (long)p0 * V + u0, p0 < P.Pr, P.Y, P.Malloc, ls);
        if (C == 2 && r1 == 0)
            enter_strip<C, WC, TRACE>(R, Y, C - 1, (long)p1 * V + u0 + 1, p1 < P.Pr, P.Y, P.Malloc, ls);
        unsigned long long xx;
        if constexpr (C == 2) xx = reinterpret_cast<const unsigned long long*>(xs)[xpair_index(r0, Pd)];
        else xx = __float_as_uint(xs[r0]);
        row_cells<C, WC, FMA, TRACE, 0>(R, Y, xx, lin, lins, ls);
        unrotate1<C, WC, TRACE>(R);
        if (r0 == N - 1 && p0 >= 0 && p0 < P.Pr)
            fold_last_row<C, WC, TRACE>(R, 0, (int)(((long)p0 * V + u0) * WC), best[0], bestcol[0], beststart[0]);
        if (C == 2 && r1 == N - 1 && p1 >= 0 && p1 < P.Pr)
            fold_last_row<C, WC, TRACE>(R, C - 1, (int)(((long)p1 * V + u0 + 1) * WC), best[C - 1],
                                        bestcol[C - 1], beststart[C - 1]);
        if (lane == 31) {
            E e;
            e.d = ls.outv;
            if constexpr (TRACE) e.s = ls.outs;
            if (has_succ_ring) {
                succ_ring[t & (RS - 1)] = e;
            } else {
                const int bl = b0 - (C - 1);               // band of the last chain
                if (bl >= 0 && bl < Mtot_bands) succ_ring[(C == 2) ? r1 : r0] = e;
            }
        }
        ++b0;
        if (++r0 == Pd) { r0 = 0; ++p0; }
    };

    for (int t0 = t_begin; t0 < t_end; t0 += K) {
        // ---- chunk-level flow control (one lane each), then converge
        if (lane == 0) {
            if (gw > 0) spin_until_geq<CLUSTER>(pp + warp, min(t0 + K - 1, pred_end), 1);
            else if (t0 + K - 1 >= Pd) spin_until_geq<CLUSTER>(pp, min(t0 + K - Pd + u_last, last_end), 2);
        }
        if (lane == 31 && has_succ_ring) spin_until_geq<CLUSTER>(cp + warp, t0 + K - RS + 1, 3);
        __syncwarp();

        // ---- fast chunk: no lane of this warp crosses row 0 (round transition) or
        // row N-1 (last-row fold) -> warp-uniform, branch-free steps
        const int blo = t0 - u_max, blen = K + 32 * C - 1;
        const bool fast = !hits_row(blo, blen, 0, Pd) && !hits_row(blo, blen, N - 1, Pd);
        if (fast) {
            // Warp-uniform ring addressing, one base pointer per rotation period:
            // lane 0 reads its left input for step t from slot t-1 of its inbox (or
            // row t-u_min of the boundary ring for warp 0; +inf entries in round 0),
            // lane 31 writes its right edge of step t to slot t of the successor's
            // inbox (or row t-u_max of the boundary ring).  t0 and the period start
            // are multiples of U, and U divides RS, so only the first read of a
            // period can wrap around the inbox.
            const int in_row = fmod_pos(t0 - u_min, Pd);
            const bool lane0_inf = (gw == 0) && (t0 < Pd);
            const int out_row = fmod_pos(t0 - u_max, Pd);
            const unsigned long long* xpe = reinterpret_cast<const unsigned long long*>(xs) + xpair_index(r0, Pd);
            const unsigned long long* xpo = reinterpret_cast<const unsigned long long*>(xs) + xpair_index(r0 + 1, Pd);
            const float* x1 = xs + r0;
#pragma unroll 1
            for (int s = 0; s < K; s += U) {
                const int tg = t0 + s;
                const E* ib0;
                const E* ib1;
                if (gw == 0) {
                    ib0 = lane0_inf ? infs : bnd + in_row + s;
                    ib1 = ib0 + 1;
                } else {
                    ib0 = my_in + ((tg - 1) & (RS - 1));
                    ib1 = my_in + (tg & (RS - 1));
                }
                E* ob = has_succ_ring ? succ_ring + (tg & (RS - 1)) : succ_ring + out_row + s;
                static_for<0, U>([&](auto hc) {
                    constexpr int h = decltype(hc)::value;
                    float lin = __shfl_up_sync(FULL, ls.outv, 1);
                    int lins = 0;
                    if constexpr (TRACE) lins = __shfl_up_sync(FULL, ls.outs, 1);
                    const E e = (h == 0) ? ib0[0] : ib1[h - 1];
                    if (lane == 0) {
                        lin = e.d;
                        if constexpr (TRACE) lins = e.s;
                    }
                    unsigned long long xx;
                    if constexpr (C == 2) xx = (h & 1) ? xpo[h >> 1] : xpe[h >> 1];
                    else xx = __float_as_uint(x1[h]);
                    row_cells<C, WC, FMA, TRACE, h>(R, Y, xx, lin, lins, ls);
                    if (lane == 31) {
                        E o;
                        o.d = ls.outv;
                        if constexpr (TRACE) o.s = ls.outs;
                        ob[h] = o;
                    }
                });
                if constexpr (C == 2) { xpe += U / 2; xpo += U / 2; }
                else x1 += U;
            }
            b0 += K;
            r0 += K;                                     // may land exactly on the next round
            if (r0 >= Pd) { r0 -= Pd; ++p0; }
        } else {
#pragma unroll 1
            for (int s = 0; s < K; ++s) slow_step(t0 + s);
        }

        // ---- publish progress
        __syncwarp();
        if (lane == 31) st_release<CLUSTER>(succ_pp, t0 + K, true);
        if (lane == 0 && gw > 0) st_release<CLUSTER>(pred_cp, t0 + K, true);
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
