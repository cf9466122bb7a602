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
//  * Strip state lives in registers (the paper's two row buffers of segment width,
//    P:L100, become one ROTATING register file of WC+1 slots, see RotRow).
//  * Right-edge hand-off: chain c -> chain c+1 of the same lane is a register; the
//    last chain -> next lane by SHFL.UP ("__shfl_up"); lane 31 -> next warp
//    through a shared-memory ring (DSMEM when the next warp is in another CTA of
//    the cluster) with release/acquire progress counters checked every K steps;
//    the last virtual lane -> virtual lane 0 of the next round through the
//    Pd-entry boundary ring (the paper's "shared memory buffer which represents the
//    last segment values").
//  * C >= 2 packs chains (2p, 2p+1) into f32x2 FADD2/FFMA2 (sm_100a): per 2 cells
//    FADD2 + FFMA2 + 2 FMNMX3 = 2 SASS/cell instead of 3; C == 4 runs two such
//    independent pairs per lane (ILP 2 on the FMNMX3 -> FFMA2 dependency chain).
//  * Steps are grouped in chunks of K; a chunk in which no lane of the warp crosses
//    a round boundary (row 0) or the last row (row N-1) is "fast": branch-free,
//    warp-uniform addressing, unrolled one rotation period at a time.  The few
//    other chunks take the per-lane "slow" path (round transition, last-row fold).
//  * TRACE carries, per cell, the start column of its argmin predecessor
//    (priority diag > up > left on equality; reading G6).
#pragma once
#include <cooperative_groups.h>
#include <climits>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
#include <cuda_fp16.h>
#include <type_traits>

// Build-time knobs (A/B variants via -D; the defaults are the measured best)
#ifndef SDTW_C4_MINB
#define SDTW_C4_MINB 3           // resident 4-warp CTAs per SM the 4-chain kernels are sized for
#endif
#ifndef SDTW_BDP_TRACE
#define SDTW_BDP_TRACE 0      // debugging: 1 compiles the (dead) caller-boundary code into start-index kernels
#endif
#ifndef SDTW_ALWAYS_WAIT
#define SDTW_ALWAYS_WAIT 0    // debugging: 1 waits for the staged strips before every slow period
#endif
#ifndef SDTW_MOV_ASM
// float-pair helpers: 3 (default) inline-PTX unpack + C++ pack; 0 all C++ (+4 registers,
// -3.7 %); 1 the old inline-PTX pack `mov.b64 %0, {%1, %2}` (wrong cells in some layouts
// and at ptxas -O1); 2 / 4 further debugging variants
#define SDTW_MOV_ASM 3
#endif
#ifndef SDTW_SCALAR_CELL2
#define SDTW_SCALAR_CELL2 0   // debugging: 1 computes the packed cells with scalar FADD / FFMA
#endif
#ifndef SDTW_SPEC_CLUSTER
#define SDTW_SPEC_CLUSTER 0   // debugging: 1 compiles the (dead) speculative-unit decode into cluster
                              // kernels too, 2 also the (dead) persistent-unit code
#endif
#ifndef SDTW_SPIN_NS
#define SDTW_SPIN_NS 256         // nanosleep per flow-control poll (r01 A/B: 256 > 64 by 0.8 %)
#endif

namespace sdtw {
namespace cg = cooperative_groups;

struct DpParams {
    const float* X;        // [Z][N] query samples (normalised or raw), device
    const float* Y;        // reference, device, Malloc floats (+inf beyond M)
    int Malloc;            // padded reference length
    int Z, N, M;
    int Pd;                // round period in steps (>= N)
    int Pr;                // number of rounds
    int K;                 // steps per hand-off chunk (multiple of WC+1)
    int RS;                // inter-warp ring entries (power of two, multiple of WC+1)
    float* out_cost;
    int64_t* out_end;
    int64_t* out_start;    // TRACE only
    const int* err_flag;   // nonzero -> write no results
    // persistent scheduling (persistent != 0): CTAs pull units u = s*Z + q (query q,
    // rounds [s*Pr/S, (s+1)*Pr/S)) from *counter; consecutive segments of a query hand
    // the boundary column over through bnd_g and seg_done[q]; every unit writes its
    // (cost, col, start) candidate to cand[q*S + s] for the finalize kernel.
    int persistent;
    int S;
    int Zq;                // real number of queries (dual-query kernel: P.Z counts pairs)
    // ragged batches: query q is X[qoff[q] .. qoff[q]+qlen[q]) with round
    // period max(qlen[q], need); N / Pd above are then the maxima (shared-memory sizing)
    const int64_t* qoff;   // nullptr = fixed length N, query q at X + q*N
    const int* qlen;
    int need;              // V + (G+1)K: the smallest ring-safe round period
    int* counter;
    const int* order;      // grab order of the units (nullptr = identity), see unit_order() in sdtw_api.cu
    int* seg_done;
    void* bnd_g;
    void* cand;
    // speculative segments (utab != nullptr): unit kind k of a query is
    // utab[k] = {pa, pb, in_k, db}: rounds [pa, pb), left boundary = the end column of
    // kind in_k of the same query (-1: +inf), db != 0: no free start (virtual row -1 =
    // +inf).  Every unit stores its end column at bnd_g[(q*S + k)*PdMax] and raises
    // seg_done[q*S + k]; see spec_table() in sdtw_api.cu.
    const int4* utab;
    // boundary DP (sdtw_boundary_dp, utab entry with in_k == -2): the unit's left boundary
    // column is bnd_user[q*N + r] (rows >= N: +inf); col_out (if set) receives the unit's
    // end column, rows [0, N), at col_out[q*N + r] (fp32 cost/end kernels only)
    const float* bnd_user;
    float* col_out;
    float negzero;         // -0.0f (start-index kernels: the predicated-move FADD operand, never folded)
    // round checkpoints (CKPT kernels): the last column of every round as the
    // unit computed it, rows [0, Pd), at ckpt[(q*Pr + p)*Pd + r] for the free-DP units (A_s,
    // B_s, sequential segments, one CTA per ring) and at ckpt_c[((q*(Sg-1) + s-1)*Rc + j)*Pd
    // + r] for the correction units C_s (their j-th round); merged into the true column
    // min(free, correction) by merge_ckpt_kernel.
    float* ckpt;
    float* ckpt_c;
    int ck_sg, ck_rc;
    int q8_tau2;
    long long* unit_log;   // diagnostics (SDTW_UNIT_LOG): per grabbed unit {sm<<40|block<<20|unit, grab, start, end} ns
    int tail_skip;         // 1: warps stop one round early where the unit's last round is beyond M (no end column consumed)
    const float* xg;       // XG kernels: query rows in the two-chain pair layout, q * PdMax * 2 floats per query           // uint8-codebook kernels with INF pruning: tau^2 (sdtw_q8.cuh)
};

template <bool TRACE> struct Entry { float d; };
template <> struct Entry<true> { float d; int s; };

// ------------------------------------------------------------ synchronisation
__device__ __forceinline__ long long globaltimer_ns() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
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
// one CTA (no cluster) every hand-off is CTA-scoped (an LDS-class acquire, no L1
// invalidation); across cluster CTAs the acquire/release must be cluster-scoped.
template <bool CLUSTER>
__device__ __forceinline__ int ld_acquire(const int* p) {
    if constexpr (CLUSTER) return ld_acquire_cluster(p);
    else return ld_acquire_cta(p);
}
template <bool CLUSTER>
__device__ __forceinline__ void st_release(int* p, int v) {
    if constexpr (CLUSTER) st_release_cluster(p, v);
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
__device__ __forceinline__ void spin_until_geq(const int* p, int need, int tag) {
    if (ld_acquire<CLUSTER>(p) >= need) return;
    spin_slow<CLUSTER>(p, need, tag);
}
__device__ __forceinline__ int ld_acquire_gpu(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_gpu(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Per-hop scope: only hand-offs that cross a CTA boundary of the cluster pay the
// cluster-scoped (L1-invalidating) acquire; hops inside a CTA stay CTA-scoped.
__device__ __forceinline__ void spin_until_geq_hop(const int* p, int need, int tag, bool remote) {
    if (remote) spin_until_geq<true>(p, need, tag);
    else spin_until_geq<false>(p, need, tag);
}
__device__ __forceinline__ void st_release_hop(int* p, int v, bool remote) {
    if (remote) st_release_cluster(p, v);
    else st_release_cta(p, v);
}
__device__ __forceinline__ int ld_acquire_hop(const int* p, bool remote) {
    return remote ? ld_acquire_cluster(p) : ld_acquire_cta(p);
}

// Chunk-level flow control executed by ALL 32 lanes of the warp: every lane loads
// the same counters (one broadcast load each) and the exit test is a warp vote, so
// the warp never splits.  A spin in lane 0 (or 31) alone leaves that lane in its own
// convergence group after the loop, and every following SHFL block then runs once
// per group (WARPSYNC.COLLECTIVE fallback): ncu on the r01 kernel showed 25 % of all
// cells computed that way at 16 threads per instruction.
// Waits until (*pa >= na || na == INT_MIN) && (*pb >= nb || nb == INT_MIN).
static __device__ __noinline__ void wait_uniform_slow(const int* pa, int na, bool ra, const int* pb, int nb, bool rb) {
    for (long long n = 0;; ++n) {
        __nanosleep(SDTW_SPIN_NS);
        bool ok = true;
        if (na != INT_MIN) ok = ld_acquire_hop(pa, ra) >= na;
        if (nb != INT_MIN) ok = ok && ld_acquire_hop(pb, rb) >= nb;
        if (__all_sync(0xffffffffu, ok)) return;
        if (n == (1LL << 24)) {
            if ((threadIdx.x & 31) == 0)
                printf("sdtw watchdog: block %d warp %d waits %d >= %d / %d >= %d\n", (int)blockIdx.x,
                       (int)(threadIdx.x >> 5), na != INT_MIN ? ld_acquire_hop(pa, ra) : 0, na,
                       nb != INT_MIN ? ld_acquire_hop(pb, rb) : 0, nb);
            __trap();
        }
    }
}
__device__ __forceinline__ void wait_uniform(const int* pa, int na, bool ra, const int* pb, int nb, bool rb) {
    bool ok = true;
    if (na != INT_MIN) ok = ld_acquire_hop(pa, ra) >= na;
    if (nb != INT_MIN) ok = ok && ld_acquire_hop(pb, rb) >= nb;
    if (__all_sync(0xffffffffu, ok)) return;
    wait_uniform_slow(pa, na, ra, pb, nb, rb);
}

// ------------------------------------------------------------ arithmetic
#if SDTW_MOV_ASM == 5
// (experiment) PTX unpack + pack through a float2 / u64 reinterpretation
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
    const float2 f = make_float2(a, b);
    return *reinterpret_cast<const unsigned long long*>(&f);
}
#elif SDTW_MOV_ASM == 3 || SDTW_MOV_ASM == 4
// 3 (default): inline-PTX unpack (register-pair halves, no instructions) + C++ pack (bit
// casts and shift/or, which ptxas turns into the same pair move).  The inline-PTX PACK
// `mov.b64 %0, {%1, %2}` gave wrong packed cells at ptxas -O1 (22 parity failures) and in
// some -O3 code layouts (two-chain cluster and four-chain start-index kernels); with the
// C++ pack every layout tried is exact, at 0.7 % of config-3 throughput.
// 4 (debugging): C++ unpack + inline-PTX pack -- fails like 1.
#if SDTW_MOV_ASM == 3
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
    return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}
#else
__device__ __forceinline__ float lo32(unsigned long long r) { return __uint_as_float((unsigned)(r & 0xffffffffu)); }
__device__ __forceinline__ float hi32(unsigned long long r) { return __uint_as_float((unsigned)(r >> 32)); }
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
    return r;
}
#endif
#elif SDTW_MOV_ASM == 2
// typed register-pair moves: mov.b64 between one .b64 and two .b32 registers (bit casts
// on the C++ side), so ptxas sees plain 32-bit halves of a 64-bit register pair
__device__ __forceinline__ float lo32(unsigned long long r) {
    unsigned a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(r));
    return __uint_as_float(a);
}
__device__ __forceinline__ float hi32(unsigned long long r) {
    unsigned a, b;
    asm("mov.b64 {%0, %1}, %2;" : "=r"(a), "=r"(b) : "l"(r));
    return __uint_as_float(b);
}
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "r"(__float_as_uint(a)), "r"(__float_as_uint(b)));
    return r;
}
#elif !SDTW_MOV_ASM
// all C++ (bit casts + shifts): exact in every layout tried, 4 more registers
__device__ __forceinline__ float lo32(unsigned long long r) { return __uint_as_float((unsigned)(r & 0xffffffffu)); }
__device__ __forceinline__ float hi32(unsigned long long r) { return __uint_as_float((unsigned)(r >> 32)); }
__device__ __forceinline__ unsigned long long pk(float a, float b) {
    return ((unsigned long long)__float_as_uint(b) << 32) | __float_as_uint(a);
}
#else
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
#endif
__device__ __forceinline__ float min3f(float a, float b, float c) { return fminf(fminf(a, b), c); }

// fp32 cell value d(x,y) + m (the oracle's `cell`), scalar
template <bool FMA>
__device__ __forceinline__ float cell1(float x, float y, float m) {
    const float t = __fsub_rn(x, y);
    if (FMA) return __fmaf_rn(t, t, m);
    return __fadd_rn(__fmul_rn(t, t), m);
}
// the same for two chains at once: one FADD2 + one FFMA2 (each lane rounded as the scalar ops)
template <bool FMA>
__device__ __forceinline__ unsigned long long cell2(unsigned long long xx, unsigned long long yy, float m0,
                                                    float m1) {
    unsigned long long tt, vv;
#if SDTW_SCALAR_CELL2
    // debugging: the same arithmetic with scalar FADD / FFMA (no f32x2 instructions)
    {
        const float t0 = __fsub_rn(lo32(xx), lo32(yy)), t1 = __fsub_rn(hi32(xx), hi32(yy));
        if (FMA) return pk(__fmaf_rn(t0, t0, m0), __fmaf_rn(t1, t1, m1));
        return pk(__fadd_rn(__fmul_rn(t0, t0), m0), __fadd_rn(__fmul_rn(t1, t1), m1));
    }
#endif
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(xx), "l"(yy));
    if (FMA) {
        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(vv) : "l"(tt), "l"(pk(m0, m1)));
    } else {
        const float t0 = lo32(tt), t1 = hi32(tt);
        vv = pk(__fadd_rn(__fmul_rn(t0, t0), m0), __fadd_rn(__fmul_rn(t1, t1), m1));
    }
    return vv;
}

// Start-column select of the TRACE variant, priority diag > up > left on equality
// (reading G6): branch-free FSETP + SEL pairs (the ternary form compiled to a
// BSSY/BRA/BSYNC diamond per cell -- 4.3x the instructions of the plain DP).
__device__ __forceinline__ int start_sel(float d, float u, float m, int sd, int su, int sl) {
    // (predicated moves instead of selp compile to the same FSETP + SEL)
    int r;
    asm("{\n\t.reg .pred pu, pd;\n\t"
        "setp.eq.f32 pu, %2, %3;\n\t"
        "setp.eq.f32 pd, %1, %3;\n\t"
        "selp.b32 %0, %5, %6, pu;\n\t"
        "selp.b32 %0, %4, %0, pd;\n\t}"
        : "=&r"(r)                 // early clobber: %0 is written before %4 is read
        : "f"(d), "f"(u), "f"(m), "r"(sd), "r"(su), "r"(sl));
    return r;
}

// The same select with the ALU pipe relieved (SDTW_START_PM, default): the ALU pipe (16
// lanes/clk/SMSP) already carries the FMNMX3 of every cell, and 2 FSETP + 2 SEL made it the
// bound of the start-index kernel (5 ALU ops per cell).  Here FSETP gives pd = (d == m) and
// FSETP.AND gives pu = (u == m) && !pd; the result register starts as sd, a PREDICATED FADD
// (@!pd) overwrites it with sl and a second (@pu) with su -- FMA-pipe moves: x + -0.0 == x
// bit for bit, denormals kept (no ftz); the int start columns are moved as their float bit
// patterns, and columns < 2^31 - 2^23 are never NaN patterns.  `nz` is -0.0 from the kernel
// parameters, so ptxas cannot fold the adds into moves.  ALU: 3 ops per cell instead of 5.
__device__ __forceinline__ int start_sel_pm(float d, float u, float m, int sd, int su, int sl, float nz) {
    float r = __int_as_float(sd);
    asm("{\n\t.reg .pred pu, pd;\n\t"
        "setp.eq.f32 pd, %1, %3;\n\t"
        "setp.eq.and.f32 pu, %2, %3, !pd;\n\t"
        "@!pd add.f32 %0, %5, %6;\n\t"
        "@pu add.f32 %0, %4, %6;\n\t}"
        : "+f"(r)
        : "f"(d), "f"(u), "f"(m), "f"(__int_as_float(su)), "f"(__int_as_float(sl)), "f"(nz));
    return __float_as_int(r);
}
#ifndef SDTW_START_PM
#define SDTW_START_PM 0
#endif

// lexicographic (cost, col): "a better than b"
__device__ __forceinline__ bool better(float ca, int ja, float cb, int jb) {
    return ca < cb || (ca == cb && ja < jb);
}

// ------------------------------------------------------------ shared memory
// Row samples: with XC = min(C, 2) floats per row, row r stores (x_r[, x_{r-1}])
// (indices mod Pd, idle rows are 0) and rows are split by residue r mod XC, so the
// lanes of a warp (rows r, r-C, r-2C, ...; C even => one residue class) read
// consecutive XC-float words.  C == 4 reads the pairs of rows r and r-2.
__host__ __device__ __forceinline__ int xrow_stride(int Pd, int XC) { return (Pd + XC - 1) / XC; }
__host__ __device__ __forceinline__ int xrow_index(int r, int Pd, int XC) {
    return (r % XC) * xrow_stride(Pd, XC) + r / XC;
}
__host__ __device__ __forceinline__ constexpr int xrow_floats(int C) { return C == 1 ? 1 : 2; }
// residue classes of the layout: the lanes of a warp read rows r, r-C, r-2C, ... ->
// one class per residue mod C keeps their words consecutive (conflict-free)
__host__ __device__ __forceinline__ constexpr int xrow_classes(int C) { return C; }

struct SmemLayout {
    int off_ctr, off_red, off_inf, off_x, off_bnd, off_ring, off_stage, bytes;
};
// xs: "single" row layout (x_r alone, plain row order; C == 2 only): half the bytes per
// row for long queries whose rows would otherwise cost a resident CTA, one more LDS per step.
// xg: the query rows live in a global pair-layout buffer (DpParams::xg), none in shared memory
__host__ __device__ inline SmemLayout smem_layout(int C, int WC, bool trace, int GW, int Pd, int RS, bool xs = false,
                                                  bool xg = false) {
    SmemLayout L;
    const int ent = trace ? 8 : 4;
    int o = 0;
    L.off_ctr = o;  o += 3 * 32 * 4;                    // pp[32], cp[32], unit broadcast
    L.off_red = o;  o += 16 * (32 + 16);                // per-warp + per-rank partials
    L.off_inf = o;  o += 32 * 8;                        // +inf inbox entries (round 0)
    o = (o + 15) & ~15;
    L.off_x = o;    o += xg ? 0 : (xs ? Pd * 4 : xrow_stride(Pd, xrow_classes(C)) * xrow_classes(C) * xrow_floats(C) * 4);
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * ent;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * ent;
    o = (o + 15) & ~15;
    L.off_stage = o; o += GW * 32 * C * WC * 4;         // next-round reference strips, per warp
    L.bytes = (o + 15) & ~15;
    return L;
}

struct Partial { float cost; int col; int start; int pad; };

// ------------------------------------------------------------ register state
// A lane's row state lives in a ROTATING register file of U = WC+1 slots per
// chain (chains 2p, 2p+1 packed in one 64-bit register when C >= 2): each cell's
// new value is written into the slot of its diag input, which dies at that cell,
// so the row moves one slot down per step and is back at its origin after U
// steps.  The fast loop is unrolled U steps so every slot index is a
// compile-time constant and no register-to-register moves are needed.
//
// Register-bank layout (C >= 2).  The register file has an even and an odd bank and
// an instruction is re-issued once per extra distinct register it reads from one
// bank (B300_MICROARCH.md "RF banking": rt = max(rt_pipe, #even, #odd)).  FFMA2
// writes a pair (even, odd), so with chain 2p always in the low half every FMNMX3 of
// that chain would read three even registers (diag, up, left) and cost 3 issue
// cycles.  Instead the ORIENTATION of a column's pair alternates with the column
// parity: column w holds (chain 2p, chain 2p+1) for even w and (2p+1, 2p) for odd w,
// so diag/left (column w-1) and up (column w) of one chain sit in opposite banks.
// The query pair is swapped for odd columns by a free FADD2 operand swizzle (.LO_HI)
// and the reference pairs are stored in their column's orientation.
#ifndef SDTW_FAST_RUNS
#define SDTW_FAST_RUNS 1
#endif
#ifndef SDTW_FAST_PERIODS
#define SDTW_FAST_PERIODS 1
#endif
#ifndef SDTW_SLOW_UNROLL
#define SDTW_SLOW_UNROLL 2
#endif
#ifndef SDTW_STATIC_SLOW
#define SDTW_STATIC_SLOW 0
#endif
#ifndef SDTW_ALT_ORIENT
#define SDTW_ALT_ORIENT 2
#endif
__host__ __device__ __forceinline__ constexpr int pair_half(int c, int w) {   // reference pairs: half of chain c at column w
    return SDTW_ALT_ORIENT ? ((c ^ w) & 1) : (c & 1);
}
// Row values: half of chain c at column w when the row sits at rotation offset off.
// Mode 2 ("diagonal" orientation, the default) flips it with the offset as well: a
// cell's new value then has the orientation of its diag input, so the two FMNMX3 of a
// pair can write their minima straight into the dead diag register pair and FFMA2 works
// in place -- no register copies at the end of a rotation period -- while diag/up of
// one chain still sit in opposite banks.  Needs even rotation periods and slow-step
// groups (U and SDTW_SLOW_UNROLL even).
__host__ __device__ __forceinline__ constexpr int orient(int c, int w, int off) {
    return SDTW_ALT_ORIENT == 2 ? ((c ^ w ^ off) & 1) : pair_half(c, w);
}
__device__ __forceinline__ float half_of(unsigned long long r, int h) { return h ? hi32(r) : lo32(r); }
__device__ __forceinline__ unsigned long long with_half(unsigned long long r, int h, float v) {
    return h ? pk(lo32(r), v) : pk(v, hi32(r));
}
template <int C, int WC, bool TRACE> struct RotRow {
    static constexpr int U = WC + 1;
    static constexpr int NP = (C + 1) / 2;   // registers per slot
    using T = typename std::conditional<C == 1, float, unsigned long long>::type;
    T D[NP][U];
    int S[TRACE ? C : 1][TRACE ? U : 1];
    __device__ __forceinline__ static constexpr int slot(int w, int h) { return ((w - h) % U + U) % U; }
    __device__ __forceinline__ float d(int c, int w) const {   // offset 0: slot w holds column w
        if constexpr (C == 1) return D[0][w];
        else return half_of(D[c >> 1][w], orient(c, w, 0));
    }
    __device__ __forceinline__ float d_at(int c, int w, int off) const {   // rotation offset off
        if constexpr (C == 1) return D[0][slot(w, off)];
        else return half_of(D[c >> 1][slot(w, off)], orient(c, w, off));
    }
    __device__ __forceinline__ int s_at(int c, int w, int off) const { return S[TRACE ? c : 0][TRACE ? slot(w, off) : 0]; }
    __device__ __forceinline__ void init(float v) {   // every half of every slot (no partial-pair writes)
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
            for (int k = 0; k < U; ++k) {
                if constexpr (C == 1) D[p][k] = v;
                else D[p][k] = pk(v, v);
            }
    }
    __device__ __forceinline__ void set_all(int c, float v, int off = 0) {  // every slot of chain c
#pragma unroll
        for (int w = 0; w < U; ++w) {                           // column w lives in slot(w, off)
            if constexpr (C == 1) D[0][slot(w, off)] = v;
            else D[c >> 1][slot(w, off)] = with_half(D[c >> 1][slot(w, off)], orient(c, w, off), v);
        }
    }
};
template <int C, int WC> struct Ys {
    static constexpr int NP = (C + 1) / 2;
    using T = typename std::conditional<C == 1, float, unsigned long long>::type;
    T Y[NP][WC];
    __device__ __forceinline__ void init(float v) {
#pragma unroll
        for (int p = 0; p < NP; ++p)
#pragma unroll
            for (int w = 0; w < WC; ++w) {
                if constexpr (C == 1) Y[p][w] = v;
                else Y[p][w] = pk(v, v);
            }
    }
    __device__ __forceinline__ void set(int c, int w, float v) {
        if constexpr (C == 1) Y[0][w] = v;
        else Y[c >> 1][w] = with_half(Y[c >> 1][w], pair_half(c, w), v);
    }
};
// Per-lane scalars carried from step to step.
template <int C> struct LaneScalars {
    float prevleft[C];   // left input of chain c in the previous row (its diag at column 0)
    int prevleft_s[C];
    float right[C];      // right edge of chain c at the previous step (chain c+1's left;
    int right_s[C];      // right[C-1] goes to lane+1 / the next warp)
};
// Row samples of one step: C floats (x_r, x_{r-1}, ...).
template <int C> struct XRow;
template <> struct XRow<1> { float v[1]; };
template <> struct XRow<2> { unsigned long long p[1]; };
template <> struct XRow<4> { unsigned long long p[2]; };
// slow path: samples of row r (any residue)
template <int C, bool XS = false>
__device__ __forceinline__ XRow<C> load_xrow(const float* xs, int r, int Pd) {
    XRow<C> x;
    if constexpr (C == 1) x.v[0] = xs[r];
    else if constexpr (XS) x.p[0] = pk(xs[r], xs[r >= 1 ? r - 1 : r - 1 + Pd]);
    else {
        const unsigned long long* xp = reinterpret_cast<const unsigned long long*>(xs);
        x.p[0] = xp[xrow_index(r, Pd, C)];
        if constexpr (C == 4) x.p[1] = xp[xrow_index(r >= 2 ? r - 2 : r - 2 + Pd, Pd, C)];
    }
    return x;
}
// fast path: step h of a rotation period starting at row r0, with xb[j] pointing
// at row r0+j (residue class (r0+j) mod C, j < C); rows stay inside one round
template <int C, int h, bool XS = false>
__device__ __forceinline__ XRow<C> load_xrow_fast(const float* const* xb) {
    XRow<C> x;
    if constexpr (C == 1) x.v[0] = xb[0][h];
    else if constexpr (XS) x.p[0] = pk(xb[0][h], xb[0][h - 1]);    // rows r0+h, r0+h-1 (>= 0 in a fast period)
    else {
        constexpr int j0 = h % C, o0 = h / C;                       // row r0+h
        x.p[0] = reinterpret_cast<const unsigned long long*>(xb[j0])[o0];
        if constexpr (C == 4) {
            constexpr int k = h - 2, j1 = ((k % C) + C) % C, o1 = (k - j1) / C;   // row r0+h-2
            x.p[1] = reinterpret_cast<const unsigned long long*>(xb[j1])[o1];
        }
    }
    return x;
}

// One row of the lane's strips (Eq. 1) at rotation offset H: reads the
// row at offset H, leaves the new row at offset H+1.  lin: chain 0's left input.
// C == 1: per cell FADD, FMNMX3, FFMA (3 SASS); C >= 2: per cell pair FADD2,
// 2x FMNMX3, FFMA2 (2 SASS/cell); the NP pairs are independent within the step.
template <int C, int WC, bool FMA, bool TRACE, int H>
__device__ __forceinline__ void row_cells(RotRow<C, WC, TRACE>& R, const Ys<C, WC>& Y, const XRow<C>& x,
                                          float lin, int lins, LaneScalars<C>& ls, float nz) {
    using RR = RotRow<C, WC, TRACE>;
    constexpr int NP = RR::NP;
    float left[C], pd[C];
    int sl[C], psd[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        left[c] = (c == 0) ? lin : ls.right[c - 1];
        sl[c] = (c == 0) ? lins : ls.right_s[c - 1];
        pd[c] = ls.prevleft[c];
        psd[c] = ls.prevleft_s[c];
        ls.prevleft[c] = left[c];
        ls.prevleft_s[c] = sl[c];
    }
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);   // up slot; diag slot (= output slot)
        if constexpr (C == 1) {
            const float up = R.D[0][ku];
            const float dg = (w == 0) ? pd[0] : R.D[0][kd];
            const float m = min3f(dg, up, left[0]);
            const float v = cell1<FMA>(x.v[0], Y.Y[0][w], m);
            if constexpr (TRACE) {
                const int su = R.S[0][ku];
                const int sdg = (w == 0) ? psd[0] : R.S[0][kd];
                const int sv = SDTW_START_PM ? start_sel_pm(dg, up, m, sdg, su, sl[0], nz)
                                             : start_sel(dg, up, m, sdg, su, sl[0]);
                R.S[0][kd] = sv;
                sl[0] = sv;
            }
            R.D[0][kd] = v;
            left[0] = v;
        } else {
#pragma unroll
            for (int p = 0; p < NP; ++p) {
                const int c0 = 2 * p, c1 = 2 * p + 1;
                // orientation of old column w (up), old column w-1 (diag), new column w
                const int ow = orient(0, w, H), od = orient(0, w - 1, H), on = orient(0, w, H + 1);
                const float u0 = half_of(R.D[p][ku], ow), u1 = half_of(R.D[p][ku], ow ^ 1);
                const float d0 = (w == 0) ? pd[c0] : half_of(R.D[p][kd], od);
                const float d1 = (w == 0) ? pd[c1] : half_of(R.D[p][kd], od ^ 1);
                const float m0 = min3f(d0, u0, left[c0]);
                const float m1 = min3f(d1, u1, left[c1]);
                // operand swaps fold into FADD2 swizzles (.LO_HI)
                const unsigned long long xw = on ? pk(hi32(x.p[p]), lo32(x.p[p])) : x.p[p];
                const unsigned long long yw = (pair_half(0, w) != on) ? pk(hi32(Y.Y[p][w]), lo32(Y.Y[p][w])) : Y.Y[p][w];
                const unsigned long long vv = on ? cell2<FMA>(xw, yw, m1, m0) : cell2<FMA>(xw, yw, m0, m1);
                if constexpr (TRACE) {
                    const int su0 = R.S[c0][ku], su1 = R.S[c1][ku];
                    const int sd0 = (w == 0) ? psd[c0] : R.S[c0][kd];
                    const int sd1 = (w == 0) ? psd[c1] : R.S[c1][kd];
                    const int sv0 = SDTW_START_PM ? start_sel_pm(d0, u0, m0, sd0, su0, sl[c0], nz)
                                                  : start_sel(d0, u0, m0, sd0, su0, sl[c0]);
                    const int sv1 = SDTW_START_PM ? start_sel_pm(d1, u1, m1, sd1, su1, sl[c1], nz)
                                                  : start_sel(d1, u1, m1, sd1, su1, sl[c1]);
                    R.S[c0][kd] = sv0;
                    R.S[c1][kd] = sv1;
                    sl[c0] = sv0;
                    sl[c1] = sv1;
                }
                R.D[p][kd] = vv;
                left[c0] = half_of(vv, on);
                left[c1] = half_of(vv, on ^ 1);
            }
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        ls.right[c] = left[c];
        ls.right_s[c] = sl[c];
    }
}

// Stage the reference strips of round p for one warp (32*C strips of WC samples,
// contiguous in global memory) into shared memory with cp.async (no registers,
// no stall): issued one round ahead, consumed by the lanes' round transitions.
template <int C, int WC>
__device__ __forceinline__ void stage_round(float* stage, const float* __restrict__ Yg, int Malloc, int Pr, long V,
                                            int u_min, int p, int lane) {
    const long col0 = ((long)p * V + u_min) * WC;
    const unsigned sbase = (unsigned)__cvta_generic_to_shared(stage);
#pragma unroll 1
    for (int i = lane; i < 32 * C * WC; i += 32) {
        const long col = col0 + i;
        if (p < Pr && col < (long)Malloc) {
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sbase + 4u * i), "l"(Yg + col) : "memory");
        } else {
            stage[i] = INFINITY;
        }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
}

// Round transition of chain c (slow path, rotation offset 0): new strip (y from
// the staged copy), virtual row -1 = 0, and S(-1, j) = j+1 so that row 0 gets S = j.
// (zrow = +inf instead of 0: no free start, the speculative correction units)
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void enter_strip(RotRow<C, WC, TRACE>& row, Ys<C, WC>& Y, int c, long strip,
                                            const float* ystage, LaneScalars<C>& ls, int off = 0,
                                            float zrow = 0.0f) {
#pragma unroll
    for (int w = 0; w < WC; ++w) Y.set(c, w, ystage[w]);
    row.set_all(c, zrow, off);
    if constexpr (TRACE) {
#pragma unroll
        for (int k = 0; k < WC + 1; ++k) row.S[c][RotRow<C, WC, TRACE>::slot(k, off)] = (int)(strip * WC) + k + 1;
    }
    ls.prevleft[c] = zrow;                 // D(-1, col0-1) = 0
    ls.prevleft_s[c] = (int)(strip * WC);
}

// Last-row fold of chain c (slow path, rotation offset 0) into (best, bestcol,
// beststart): strict '<' keeps the smallest column on ties (strips are visited in
// increasing column order).  The row minimum is found first; the argmin scan only
// runs on a new best.
template <int C, int WC, bool TRACE>
__device__ __forceinline__ void fold_last_row(const RotRow<C, WC, TRACE>& row, int c, int col0, float& best,
                                              int& bestcol, int& beststart, int off = 0) {
    float m = row.d_at(c, 0, off);
#pragma unroll
    for (int w = 1; w < WC; ++w) m = fminf(m, row.d_at(c, w, off));
    if (m < best) {
        best = m;
#pragma unroll
        for (int w = WC - 1; w >= 0; --w) {
            if (row.d_at(c, w, off) == m) {
                bestcol = col0 + w;
                if constexpr (TRACE) beststart = row.s_at(c, w, off);
            }
        }
    }
}

// Move the row from rotation offset SH back to offset 0 (slow path only).
template <int SH, int C, int WC, bool TRACE>
__device__ __forceinline__ void unrotate(RotRow<C, WC, TRACE>& R) {
    using RR = RotRow<C, WC, TRACE>;
    RotRow<C, WC, TRACE> T;
#pragma unroll
    for (int w = 0; w < RR::U; ++w) {
#pragma unroll
        for (int p = 0; p < RR::NP; ++p) T.D[p][w] = R.D[p][RR::slot(w, SH)];
        if constexpr (TRACE) {
#pragma unroll
            for (int c = 0; c < C; ++c) T.S[c][w] = R.S[c][RR::slot(w, SH)];
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
__device__ __forceinline__ int fmod_pos(int a, int m) { int r = a % m; return r < 0 ? r + m : r; }
// does the band interval [blo, blo+len) contain a band whose row (band mod Pd) == row?
__device__ __forceinline__ bool hits_row(int blo, int len, int row, int Pd) { return fmod_pos(row - blo, Pd) < len; }

// ============================================================================ kernel
// XG: query rows read from the global pair-layout buffer P.xg (written by xg_layout_kernel) instead
// of shared memory -- long queries, whose rows would otherwise cost a resident CTA
template <int C, int WC, bool FMA, bool TRACE, bool CLUSTER, bool XS = false, bool CKPT = false, bool XG = false>
__global__ void __launch_bounds__(C == 4 ? 128 : 256, C == 4 ? SDTW_C4_MINB : 2) sdtw_dp_kernel(const DpParams P) {
    static_assert(!XS || C == 2, "single-row layout is for two chains");
    static_assert(!XG || (C == 2 && !XS && !TRACE && !CLUSTER), "global query rows: two-chain cost/end kernels");
    static_assert(!CKPT || (!TRACE && !CLUSTER && SDTW_FAST_RUNS), "round checkpoints: cost/end kernels without clusters");
    static_assert(C == 1 || C == 2 || C == 4, "chains per lane");
    static_assert(((WC + 1) & WC) == 0 && (32 * C) % (WC + 1) == 0 && (WC + 1) % C == 0,
                  "rotation period U = WC+1 must be a power of two dividing 32*C and divisible by C");
    extern __shared__ __align__(16) unsigned char smem[];
    using E = Entry<TRACE>;
    using RowT = RotRow<C, WC, TRACE>;
    constexpr int U = RowT::U;
    constexpr int PS = SDTW_FAST_PERIODS * U;        // steps per fast/slow decision (K % PS == 0)

    cg::cluster_group cluster = cg::this_cluster();
    const int CL = CLUSTER ? (int)cluster.num_blocks() : 1;
    const int rank = CLUSTER ? (int)cluster.block_rank() : 0;
    const int GW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = GW * CL;
    const int gw = rank * GW + warp;
    const int V = 32 * C * G;
    const int PdMax = P.Pd, K = P.K, RS = P.RS;
    const float nz = P.negzero;
    const SmemLayout L = smem_layout(C, WC, TRACE, GW, PdMax, RS, XS, XG);

    int* pp = reinterpret_cast<int*>(smem + L.off_ctr);        // producer progress seen by warp w
    int* cp = pp + 32;                                          // consumer progress of w's successor
    float* xs_sm = reinterpret_cast<float*>(smem + L.off_x);
    E* bnd = reinterpret_cast<E*>(smem + L.off_bnd);
    E* ring = reinterpret_cast<E*>(smem + L.off_ring);
    Partial* red = reinterpret_cast<Partial*>(smem + L.off_red);
    E* infs = reinterpret_cast<E*>(smem + L.off_inf);

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
    } else if constexpr (CLUSTER) {
        succ_ring = cluster.map_shared_rank(bnd, 0);         // boundary ring of rank 0
        succ_pp = cluster.map_shared_rank(pp, 0);            // pp[0] of rank 0
    } else {
        succ_ring = bnd;
        succ_pp = pp;
    }
    int* pred_cp = nullptr;                                   // where we report consumption
    if (gw > 0) pred_cp = (warp > 0) ? cp + warp - 1 : cluster.map_shared_rank(cp + GW - 1, rank - 1);
    const E* my_in = (gw == 0) ? bnd : ring + warp * RS;
    // does my inbound (outbound) hand-off cross a CTA boundary of the cluster?
    const bool pred_remote = CLUSTER && warp == 0;          // previous rank, or the wrap from the last rank
    const bool succ_remote = CLUSTER && warp == GW - 1;     // next rank, or the wrap to rank 0
    const int u_min = 32 * C * gw;                 // virtual lane of lane 0, chain 0
    const int u_max = u_min + 32 * C - 1;          // virtual lane of lane 31, last chain
    const int u0 = C * (32 * gw + lane);
    const int u_last = V - 1;

    constexpr int XC = XS ? 1 : xrow_floats(C);
    constexpr int NC = XS ? 1 : xrow_classes(C);
    int* unit_sh = pp + 64;                                     // broadcast of the grabbed unit
    for (int unit_iter = 0;; ++unit_iter) {
    // ---- which unit: (query q, rounds [pa, pb))
    int q, seg = 0, pa = 0, pb = P.Pr;
    int in_k = -1;                                          // speculative: source kind of the boundary
    float zrow = 0.0f;                                      // virtual row -1 (+inf: no free start)
    constexpr bool SPEC = !CLUSTER || SDTW_SPEC_CLUSTER;    // speculative units: one CTA per ring
    constexpr bool BDP = SPEC && (!TRACE || SDTW_BDP_TRACE); // caller boundary / column (sdtw_boundary_dp)
    if ((!CLUSTER || SDTW_SPEC_CLUSTER == 2) && P.persistent) {
        if (threadIdx.x == 0) {
            const int raw = atomicAdd(P.counter, 1);
            *unit_sh = (P.order && raw < P.Z * P.S) ? P.order[raw] : raw;
            unit_sh[1] = raw;                                   // (diagnostics: re-read at the unit's end)
            long long* log_slot = (P.unit_log && raw < P.Z * P.S) ? P.unit_log + 4L * raw : nullptr;
            if (log_slot) {
                unsigned sm;
                asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
                log_slot[0] = ((long long)sm << 40) | ((long long)blockIdx.x << 20) | *unit_sh;
                log_slot[1] = globaltimer_ns();
            }
        }
        __syncthreads();
        const int u = *unit_sh;
        __syncthreads();
        if (u >= P.Z * P.S) break;
        q = u % P.Z;
        seg = u / P.Z;
        int wait_slot = -1, wait_val = 0;
        if (SPEC && P.utab) {
            const int4 d = P.utab[seg];
            pa = d.x; pb = d.y; in_k = d.z; zrow = d.w ? INFINITY : 0.0f;
            if (in_k >= 0) { wait_slot = q * P.S + in_k; wait_val = 1; }
        } else {
            pa = (int)((long)seg * P.Pr / P.S);
            pb = (int)((long)(seg + 1) * P.Pr / P.S);
            if (seg > 0) { wait_slot = q; wait_val = seg; }  // previous segment's boundary column
        }
        if (wait_slot >= 0) {
            long n = 0;                                    // (every thread polls: no split warps)
            while (ld_acquire_gpu(P.seg_done + wait_slot) < wait_val) {
                __nanosleep(256);
                if (++n == (1LL << 26)) { printf("sdtw watchdog: unit %d waits segment\n", u); __trap(); }
            }
        }
        if (P.unit_log && threadIdx.x == 0 && unit_sh[1] < P.Z * P.S) P.unit_log[4L * unit_sh[1] + 2] = globaltimer_ns();
        __syncthreads();
    } else {
        if (unit_iter > 0) break;
        q = blockIdx.x / CL;
    }
    // query length and round period of this unit (ragged batches: per query)
    int N = P.N, Pd = PdMax;
    const float* xq = P.X + (long)q * N;
    if (P.qlen) {
        N = P.qlen[q];
        Pd = max(N, P.need);
        xq = P.X + P.qoff[q];
    }
    const int Pl = pb - pa;                                 // rounds in this unit
    const int Mtot_bands = Pl * Pd;
    // query rows of this unit: shared memory (filled by the prologue) or the global pair layout
    const float* xs = XG ? P.xg + (long)q * PdMax * 2 : xs_sm;
    // round checkpoints of this unit: local round l -> ckb + l*Pd (rows [0, Pd))
    float* ckb = nullptr;
    if constexpr (CKPT) {
        const int kind = seg;
        if (SPEC && P.utab && kind >= 2 * P.ck_sg)          // correction unit C_s, s = kind - 2Sg + 1
            ckb = P.ckpt_c + ((long)q * (P.ck_sg - 1) + (kind - 2 * P.ck_sg)) * P.ck_rc * (long)PdMax;
        else
            ckb = P.ckpt + ((long)q * P.Pr + pa) * (long)PdMax;
    }

    // ---- prologue: query rows -> smem, boundary ring (+inf, or the previous
    // segment's last column), counters
    const bool spec = SPEC && P.utab;
    const E* bg = reinterpret_cast<const E*>(P.bnd_g) + (spec ? ((long)q * P.S + max(in_k, 0)) : (long)q) * PdMax;
    const bool bnd_in = spec ? in_k >= 0 : pa > 0;
    // warp 0's first-round inbox is +inf only at the very start of the reference without a
    // caller-supplied boundary column (sdtw_boundary_dp starts at round 0 from one)
    const bool lead_inf = pa == 0 && !(BDP && in_k == -2);
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        if constexpr (!XG) {
            float* dst = XS ? xs_sm + r : xs_sm + (long)xrow_index(r, Pd, NC) * XC;
#pragma unroll
            for (int j = 0; j < XC; ++j) {
                int rr = r - j;
                if (rr < 0) rr += Pd;
                dst[j] = (rr < N) ? xq[rr] : 0.0f;
            }
        }
        E e;
        if (bnd_in) {
            e = bg[r];
        } else {
            if constexpr (BDP) e.d = (in_k == -2 && r < N) ? P.bnd_user[(long)q * N + r] : INFINITY;
            else e.d = INFINITY;
            if constexpr (TRACE) e.s = 0;
        }
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
    if constexpr (CLUSTER) cluster.sync();
    else __syncthreads();

    // ---- per-lane state.  Whole registers are initialised (both halves of every
    // pair): set_all / Ys::set re-pack the OTHER half of a pair, and reading an
    // uninitialised half is undefined (the wrong-cell bug).
    RowT R;
    Ys<C, WC> Y;
    R.init(INFINITY);
    Y.init(INFINITY);
#pragma unroll
    for (int c = 0; c < C; ++c) {
        if constexpr (TRACE) {
#pragma unroll
            for (int k = 0; k < U; ++k) R.S[c][k] = 0;
        }
    }
    LaneScalars<C> ls;
    float best[C];
    int bestcol[C], beststart[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        ls.prevleft[c] = INFINITY; ls.prevleft_s[c] = 0; ls.right[c] = INFINITY; ls.right_s[c] = 0;
        best[c] = INFINITY; bestcol[c] = 0x7fffffff; beststart[c] = 0;
    }

    // band / row / round of chain 0 at this warp's first step t = u_min
    int b0 = -C * lane;
    int p0 = (b0 < 0) ? -1 : 0;
    int r0 = (b0 < 0) ? b0 + Pd : 0;

    // warp g runs steps [32*C*g, 32*C*g + span): its lanes' bands cover [0, Pl*Pd)
    const int span = (32 * C - 1 + Mtot_bands + K - 1) / K * K;
    const int t_begin = u_min;
    const int t_end = t_begin + span;
    // a predecessor never publishes past its own end: the successor's trailing
    // (idle-band) chunks must not wait for more
    const int pred_end = t_end - 32 * C;                 // = t_end of warp gw-1
    const int last_end = 32 * C * (G - 1) + span;        // = t_end of warp G-1
    // Tail skip (P.tail_skip, calls that consume no end column): in the unit's last round a
    // warp whose strips all lie beyond the reference (the partial last round of the whole
    // reference: config 2 has 26.04 rounds) would compute only +inf cells; it stops once its
    // bands of the earlier rounds are done (t_stop) and then publishes its nominal end, so
    // every neighbour's wait is unchanged.  Monotone in g: the skipping warps are a suffix.
    // The few steps a skipping warp runs into the last round read +inf reference samples (and,
    // past its predecessor's stop, stale inbox entries): +inf cells, never folded -- no lane
    // reaches row N-1 of that round before t_stop when N >= 32C + K.
    const int t_stop = (!CKPT && !TRACE && P.tail_skip && Pl > 1 && N >= 32 * C + K && ((long)(pa + Pl - 1) * V + u_min) * WC >= (long)P.M)
                           ? t_begin + (32 * C - 1 + Mtot_bands - Pd + K - 1) / K * K : t_end;
    const unsigned FULL = 0xffffffffu;

    // Reference strips for the lanes' round transitions are staged in shared memory
    // one round ahead (pf_round = round currently staged).
    float* ystage = reinterpret_cast<float*>(smem + L.off_stage) + warp * (32 * C * WC);
    int pf_round = 0;                                        // local round staged
    stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa, lane);

    // One step on the slow path (rotation offset 0 before and after): per-lane round
    // transitions before, and last-row folds after, the step's cells.
    // One step on the slow path at rotation offset H (H+1 after): per-lane round
    // transitions before, and last-row folds after, the step's cells.  Only the two
    // per-lane event blocks branch; everything else is select/predicated code.
    // A chain entering a round past the unit's last one (pc >= Pl) reads a stale
    // staged strip: its cells are never folded nor handed to the boundary ring.
    const float* ylane = ystage + lane * C * WC;
    const E* in_w0 = bnd;                                     // warp 0's inbox = the boundary ring
    auto slow_step = [&](auto hc, int t) {
        constexpr int H = decltype(hc)::value;
        float lin = __shfl_up_sync(FULL, ls.right[C - 1], 1);
        int lins = 0;
        if constexpr (TRACE) lins = __shfl_up_sync(FULL, ls.right_s[C - 1], 1);
        {
            E e = (gw == 0) ? in_w0[r0] : my_in[(t - 1) & (RS - 1)];
            const bool inf_in = gw == 0 && p0 < 1 && lead_inf;   // first round of the first segment
            if (lane == 0) {
                lin = inf_in ? INFINITY : e.d;
                if constexpr (TRACE) lins = inf_in ? 0 : e.s;
            }
        }
        int rcs[C], pcs[C];                      // chain c is at row r0-c of round pc
#pragma unroll
        for (int c = 0; c < C; ++c) {
            rcs[c] = (r0 >= c) ? r0 - c : r0 - c + Pd;
            pcs[c] = (r0 >= c) ? p0 : p0 - 1;
        }
#pragma unroll
        for (int c = 0; c < C; ++c)
            if (rcs[c] == 0)
                enter_strip<C, WC, TRACE>(R, Y, c, (long)(pa + pcs[c]) * V + u0 + c, ylane + c * WC, ls, H,
                                          SPEC ? zrow : 0.0f);
        const XRow<C> x = load_xrow<C, XS>(xs, r0, Pd);
        row_cells<C, WC, FMA, TRACE, H>(R, Y, x, lin, lins, ls, nz);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (rcs[c] == N - 1 && pcs[c] >= 0 && pcs[c] < Pl)
                fold_last_row<C, WC, TRACE>(R, c, (int)(((long)(pa + pcs[c]) * V + u0 + c) * WC), best[c],
                                            bestcol[c], beststart[c], H + 1);
        }
        {
            E o;
            o.d = ls.right[C - 1];
            if constexpr (TRACE) o.s = ls.right_s[C - 1];
            const int bl = b0 - (C - 1);                 // band of the last chain, row rcs[C-1]
            E* dst = has_succ_ring ? succ_ring + (t & (RS - 1)) : succ_ring + rcs[C - 1];
            if (lane == 31 && (has_succ_ring || (bl >= 0 && bl < Mtot_bands))) *dst = o;
        }
        ++b0;
        if (++r0 == Pd) { r0 = 0; ++p0; }
    };

    // Warp-uniform period bookkeeping, kept incrementally (no integer division in the
    // hot loop; ncu r01: the modulo-based version cost ~150 instructions per period):
    // rw = row of band tg-u_min (lane 0, chain 0) in [0, Pd), pw = its round.  Over a
    // period the warp's bands cover rows [rw-32C+1, rw+U-1] (unreduced).
    int rw = 0, pw = 0;
    int stage_t = u_max + 1;                                 // step at which round pf_round+1 is staged
    const float* xb[NC];                                      // per-lane row-sample pointers (rows r0+j)
    auto reset_xb = [&]() {
#pragma unroll
        for (int j = 0; j < NC; ++j) {
            int rr = r0 + j;
            if (rr >= Pd) rr -= Pd;
            xb[j] = XS ? xs + rr : xs + (long)xrow_index(rr, Pd, NC) * XC;
        }
    };
    reset_xb();
    const int Nm1 = N - 1;

    for (int t0 = t_begin; t0 < t_stop; t0 += K) {
        // ---- chunk-level flow control (all lanes, warp-uniform)
        {
            const int np = gw > 0 ? min(t0 + K - 1, pred_end)
                                  : (t0 + K - 1 >= Pd ? min(t0 + K - Pd + u_last, last_end) : INT_MIN);
            const int ns = has_succ_ring ? t0 + K - RS + 1 : INT_MIN;
            wait_uniform(pp + warp, np, pred_remote, cp + warp, ns, succ_remote);
        }

        // ---- per PS = SDTW_FAST_PERIODS rotation periods (U steps each): "fast" when no
        // lane of this warp crosses
        // row 0 (round transition) or row N-1 (last-row fold) inside it ->
        // warp-uniform, branch-free steps; otherwise U per-lane slow steps.
#pragma unroll 1
#if SDTW_FAST_RUNS
        // Runs of fast periods: one decision per run (the rows of this warp's lanes stay
        // inside the round and off row N-1 for nf periods), then nf rotation periods of
        // the same unrolled body with the ring / row pointers advanced per period.
        for (int s = 0; s < K;) {
            const int tg = t0 + s;
            const int lo = rw - (32 * C - 1);
            int nf = 0;
            if (lo > 0) {
                const int lim = (lo > Nm1) ? Pd : Nm1;      // first row the window must not reach
                nf = min((lim - rw) / PS, (K - s) / PS);
            }
            if (nf > 0) {
                const bool inf_in = gw == 0 && pw == 0 && lead_inf;
#pragma unroll 1
                for (int f = 0; f < nf; ++f) {
                    const int tp = tg + f * PS;
                    const E* ib0;
                    const E* ib1;
                    if (gw == 0) {
                        ib0 = inf_in ? infs : bnd + rw + f * PS;
                        ib1 = ib0 + 1;
                    } else {
                        ib0 = my_in + ((tp - 1) & (RS - 1));
                        ib1 = my_in + (tp & (RS - 1));
                    }
                    E* ob = has_succ_ring ? succ_ring + (tp & (RS - 1)) : succ_ring + lo + f * PS;
                    static_for<0, PS>([&](auto hc) {
                        constexpr int h = decltype(hc)::value;
                        float lin = __shfl_up_sync(FULL, ls.right[C - 1], 1);
                        int lins = 0;
                        if constexpr (TRACE) lins = __shfl_up_sync(FULL, ls.right_s[C - 1], 1);
                        const E e = (h == 0) ? ib0[0] : ib1[h - 1];
                        if (lane == 0) {
                            lin = e.d;
                            if constexpr (TRACE) lins = e.s;
                        }
                        const XRow<C> x = load_xrow_fast<C, h, XS>(xb);
                        row_cells<C, WC, FMA, TRACE, h % U>(R, Y, x, lin, lins, ls, nz);
                        if (lane == 31) {
                            E o;
                            o.d = ls.right[C - 1];
                            if constexpr (TRACE) o.s = ls.right_s[C - 1];
                            ob[h] = o;
                        }
                    });
#pragma unroll
                    for (int j = 0; j < NC; ++j) xb[j] += (PS / NC) * XC;
                }
                b0 += nf * PS;
                r0 += nf * PS;                               // may land exactly on the next round
                if (r0 >= Pd) { r0 -= Pd; ++p0; }
                s += nf * PS;
                rw += nf * PS;
                if (rw >= Pd) { rw -= Pd; ++pw; }
            } else {
                const int hi = rw + PS - 1;
                const bool hit0 = lo <= 0 || hi >= Pd;
                    if (hit0 || SDTW_ALWAYS_WAIT) {              // a transition reads the staged strips
                        asm volatile("cp.async.wait_all;" ::: "memory");
                        __syncwarp();
                    }
#if SDTW_STATIC_SLOW
                    // unrolled with compile-time rotation (no register moves)
                    static_for<0, PS>([&](auto hc) {
                        slow_step(std::integral_constant<int, decltype(hc)::value % U>{}, tg + decltype(hc)::value);
                        __syncwarp();
                    });
#else
                    // SK steps with compile-time rotation per iteration, then one register
                    // shuffle back to offset 0 (SK divides U)
                    constexpr int SK = (SDTW_SLOW_UNROLL < U) ? SDTW_SLOW_UNROLL : U;
                    static_assert(SDTW_ALT_ORIENT != 2 || C == 1 || (SK % 2 == 0 && U % 2 == 0),
                                  "diagonal orientation needs even rotation groups");
#pragma unroll 1
                    for (int h = 0; h < PS; h += SK) {
                        static_for<0, SK>([&](auto hc) {
                            slow_step(hc, tg + h + decltype(hc)::value);
                            __syncwarp();                    // reconverge before the next step's SHFL
                        });
                        unrotate<SK, C, WC, TRACE>(R);
                    }
#endif
                reset_xb();
                s += PS;
                rw += PS;
                if (rw >= Pd) { rw -= Pd; ++pw; }
            }
            // the last lane of this warp has entered round pf_round: stage round pf_round+1
            if (t0 + s > stage_t && pf_round + 1 < Pl) {
                ++pf_round;
                stage_t += Pd;
                __syncwarp();
                stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa + pf_round, lane);
            }
        }
#else
        for (int s = 0; s < K; s += PS) {
            const int tg = t0 + s;
            const int lo = rw - (32 * C - 1), hi = rw + PS - 1;
            const bool hit0 = lo <= 0 || hi >= Pd;
            const bool hitN = (lo <= Nm1 && Nm1 <= hi) || lo <= Nm1 - Pd || Nm1 + Pd <= hi;
            if (!hit0 && !hitN) {
                // Warp-uniform ring addressing: lane 0 reads its left input for step t
                // from slot t-1 of its inbox (or row rw+h of the boundary ring for
                // warp 0; +inf entries in round 0), lane 31 writes its right edge of
                // step t to slot t of the successor's inbox (or row lo+h of the
                // boundary ring).  tg is a multiple of U and U divides RS, so only the
                // first read of a period can wrap around the inbox.
                const E* ib0;
                const E* ib1;
                if (gw == 0) {
                    ib0 = (pw == 0 && lead_inf) ? infs : bnd + rw;
                    ib1 = ib0 + 1;
                } else {
                    ib0 = my_in + ((tg - 1) & (RS - 1));
                    ib1 = my_in + (tg & (RS - 1));
                }
                E* ob = has_succ_ring ? succ_ring + (tg & (RS - 1)) : succ_ring + lo;
                static_for<0, PS>([&](auto hc) {
                    constexpr int h = decltype(hc)::value;
                    float lin = __shfl_up_sync(FULL, ls.right[C - 1], 1);
                    int lins = 0;
                    if constexpr (TRACE) lins = __shfl_up_sync(FULL, ls.right_s[C - 1], 1);
                    const E e = (h == 0) ? ib0[0] : ib1[h - 1];
                    if (lane == 0) {
                        lin = e.d;
                        if constexpr (TRACE) lins = e.s;
                    }
                    const XRow<C> x = load_xrow_fast<C, h, XS>(xb);
                    row_cells<C, WC, FMA, TRACE, h % U>(R, Y, x, lin, lins, ls, nz);
                    if (lane == 31) {
                        E o;
                        o.d = ls.right[C - 1];
                        if constexpr (TRACE) o.s = ls.right_s[C - 1];
                        ob[h] = o;
                    }
                });
                b0 += PS;
                r0 += PS;                                    // may land exactly on the next round
                if (r0 >= Pd) { r0 -= Pd; ++p0; }
#pragma unroll
                for (int j = 0; j < NC; ++j) xb[j] += (PS / NC) * XC;   // rows r0+j keep their residue (U % C == 0);
                // a wrap of r0 makes the next period slow, which resets xb
            } else {
                if (hit0) {                                  // a transition reads the staged strips
                    asm volatile("cp.async.wait_all;" ::: "memory");
                    __syncwarp();
                }
#if SDTW_STATIC_SLOW
                // unrolled with compile-time rotation (no register moves)
                static_for<0, PS>([&](auto hc) {
                    slow_step(std::integral_constant<int, decltype(hc)::value % U>{}, tg + decltype(hc)::value);
                    __syncwarp();
                });
#else
                // SK steps with compile-time rotation per iteration, then one register
                // shuffle back to offset 0 (SK divides U)
                constexpr int SK = (SDTW_SLOW_UNROLL < U) ? SDTW_SLOW_UNROLL : U;
                static_assert(SDTW_ALT_ORIENT != 2 || C == 1 || (SK % 2 == 0 && U % 2 == 0),
                              "diagonal orientation needs even rotation groups");
#pragma unroll 1
                for (int h = 0; h < PS; h += SK) {
                    static_for<0, SK>([&](auto hc) {
                        slow_step(hc, tg + h + decltype(hc)::value);
                        __syncwarp();                    // reconverge before the next step's SHFL
                    });
                    unrotate<SK, C, WC, TRACE>(R);
                }
#endif
                reset_xb();
            }
            rw += PS;
            if (rw >= Pd) { rw -= Pd; ++pw; }
            // the last lane of this warp has entered round pf_round: stage round pf_round+1
            if (tg + PS > stage_t && pf_round + 1 < Pl) {
                ++pf_round;
                stage_t += Pd;
                __syncwarp();
                stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa + pf_round, lane);
            }
        }

#endif

        // ---- publish progress
        __syncwarp();
        if constexpr (CKPT) {
            // round checkpoints: the last warp copies the wrap-ring rows it wrote in this chunk
            // (its last chain's bands t - u_max for t in [t0, t0+K); K < Pd, so none has been
            // overwritten yet) to global memory -- coalesced, once per chunk, off the fast path
            if (!has_succ_ring) {
                for (int t = t0 + lane; t < t0 + K; t += 32) {
                    const int b = t - u_max;
                    if (b >= 0 && b < Mtot_bands) {
                        const int pr = b / Pd, row = b - pr * Pd;
                        ckb[(long)pr * PdMax + row] = bnd[row].d;
                    }
                }
            }
        }
        if (lane == 31) st_release_hop(succ_pp, t0 + K, succ_remote);
        if (lane == 0 && gw > 0) st_release_hop(pred_cp, t0 + K, pred_remote);
    }
    // a tail-skipping warp consumes nothing more: its (non-skipping) predecessor must never
    // wait for ring space again (reset by the next unit's prologue)
    if (t_stop < t_end) {      // tail skipped: nominal end for the successor (and warp 0), and the
        if (lane == 31) st_release_hop(succ_pp, t_end, succ_remote);        // predecessor never
        if (lane == 0 && gw > 0) st_release_hop(pred_cp, INT_MAX / 2, pred_remote);   // waits on us again
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
        if constexpr (CLUSTER) {
            Partial* dst = cluster.map_shared_rank(red + 32, 0);
            dst[rank] = Partial{bc, bj, bs, 0};
        }
    }
    if constexpr (CLUSTER) cluster.sync();
    if (rank == 0 && threadIdx.x == 0) {
        if constexpr (CLUSTER) {
            for (int k = 1; k < CL; ++k) {
                const Partial pr = red[32 + k];
                if (better(pr.cost, pr.col, bc, bj)) { bc = pr.cost; bj = pr.col; bs = pr.start; }
            }
        }
        if ((!CLUSTER || SDTW_SPEC_CLUSTER == 2) && P.persistent) {
            reinterpret_cast<Partial*>(P.cand)[(long)q * P.S + seg] = Partial{bc, bj, bs, 0};
        } else if (*P.err_flag == 0) {
            if (bj == 0x7fffffff) { bj = 0; bs = 0; }   // every cell overflowed (raw mode only)
            P.out_cost[q] = bc;
            P.out_end[q] = bj;
            if (TRACE && P.out_start) P.out_start[q] = bs;
        }
    }
    if ((!CLUSTER || SDTW_SPEC_CLUSTER == 2) && P.persistent) {
        // hand this segment's last column to the next segment of the query
        if (spec || seg + 1 < P.S) {
            E* bo = reinterpret_cast<E*>(P.bnd_g) + (spec ? (long)q * P.S + seg : (long)q) * PdMax;
            for (int r = threadIdx.x; r < Pd; r += blockDim.x) bo[r] = bnd[r];
        }
        if constexpr (BDP) {
            if (spec && P.col_out && *P.err_flag == 0)       // no partial results on error
                for (int r = threadIdx.x; r < N; r += blockDim.x) P.col_out[(long)q * N + r] = bnd[r].d;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (spec) st_release_gpu(P.seg_done + q * P.S + seg, 1);
            else st_release_gpu(P.seg_done + q, seg + 1);
            if (P.unit_log && unit_sh[1] < P.Z * P.S) P.unit_log[4L * unit_sh[1] + 3] = globaltimer_ns();
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    }   // unit loop
}

// Persistent scheduling epilogue: per query, the lexicographic (cost, col) minimum
// over its segments' candidates (and that candidate's start column).
// XG kernels: the query rows of every query in the shared-memory pair layout of the two-chain
// kernel (row r -> word xrow_index(r, Pd, 2) = (x_r, x_{r-1}), rows >= N zero), in global
// memory, PdMax * 2 floats per query; Pd per query = max(N_q, need) for ragged batches.
static __global__ void __launch_bounds__(256) xg_layout_kernel(const float* __restrict__ X, int N, int PdMax, int need,
                                                               const int64_t* __restrict__ qoff,
                                                               const int* __restrict__ qlen, float* xg) {
    const int q = blockIdx.x;
    int n = N, Pd = PdMax;
    const float* xq = X + (long)q * N;
    if (qlen) {
        n = qlen[q];
        Pd = max(n, need);
        xq = X + qoff[q];
    }
    float* base = xg + (long)q * PdMax * 2;
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        float* dst = base + (long)xrow_index(r, Pd, 2) * 2;
        const int r1 = r >= 1 ? r - 1 : r - 1 + Pd;
        dst[0] = r < n ? xq[r] : 0.0f;
        dst[1] = r1 < n ? xq[r1] : 0.0f;
    }
}

static __global__ void finalize_kernel(const Partial* __restrict__ cand, int Z, int S, const int* err_flag, float* out_cost,
                                int64_t* out_end, int64_t* out_start) {
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Z || *err_flag) return;
    Partial b = cand[(long)q * S];
    for (int s = 1; s < S; ++s) {
        const Partial c = cand[(long)q * S + s];
        if (better(c.cost, c.col, b.cost, b.col)) b = c;
    }
    if (b.col == 0x7fffffff) { b.col = 0; b.start = 0; }   // every cell overflowed (raw mode only)
    out_cost[q] = b.cost;
    out_end[q] = b.col;
    if (out_start) out_start[q] = b.start;
}

// Speculative segments epilogue, one CTA per query.  Unit kinds:
// A_s = k in [0, Sg) (first Rc rounds of segment s, +inf left boundary), B_s = Sg + s
// (the rest of segment s), C_s = 2Sg + s - 1 for s >= 1 (A_s's rounds again, left
// boundary = B_{s-1}'s end column, no free start).  The exact DP is the cell-wise min of
// the free DP (A, B) and the boundary DP (C) -- the cell is monotone in its min input
// and rounding is monotone -- and once the boundary DP is >= the free DP on a whole
// column it stays so, so: result = lexmin over the A/B candidates and, per segment
// whose C end column is >= the A end column on rows [0, N) ("overtaken"), its C
// candidate.  With start columns (stride 2: {d, s} entries) the check is strict (C > A,
// or both +inf) and an exact (cost, col) tie between the best A/B and the best C
// candidate is ambiguous too: on strictly-won cells the winner's start is the true one,
// on ties the priority rule of the merged DP decides.  A query with a
// segment not overtaken (or such a tie) is marked for recomputation (fix[q] = 1).
static __global__ void finalize_spec_kernel(const Partial* __restrict__ cand, const void* __restrict__ bnd_v, int Z,
                                            int S, int Sg, int PdMax, int N, const int* qlen, const int* err_flag,
                                            float* out_cost, int64_t* out_end, int64_t* out_start, int* fix,
                                            int half = 0) {
    const int q = blockIdx.x;
    if (q >= Z || *err_flag) return;
    if (qlen) N = qlen[q];                                 // ragged batch: this query's rows
    const bool trace = out_start != nullptr;
    const int es = trace ? 2 : 1;                          // floats per boundary entry
    const float* bnd_g = static_cast<const float*>(bnd_v);
    const __half* bnd_h = static_cast<const __half*>(bnd_v);   // packed-half kernel: binary16 entries
    const Partial* cq = cand + (long)q * S;
    Partial b = cq[0];
    for (int k = 1; k < 2 * Sg; ++k) {
        const Partial c = cq[k];
        if (better(c.cost, c.col, b.cost, b.col)) b = c;
    }
    Partial bc{INFINITY, 0x7fffffff, 0, 0};                // best correction candidate
    int undominated = 0;
    for (int s = 1; s < Sg; ++s) {
        const long ao = ((long)q * S + s) * PdMax, co = ((long)q * S + 2 * Sg + s - 1) * PdMax;
        int lt = 0;
        for (int r = threadIdx.x; r < N; r += blockDim.x) {
            const float av = half ? __half2float(bnd_h[ao + r]) : bnd_g[(ao + r) * es];
            const float cv = half ? __half2float(bnd_h[co + r]) : bnd_g[(co + r) * es];
            lt |= trace ? !(cv > av || (cv == INFINITY && av == INFINITY)) : cv < av;
        }
        lt = __syncthreads_or(lt);
        if (lt) { undominated = 1; continue; }
        const Partial cc = cq[2 * Sg + s - 1];
        if (better(cc.cost, cc.col, bc.cost, bc.col)) bc = cc;
    }
    if (threadIdx.x == 0) {
        if (trace && bc.cost == b.cost && bc.col == b.col && b.col != 0x7fffffff) undominated = 1;
        if (better(bc.cost, bc.col, b.cost, b.col)) b = bc;
        if (b.col == 0x7fffffff) { b.col = 0; b.start = 0; }   // every cell overflowed (raw mode only)
        out_cost[q] = b.cost;
        out_end[q] = b.col;
        if (trace) out_start[q] = b.start;
        fix[q] = undominated;
    }
}

}  // namespace sdtw
