// sdtw_dp2.cuh -- the two-chains-per-lane wavefront DP kernel for the reduced-precision
// variants: packed half (the paper's own precision, PAPER.md P:L98
// "__half2", "__hmin2") and the uint8-codebook integer path (NEXT-3, PAPER.md P:L165,
// sdtw_q8.cuh).
//
// Same schedule as sdtw_dp.cuh (ring of warps, rotating register file, fast runs and
// slow periods, chunked release/acquire hand-offs, persistent (query, round-segment)
// units, speculative segments); only the lane arithmetic changes, supplied by a policy A:
//   Half2Arith  a lane's two chains share one 32-bit __half2 register per column (chain 0
//               in the low half), so one cell pair is VHMNMX (3-input half2 min, both
//               chains) + HADD2 (x - y) + HFMA2 (t*t + m) = 1.5 SASS per cell (f32x2: 2).
//               Every value is rounded to binary16 after every operation (the oracle's
//               `half=True` mode, tests/test_oracle16_pins.py); queries and reference are
//               rounded to binary16 when they enter shared memory / registers.  Costs
//               overflow to +inf above 65504.
//   Q8Arith<P>  uint8 codes, int32 costs (sdtw_q8.cuh): per cell VIMNMX3 + IADD + IMAD
//               (+ the INF-pruning select when P).
// Start index, clusters and the dual-query layout are not provided in these precisions.
// The per-unit (cost, column) candidates carry A::key(v), an order-preserving fp32 image
// of the chain value, so the finalize kernels of sdtw_dp.cuh serve every precision.
#pragma once
#include <cuda_fp16.h>
#include "sdtw_dp.cuh"

namespace sdtw {

struct Half2Arith {
    using V = __half2;      // one column of both chains
    using S = __half;       // one chain value (ring / boundary entries)
    using XW = unsigned;    // shared-memory word (x_r, x_{r-1})
    static constexpr int kSBytes = 2, kXWBytes = 4;
    static constexpr bool kMaskPad = false;    // padded columns hold +inf: never the minimum
    __device__ static __forceinline__ S inf() { return __ushort_as_half((unsigned short)0x7C00); }
    __device__ static __forceinline__ S zero() { return __ushort_as_half((unsigned short)0); }
    __device__ static __forceinline__ V splat(S v) { return __halves2half2(v, v); }
    __device__ static __forceinline__ V with(V p, int c, S v) {
        return c ? __halves2half2(__low2half(p), v) : __halves2half2(v, __high2half(p));
    }
    __device__ static __forceinline__ S get(V p, int c) { return c ? __high2half(p) : __low2half(p); }
    __device__ static __forceinline__ XW xword(float a, float b) {
        const __half2 h = __halves2half2(__float2half_rn(a), __float2half_rn(b));
        return *reinterpret_cast<const unsigned*>(&h);
    }
    __device__ static __forceinline__ V xval(XW w) { return *reinterpret_cast<const __half2*>(&w); }
    __device__ static __forceinline__ S yval(float y) { return __float2half_rn(y); }
    // left inputs of a step: chain 0 <- lane-1's chain 1 (or the inbox e), chain 1 <- own chain 0
    __device__ static __forceinline__ V left_in(V right, S e, bool use_in) {
        const unsigned s = __shfl_up_sync(0xffffffffu, *reinterpret_cast<const unsigned*>(&right), 1);
        const __half c0 = use_in ? e : __high2half(*reinterpret_cast<const __half2*>(&s));
        return __halves2half2(c0, __low2half(right));
    }
    __device__ static __forceinline__ V cell(V dg, V up, V left, V xx, V y, int) {
        const __half2 m = __hmin2(__hmin2(dg, up), left);
        const __half2 t = __hsub2(xx, y);
        return __hfma2(t, t, m);
    }
    __device__ static __forceinline__ float key(S v) { return __half2float(v); }
};

struct SmemLayout2 {
    int off_ctr, off_red, off_inf, off_x, off_bnd, off_ring, off_stage, bytes;
};
// sb: bytes per chain value (ring / boundary entries), xwb: bytes per (x_r, x_{r-1}) word
__host__ __device__ inline SmemLayout2 smem_layout2(int sb, int xwb, int WC, int GW, int Pd, int RS) {
    SmemLayout2 L;
    int o = 0;
    L.off_ctr = o;  o += 3 * 32 * 4;
    L.off_red = o;  o += 16 * (32 + 16);
    L.off_inf = o;  o += 64 * sb;                             // +inf entries (round 0)
    o = (o + 15) & ~15;
    L.off_x = o;    o += xrow_stride(Pd, 2) * 2 * xwb;        // (x_r, x_{r-1}) words, by row parity
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * sb;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * sb;
    o = (o + 15) & ~15;
    L.off_stage = o; o += GW * 32 * 2 * WC * 4;               // fp32 strips, converted on entry
    L.bytes = (o + 15) & ~15;
    return L;
}
template <class A>
__host__ __device__ inline SmemLayout2 smem_layout2(int WC, int GW, int Pd, int RS) {
    return smem_layout2(A::kSBytes, A::kXWBytes, WC, GW, Pd, RS);
}

template <class A, int WC> struct Row2 {
    static constexpr int U = WC + 1;
    typename A::V D[U];
    __device__ __forceinline__ static constexpr int slot(int w, int h) { return ((w - h) % U + U) % U; }
};

// One row of both chains' strips at rotation offset H: lin = (chain 0's left input, chain
// 1's left input); pd = the diag inputs of column 0 (updated); right = new right edges.
template <class A, int WC, int H>
__device__ __forceinline__ void row2(Row2<A, WC>& R, const typename A::V (&Yv)[WC], typename A::V xx,
                                     typename A::V lin, typename A::V& pd, typename A::V& right, int prm) {
    using RR = Row2<A, WC>;
    using V = typename A::V;
    V left = lin;
    const V d0 = pd;
    pd = lin;
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);
        const V up = R.D[ku];
        const V dg = (w == 0) ? d0 : R.D[kd];
        const V v = A::cell(dg, up, left, xx, Yv[w], prm);
        R.D[kd] = v;
        left = v;
    }
    right = left;
}

template <class A, int SH, int WC>
__device__ __forceinline__ void unrotate2(Row2<A, WC>& R) {
    Row2<A, WC> T;
#pragma unroll
    for (int w = 0; w < Row2<A, WC>::U; ++w) T.D[w] = R.D[Row2<A, WC>::slot(w, SH)];
    R = T;
}

// prm: the policy's per-launch integer parameter (Q8Arith: the squared pruning threshold)
template <class A, int WC>
__global__ void __launch_bounds__(256, 2) sdtw_dp2_kernel(const DpParams P) {
    static_assert(((WC + 1) & WC) == 0 && 64 % (WC + 1) == 0, "rotation period U = WC+1 must divide 64");
    extern __shared__ __align__(16) unsigned char smem[];
    using RR = Row2<A, WC>;
    using V = typename A::V;
    using S = typename A::S;
    using XW = typename A::XW;
    constexpr int C = 2;
    constexpr int U = RR::U;
    constexpr int PS = U;
    const int GW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = GW;
    const int gw = warp;
    const int V_ = 32 * C * G;        // virtual lanes of the ring
    const int PdMax = P.Pd, K = P.K, RS = P.RS;
    const SmemLayout2 L = smem_layout2<A>(WC, GW, PdMax, RS);
    const S HINF = A::inf();
    const S HZERO = A::zero();
    const int prm = P.q8_tau2;

    int* pp = reinterpret_cast<int*>(smem + L.off_ctr);
    int* cp = pp + 32;
    XW* xs = reinterpret_cast<XW*>(smem + L.off_x);
    S* bnd = reinterpret_cast<S*>(smem + L.off_bnd);
    S* ring = reinterpret_cast<S*>(smem + L.off_ring);
    Partial* red = reinterpret_cast<Partial*>(smem + L.off_red);
    S* infs = reinterpret_cast<S*>(smem + L.off_inf);

    const bool has_succ_ring = (gw < G - 1);
    S* succ_ring = has_succ_ring ? ring + (warp + 1) * RS : bnd;
    int* succ_pp = has_succ_ring ? pp + warp + 1 : pp;
    int* pred_cp = (gw > 0) ? cp + warp - 1 : nullptr;
    const S* my_in = (gw == 0) ? bnd : ring + warp * RS;
    const int u_min = 32 * C * gw;
    const int u_max = u_min + 32 * C - 1;
    const int u0 = C * (32 * gw + lane);
    const int u_last = V_ - 1;
    const unsigned FULL = 0xffffffffu;

    int* unit_sh = pp + 64;
    for (int unit_iter = 0;; ++unit_iter) {
    int q, seg = 0, pa = 0, pb = P.Pr;
    int in_k = -1;                                  // speculative segments (sdtw_dp.cuh, DpParams::utab)
    S zrow = HZERO;                            // virtual row -1 (+inf: no free start)
    if (P.persistent) {
        if (threadIdx.x == 0) {
            const int raw = atomicAdd(P.counter, 1);
            *unit_sh = (P.order && raw < P.Z * P.S) ? P.order[raw] : raw;
        }
        __syncthreads();
        const int u = *unit_sh;
        __syncthreads();
        if (u >= P.Z * P.S) break;
        q = u % P.Z;
        seg = u / P.Z;
        int wait_slot = -1, wait_val = 0;
        if (P.utab) {
            const int4 d = P.utab[seg];
            pa = d.x; pb = d.y; in_k = d.z; zrow = d.w ? HINF : HZERO;
            if (in_k >= 0) { wait_slot = q * P.S + in_k; wait_val = 1; }
        } else {
            pa = (int)((long)seg * P.Pr / P.S);
            pb = (int)((long)(seg + 1) * P.Pr / P.S);
            if (seg > 0) { wait_slot = q; wait_val = seg; }
        }
        if (wait_slot >= 0) {
            long n = 0;
            while (ld_acquire_gpu(P.seg_done + wait_slot) < wait_val) {
                __nanosleep(256);
                if (++n == (1LL << 26)) { printf("sdtw16 watchdog: unit %d waits segment\n", u); __trap(); }
            }
        }
        __syncthreads();
    } else {
        if (unit_iter > 0) break;
        q = blockIdx.x;
    }
    int N = P.N, Pd = PdMax;
    const float* xq = P.X + (long)q * N;
    if (P.qlen) {
        N = P.qlen[q];
        Pd = max(N, P.need);
        xq = P.X + P.qoff[q];
    }
    const int Pl = pb - pa;
    const int Mtot_bands = Pl * Pd;

    // prologue: query rows -> (x_r, x_{r-1}) words, boundary ring, counters
    const bool spec = P.utab != nullptr;
    const S* bg = reinterpret_cast<const S*>(P.bnd_g) + (spec ? (long)q * P.S + max(in_k, 0) : (long)q) * PdMax;
    const bool bnd_in = spec ? in_k >= 0 : pa > 0;
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        const int rp = (r >= 1) ? r - 1 : r - 1 + Pd;
        xs[xrow_index(r, Pd, 2)] = A::xword((r < N) ? xq[r] : 0.0f, (rp < N) ? xq[rp] : 0.0f);
        bnd[r] = bnd_in ? bg[r] : HINF;
    }
    if (threadIdx.x < 64) infs[threadIdx.x] = HINF;
    if (threadIdx.x < 32) {
        pp[threadIdx.x] = 0;
        cp[threadIdx.x] = 32 * C * (threadIdx.x + 1);
    }
    __syncthreads();

    RR R;
    V Yh[WC];
    const V INF2 = A::splat(HINF);
#pragma unroll
    for (int k = 0; k < U; ++k) R.D[k] = INF2;
#pragma unroll
    for (int w = 0; w < WC; ++w) Yh[w] = INF2;
    V pd = INF2, right = INF2;
    float best[C] = {INFINITY, INFINITY};
    int bestcol[C] = {0x7fffffff, 0x7fffffff};

    int b0 = -C * lane;
    int p0 = (b0 < 0) ? -1 : 0;
    int r0 = (b0 < 0) ? b0 + Pd : 0;
    const int span = (32 * C - 1 + Mtot_bands + K - 1) / K * K;
    const int t_begin = u_min;
    const int t_end = t_begin + span;
    const int pred_end = t_end - 32 * C;
    const int last_end = 32 * C * (G - 1) + span;
    // tail skip (as in sdtw_dp.cuh): a warp whose strips in the reference's partial last round
    // all start at or beyond M stops after its earlier bands and publishes its nominal end
    const int t_stop = (P.tail_skip && Pl > 1 && N >= 32 * C + K && ((long)(pa + Pl - 1) * V_ + u_min) * WC >= (long)P.M)
                           ? t_begin + (32 * C - 1 + Mtot_bands - Pd + K - 1) / K * K : t_end;

    float* ystage = reinterpret_cast<float*>(smem + L.off_stage) + warp * (32 * C * WC);
    int pf_round = 0;
    stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V_, u_min, pa, lane);
    const float* ylane = ystage + lane * C * WC;

    // left inputs of the step: chain 0 <- lane-1's chain 1 (or the inbox), chain 1 <- own chain 0
    auto left_in = [&](S in0, bool use_in) { return A::left_in(right, in0, use_in); };

    auto slow_step = [&](auto hc, int t) {
        constexpr int H = decltype(hc)::value;
        const S e = (gw == 0) ? bnd[r0] : my_in[(t - 1) & (RS - 1)];
        const bool inf_in = gw == 0 && p0 < 1 && pa == 0;
        const V lin = left_in(inf_in ? HINF : e, lane == 0);
        int rcs[C], pcs[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            rcs[c] = (r0 >= c) ? r0 - c : r0 - c + Pd;
            pcs[c] = (r0 >= c) ? p0 : p0 - 1;
        }
        V pdv = pd;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (rcs[c] == 0) {                               // round transition of chain c
                const float* ys = ylane + c * WC;
#pragma unroll
                for (int w = 0; w < WC; ++w) Yh[w] = A::with(Yh[w], c, A::yval(ys[w]));
#pragma unroll
                for (int k = 0; k < U; ++k) R.D[k] = A::with(R.D[k], c, zrow);
                pdv = A::with(pdv, c, zrow);
            }
        }
        pd = pdv;
        const V xx = A::xval(xs[xrow_index(r0, Pd, 2)]);
        row2<A, WC, H>(R, Yh, xx, lin, pd, right, prm);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (rcs[c] == N - 1 && pcs[c] >= 0 && pcs[c] < Pl) {     // last-row fold of chain c
                const int col0 = (int)(((long)(pa + pcs[c]) * V_ + u0 + c) * WC);
                float mv = INFINITY;
                int mj = 0x7fffffff;
#pragma unroll
                for (int w = 0; w < WC; ++w) {                      // strict <: smallest column
                    const float v = A::key(A::get(R.D[RR::slot(w, H + 1)], c));
                    if ((!A::kMaskPad || col0 + w < P.M) && v < mv) { mv = v; mj = col0 + w; }
                }
                if (mv < best[c]) { best[c] = mv; bestcol[c] = mj; }
            }
        }
        {
            const int bl = b0 - (C - 1);
            S* dst = has_succ_ring ? succ_ring + (t & (RS - 1)) : succ_ring + rcs[C - 1];
            if (lane == 31 && (has_succ_ring || (bl >= 0 && bl < Mtot_bands))) *dst = A::get(right, 1);
        }
        ++b0;
        if (++r0 == Pd) { r0 = 0; ++p0; }
    };

    int rw = 0, pw = 0;
    int stage_t = u_max + 1;
    const XW* xb[2];
    auto reset_xb = [&]() {
#pragma unroll
        for (int j = 0; j < 2; ++j) {
            int rr = r0 + j;
            if (rr >= Pd) rr -= Pd;
            xb[j] = xs + xrow_index(rr, Pd, 2);
        }
    };
    reset_xb();
    const int Nm1 = N - 1;

    for (int t0 = t_begin; t0 < t_stop; t0 += K) {
        {
            const int np = gw > 0 ? min(t0 + K - 1, pred_end)
                                  : (t0 + K - 1 >= Pd ? min(t0 + K - Pd + u_last, last_end) : INT_MIN);
            const int ns = has_succ_ring ? t0 + K - RS + 1 : INT_MIN;
            wait_uniform(pp + warp, np, false, cp + warp, ns, false);
        }
        for (int s = 0; s < K;) {
            const int tg = t0 + s;
            const int lo = rw - (32 * C - 1);
            int nf = 0;
            if (lo > 0) {
                const int lim = (lo > Nm1) ? Pd : Nm1;
                nf = min((lim - rw) / PS, (K - s) / PS);
            }
            if (nf > 0) {
                const bool inf_in = gw == 0 && pw == 0 && pa == 0;
#pragma unroll 1
                for (int f = 0; f < nf; ++f) {
                    const int tp = tg + f * PS;
                    const S* ib0;
                    const S* ib1;
                    if (gw == 0) {
                        ib0 = inf_in ? infs : bnd + rw + f * PS;
                        ib1 = ib0 + 1;
                    } else {
                        ib0 = my_in + ((tp - 1) & (RS - 1));
                        ib1 = my_in + (tp & (RS - 1));
                    }
                    S* ob = has_succ_ring ? succ_ring + (tp & (RS - 1)) : succ_ring + lo + f * PS;
                    static_for<0, PS>([&](auto hc) {
                        constexpr int h = decltype(hc)::value;
                        const S e = (h == 0) ? ib0[0] : ib1[h - 1];
                        const V lin = left_in(e, lane == 0);
                        // rows r0+h of this period: residue class (r0+h)&1, index (r0+h)>>1
                        const V xx = A::xval(xb[h & 1][h >> 1]);
                        row2<A, WC, h % U>(R, Yh, xx, lin, pd, right, prm);
                        if (lane == 31) ob[h] = A::get(right, 1);
                    });
                    xb[0] += PS / 2;
                    xb[1] += PS / 2;
                }
                b0 += nf * PS;
                r0 += nf * PS;
                if (r0 >= Pd) { r0 -= Pd; ++p0; }
                s += nf * PS;
                rw += nf * PS;
                if (rw >= Pd) { rw -= Pd; ++pw; }
            } else {
                const int hi = rw + PS - 1;
                if (lo <= 0 || hi >= Pd) {
                    asm volatile("cp.async.wait_all;" ::: "memory");
                    __syncwarp();
                }
#pragma unroll 1
                for (int h = 0; h < PS; h += 2) {
                    static_for<0, 2>([&](auto hc) {
                        slow_step(hc, tg + h + decltype(hc)::value);
                        __syncwarp();
                    });
                    unrotate2<A, 2, WC>(R);
                }
                reset_xb();
                s += PS;
                rw += PS;
                if (rw >= Pd) { rw -= Pd; ++pw; }
            }
            if (t0 + s > stage_t && pf_round + 1 < Pl) {
                ++pf_round;
                stage_t += Pd;
                __syncwarp();
                stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V_, u_min, pa + pf_round, lane);
            }
        }
        __syncwarp();
        if (lane == 31) st_release_cta(succ_pp, t0 + K);
        if (lane == 0 && gw > 0) st_release_cta(pred_cp, t0 + K);
    }
    if (t_stop < t_end) {      // tail skipped: nominal end for the successor, no more waits for ring space
        if (lane == 31) st_release_cta(succ_pp, t_end);
        if (lane == 0 && gw > 0) st_release_cta(pred_cp, INT_MAX / 2);
    }

    // (cost, col) over chains, lanes, warps
    float bc = best[0];
    int bj = bestcol[0];
    if (better(best[1], bestcol[1], bc, bj)) { bc = best[1]; bj = bestcol[1]; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float oc = __shfl_xor_sync(FULL, bc, o);
        const int oj = __shfl_xor_sync(FULL, bj, o);
        if (better(oc, oj, bc, bj)) { bc = oc; bj = oj; }
    }
    if (lane == 0) red[warp] = Partial{bc, bj, 0, 0};
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < GW; ++w)
            if (better(red[w].cost, red[w].col, bc, bj)) { bc = red[w].cost; bj = red[w].col; }
        if (P.persistent) {
            reinterpret_cast<Partial*>(P.cand)[(long)q * P.S + seg] = Partial{bc, bj, 0, 0};
        } else if (*P.err_flag == 0) {
            if (bj == 0x7fffffff) bj = 0;
            P.out_cost[q] = bc;
            P.out_end[q] = bj;
        }
    }
    if (P.persistent) {
        if (spec || seg + 1 < P.S) {
            S* bo = reinterpret_cast<S*>(P.bnd_g) + (spec ? (long)q * P.S + seg : (long)q) * PdMax;
            for (int r = threadIdx.x; r < Pd; r += blockDim.x) bo[r] = bnd[r];
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            __threadfence();
            if (spec) st_release_gpu(P.seg_done + q * P.S + seg, 1);
            else st_release_gpu(P.seg_done + q, seg + 1);
        }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    }   // unit loop
}

}  // namespace sdtw
