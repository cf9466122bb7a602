// sdtw_dp16.cuh -- the packed-half wavefront DP kernel (the paper's
// own precision, "__half2", "__hmin2").
//
// Same schedule as sdtw_dp.cuh (ring of warps, rotating register file, fast runs and
// slow periods, chunked release/acquire hand-offs, persistent (query, round-segment)
// units); only the lane arithmetic changes: a lane's two chains share one 32-bit __half2
// register per column (chain 0 in the low half), so one cell pair is
//     VHMNMX (3-input half2 min, both chains) + HADD2 (x - y) + HFMA2 (t*t + m)
// = 1.5 SASS per cell (f32x2: 2).  Every value is rounded to binary16 after every
// operation (the oracle's `half=True` mode, tests/test_oracle16_pins.py); the queries and
// the reference are rounded to binary16 when they enter shared memory / registers.
// Costs overflow to +inf above 65504 (the paper's precision); start index, clusters and the
// dual-query layout are not provided in this precision.
#pragma once
#include <cuda_fp16.h>
#include "sdtw_dp.cuh"

namespace sdtw {

struct SmemLayout16 {
    int off_ctr, off_red, off_inf, off_x, off_bnd, off_ring, off_stage, bytes;
};
__host__ __device__ inline SmemLayout16 smem_layout16(int WC, int GW, int Pd, int RS) {
    SmemLayout16 L;
    int o = 0;
    L.off_ctr = o;  o += 3 * 32 * 4;
    L.off_red = o;  o += 16 * (32 + 16);
    L.off_inf = o;  o += 64 * 2;                              // +inf half entries (round 0)
    o = (o + 15) & ~15;
    L.off_x = o;    o += xrow_stride(Pd, 2) * 2 * 4;          // (x_r, x_{r-1}) half2 words
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * 2;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * 2;
    o = (o + 15) & ~15;
    L.off_stage = o; o += GW * 32 * 2 * WC * 4;               // fp32 strips, rounded on entry
    L.bytes = (o + 15) & ~15;
    return L;
}

__device__ __forceinline__ unsigned h2_bits(__half2 p) { return *reinterpret_cast<unsigned*>(&p); }
__device__ __forceinline__ __half2 h2_from(unsigned u) { return *reinterpret_cast<__half2*>(&u); }
__device__ __forceinline__ __half2 h2_with(__half2 p, int c, __half v) {
    return c ? __halves2half2(__low2half(p), v) : __halves2half2(v, __high2half(p));
}
__device__ __forceinline__ __half h2_get(__half2 p, int c) { return c ? __high2half(p) : __low2half(p); }

template <int WC> struct Row16 {
    static constexpr int U = WC + 1;
    __half2 D[U];
    __device__ __forceinline__ static constexpr int slot(int w, int h) { return ((w - h) % U + U) % U; }
};

// One row of both chains' strips at rotation offset H: lin = (chain 0's left input, chain
// 1's left input); pd = the diag inputs of column 0 (updated); right = new right edges.
template <int WC, int H>
__device__ __forceinline__ void row16(Row16<WC>& R, const __half2 (&Yh)[WC], __half2 xx, __half2 lin,
                                      __half2& pd, __half2& right) {
    using RR = Row16<WC>;
    __half2 left = lin;
    const __half2 d0 = pd;
    pd = lin;
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);
        const __half2 up = R.D[ku];
        const __half2 dg = (w == 0) ? d0 : R.D[kd];
        const __half2 m = __hmin2(__hmin2(dg, up), left);
        const __half2 t = __hsub2(xx, Yh[w]);
        const __half2 v = __hfma2(t, t, m);
        R.D[kd] = v;
        left = v;
    }
    right = left;
}

template <int SH, int WC>
__device__ __forceinline__ void unrotate16(Row16<WC>& R) {
    Row16<WC> T;
#pragma unroll
    for (int w = 0; w < Row16<WC>::U; ++w) T.D[w] = R.D[Row16<WC>::slot(w, SH)];
    R = T;
}

template <int WC>
__global__ void __launch_bounds__(256, 2) sdtw_dp16_kernel(const DpParams P) {
    static_assert(((WC + 1) & WC) == 0 && 64 % (WC + 1) == 0, "rotation period U = WC+1 must divide 64");
    extern __shared__ __align__(16) unsigned char smem[];
    using RR = Row16<WC>;
    constexpr int C = 2;
    constexpr int U = RR::U;
    constexpr int PS = U;
    const int GW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = GW;
    const int gw = warp;
    const int V = 32 * C * G;
    const int PdMax = P.Pd, K = P.K, RS = P.RS;
    const SmemLayout16 L = smem_layout16(WC, GW, PdMax, RS);
    const __half HINF = __ushort_as_half((unsigned short)0x7C00);
    const __half HZERO = __ushort_as_half((unsigned short)0);

    int* pp = reinterpret_cast<int*>(smem + L.off_ctr);
    int* cp = pp + 32;
    unsigned* xs = reinterpret_cast<unsigned*>(smem + L.off_x);
    __half* bnd = reinterpret_cast<__half*>(smem + L.off_bnd);
    __half* ring = reinterpret_cast<__half*>(smem + L.off_ring);
    Partial* red = reinterpret_cast<Partial*>(smem + L.off_red);
    __half* infs = reinterpret_cast<__half*>(smem + L.off_inf);

    const bool has_succ_ring = (gw < G - 1);
    __half* succ_ring = has_succ_ring ? ring + (warp + 1) * RS : bnd;
    int* succ_pp = has_succ_ring ? pp + warp + 1 : pp;
    int* pred_cp = (gw > 0) ? cp + warp - 1 : nullptr;
    const __half* my_in = (gw == 0) ? bnd : ring + warp * RS;
    const int u_min = 32 * C * gw;
    const int u_max = u_min + 32 * C - 1;
    const int u0 = C * (32 * gw + lane);
    const int u_last = V - 1;
    const unsigned FULL = 0xffffffffu;

    int* unit_sh = pp + 64;
    for (int unit_iter = 0;; ++unit_iter) {
    int q, seg = 0, pa = 0, pb = P.Pr;
    int in_k = -1;                                  // speculative segments (sdtw_dp.cuh, DpParams::utab)
    __half zrow = HZERO;                            // virtual row -1 (+inf: no free start)
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

    // prologue: query rows -> half2 (x_r, x_{r-1}) words, boundary ring, counters
    const bool spec = P.utab != nullptr;
    const __half* bg = reinterpret_cast<const __half*>(P.bnd_g) + (spec ? (long)q * P.S + max(in_k, 0) : (long)q) * PdMax;
    const bool bnd_in = spec ? in_k >= 0 : pa > 0;
    for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
        const int rp = (r >= 1) ? r - 1 : r - 1 + Pd;
        const __half a = __float2half_rn((r < N) ? xq[r] : 0.0f);
        const __half b = __float2half_rn((rp < N) ? xq[rp] : 0.0f);
        xs[xrow_index(r, Pd, 2)] = h2_bits(__halves2half2(a, b));
        bnd[r] = bnd_in ? bg[r] : HINF;
    }
    if (threadIdx.x < 64) infs[threadIdx.x] = HINF;
    if (threadIdx.x < 32) {
        pp[threadIdx.x] = 0;
        cp[threadIdx.x] = 32 * C * (threadIdx.x + 1);
    }
    __syncthreads();

    RR R;
    __half2 Yh[WC];
    const __half2 INF2 = __halves2half2(HINF, HINF);
#pragma unroll
    for (int k = 0; k < U; ++k) R.D[k] = INF2;
#pragma unroll
    for (int w = 0; w < WC; ++w) Yh[w] = INF2;
    __half2 pd = INF2, right = INF2;
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

    float* ystage = reinterpret_cast<float*>(smem + L.off_stage) + warp * (32 * C * WC);
    int pf_round = 0;
    stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa, lane);
    const float* ylane = ystage + lane * C * WC;

    // left inputs of the step: chain 0 <- lane-1's chain 1 (or the inbox), chain 1 <- own chain 0
    auto left_in = [&](__half in0, bool use_in) {
        const unsigned s = __shfl_up_sync(FULL, h2_bits(right), 1);
        const __half c0 = use_in ? in0 : __high2half(h2_from(s));
        return __halves2half2(c0, __low2half(right));
    };

    auto slow_step = [&](auto hc, int t) {
        constexpr int H = decltype(hc)::value;
        const __half e = (gw == 0) ? bnd[r0] : my_in[(t - 1) & (RS - 1)];
        const bool inf_in = gw == 0 && p0 < 1 && pa == 0;
        const __half2 lin = left_in(inf_in ? HINF : e, lane == 0);
        int rcs[C], pcs[C];
#pragma unroll
        for (int c = 0; c < C; ++c) {
            rcs[c] = (r0 >= c) ? r0 - c : r0 - c + Pd;
            pcs[c] = (r0 >= c) ? p0 : p0 - 1;
        }
        __half2 pdv = pd;
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (rcs[c] == 0) {                               // round transition of chain c
                const float* ys = ylane + c * WC;
#pragma unroll
                for (int w = 0; w < WC; ++w) Yh[w] = h2_with(Yh[w], c, __float2half_rn(ys[w]));
#pragma unroll
                for (int k = 0; k < U; ++k) R.D[k] = h2_with(R.D[k], c, zrow);
                pdv = h2_with(pdv, c, zrow);
            }
        }
        pd = pdv;
        const __half2 xx = h2_from(xs[xrow_index(r0, Pd, 2)]);
        row16<WC, H>(R, Yh, xx, lin, pd, right);
#pragma unroll
        for (int c = 0; c < C; ++c) {
            if (rcs[c] == N - 1 && pcs[c] >= 0 && pcs[c] < Pl) {     // last-row fold of chain c
                __half2 m2 = R.D[RR::slot(0, H + 1)];
#pragma unroll
                for (int w = 1; w < WC; ++w) m2 = __hmin2(m2, R.D[RR::slot(w, H + 1)]);
                const float mv = __half2float(h2_get(m2, c));
                if (mv < best[c]) {
                    best[c] = mv;
                    const int col0 = (int)(((long)(pa + pcs[c]) * V + u0 + c) * WC);
#pragma unroll
                    for (int w = WC - 1; w >= 0; --w)
                        if (__half2float(h2_get(R.D[RR::slot(w, H + 1)], c)) == mv) bestcol[c] = col0 + w;
                }
            }
        }
        {
            const int bl = b0 - (C - 1);
            __half* dst = has_succ_ring ? succ_ring + (t & (RS - 1)) : succ_ring + rcs[C - 1];
            if (lane == 31 && (has_succ_ring || (bl >= 0 && bl < Mtot_bands))) *dst = __high2half(right);
        }
        ++b0;
        if (++r0 == Pd) { r0 = 0; ++p0; }
    };

    int rw = 0, pw = 0;
    int stage_t = u_max + 1;
    const unsigned* xb[2];
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

    for (int t0 = t_begin; t0 < t_end; t0 += K) {
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
                    const __half* ib0;
                    const __half* ib1;
                    if (gw == 0) {
                        ib0 = inf_in ? infs : bnd + rw + f * PS;
                        ib1 = ib0 + 1;
                    } else {
                        ib0 = my_in + ((tp - 1) & (RS - 1));
                        ib1 = my_in + (tp & (RS - 1));
                    }
                    __half* ob = has_succ_ring ? succ_ring + (tp & (RS - 1)) : succ_ring + lo + f * PS;
                    static_for<0, PS>([&](auto hc) {
                        constexpr int h = decltype(hc)::value;
                        const __half e = (h == 0) ? ib0[0] : ib1[h - 1];
                        const __half2 lin = left_in(e, lane == 0);
                        // rows r0+h of this period: residue class (r0+h)&1, index (r0+h)>>1
                        const __half2 xx = h2_from(xb[h & 1][h >> 1]);
                        row16<WC, h % U>(R, Yh, xx, lin, pd, right);
                        if (lane == 31) ob[h] = __high2half(right);
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
                    unrotate16<2, WC>(R);
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
                stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa + pf_round, lane);
            }
        }
        __syncwarp();
        if (lane == 31) st_release_cta(succ_pp, t0 + K);
        if (lane == 0 && gw > 0) st_release_cta(pred_cp, t0 + K);
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
            __half* bo = reinterpret_cast<__half*>(P.bnd_g) + (spec ? (long)q * P.S + seg : (long)q) * PdMax;
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
