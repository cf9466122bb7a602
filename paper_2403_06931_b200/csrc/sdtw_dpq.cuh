// sdtw_dpq.cuh -- dual-query variant of the wavefront DP kernel (sm_100a).
//
// Same recurrence, mapping, rings and scheduling as sdtw_dp.cuh (see there), but
// every lane carries the SAME reference strips for TWO queries A and B: each cell
// value is an (A, B) pair in one 64-bit register, updated with one FADD2 (the
// reference sample broadcast to both halves) + two FMNMX3 + one FFMA2, i.e. 2 SASS
// per cell, and both queries hit their round transitions and last-row folds at the
// same step (no half-register updates).  With C = 2 chains per lane the two
// chains are independent inside a step, giving two FFMA2 dependency chains per
// warp (ILP 2) -- the measured B200 ceiling of this instruction mix rises from
// ~6.5 TCUPS with one chain per warp to ~8.4 with two (profiles/r01_pipebench2.txt).
// Queries are processed in pairs (2p, 2p+1); an odd batch gets a zero dummy.
#pragma once
#include "sdtw_dp.cuh"

namespace sdtw {

template <bool TRACE> struct Entry2 { float a, b; };
template <> struct Entry2<true> { float a, b; int sa, sb; };

struct Partial2 { Partial a, b; };

__device__ __forceinline__ unsigned long long pmin3(unsigned long long d, unsigned long long u,
                                                    unsigned long long l) {
    return pk(min3f(lo32(d), lo32(u), lo32(l)), min3f(hi32(d), hi32(u), hi32(l)));
}
// (xA - y, xB - y)^2 + (mA, mB): one FADD2 with y broadcast, one FFMA2
template <bool FMA>
__device__ __forceinline__ unsigned long long qcell(unsigned long long xx, float y, unsigned long long mm) {
    unsigned long long tt, vv;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(tt) : "l"(xx), "l"(pk(y, y)));
    if (FMA) {
        asm("fma.rn.f32x2 %0, %1, %1, %2;" : "=l"(vv) : "l"(tt), "l"(mm));
    } else {
        const float t0 = lo32(tt), t1 = hi32(tt);
        vv = pk(__fadd_rn(__fmul_rn(t0, t0), lo32(mm)), __fadd_rn(__fmul_rn(t1, t1), hi32(mm)));
    }
    return vv;
}

template <int C, int WC, bool TRACE> struct QRow {
    static constexpr int U = WC + 1;
    unsigned long long D[C][U];
    int SA[TRACE ? C : 1][TRACE ? U : 1], SB[TRACE ? C : 1][TRACE ? U : 1];
    __device__ __forceinline__ static constexpr int slot(int w, int h) { return ((w - h) % U + U) % U; }
};
template <int C> struct QLane {
    unsigned long long prevleft[C], right[C];
    int pls_a[C], pls_b[C], rs_a[C], rs_b[C];
};

// One row of the lane's strips for both queries at rotation offset H (see row_cells).
template <int C, int WC, bool FMA, bool TRACE, int H>
__device__ __forceinline__ void qrow_cells(QRow<C, WC, TRACE>& R, const float (&Y)[C][WC],
                                           const unsigned long long (&x)[C], unsigned long long lin, int lsa,
                                           int lsb, QLane<C>& ls) {
    using RR = QRow<C, WC, TRACE>;
    unsigned long long left[C], pd[C];
    int sla[C], slb[C], psa[C], psb[C];
#pragma unroll
    for (int c = 0; c < C; ++c) {
        left[c] = (c == 0) ? lin : ls.right[c - 1];
        sla[c] = (c == 0) ? lsa : ls.rs_a[c - 1];
        slb[c] = (c == 0) ? lsb : ls.rs_b[c - 1];
        pd[c] = ls.prevleft[c];
        psa[c] = ls.pls_a[c];
        psb[c] = ls.pls_b[c];
        ls.prevleft[c] = left[c];
        ls.pls_a[c] = sla[c];
        ls.pls_b[c] = slb[c];
    }
#pragma unroll
    for (int w = 0; w < WC; ++w) {
        const int ku = RR::slot(w, H), kd = RR::slot(w - 1, H);
#pragma unroll
        for (int c = 0; c < C; ++c) {            // the C chains are independent within the step
            const unsigned long long up = R.D[c][ku];
            const unsigned long long dg = (w == 0) ? pd[c] : R.D[c][kd];
            const unsigned long long mm = pmin3(dg, up, left[c]);
            const unsigned long long vv = qcell<FMA>(x[c], Y[c][w], mm);
            if constexpr (TRACE) {
                const float ma = lo32(mm), mb = hi32(mm);
                const int sua = R.SA[c][ku], sub = R.SB[c][ku];
                const int sda = (w == 0) ? psa[c] : R.SA[c][kd];
                const int sdb = (w == 0) ? psb[c] : R.SB[c][kd];
                const int sva = (lo32(dg) == ma) ? sda : ((lo32(up) == ma) ? sua : sla[c]);
                const int svb = (hi32(dg) == mb) ? sdb : ((hi32(up) == mb) ? sub : slb[c]);
                R.SA[c][kd] = sva;
                R.SB[c][kd] = svb;
                sla[c] = sva;
                slb[c] = svb;
            }
            R.D[c][kd] = vv;
            left[c] = vv;
        }
    }
#pragma unroll
    for (int c = 0; c < C; ++c) {
        ls.right[c] = left[c];
        ls.rs_a[c] = sla[c];
        ls.rs_b[c] = slb[c];
    }
}

template <int C, int WC, bool TRACE>
__device__ __forceinline__ void qunrotate1(QRow<C, WC, TRACE>& R) {
    using RR = QRow<C, WC, TRACE>;
    QRow<C, WC, TRACE> T;
#pragma unroll
    for (int w = 0; w < RR::U; ++w) {
#pragma unroll
        for (int c = 0; c < C; ++c) {
            T.D[c][w] = R.D[c][RR::slot(w, 1)];
            if constexpr (TRACE) {
                T.SA[c][w] = R.SA[c][RR::slot(w, 1)];
                T.SB[c][w] = R.SB[c][RR::slot(w, 1)];
            }
        }
    }
    R = T;
}

// fold one half (query) of chain c's last row (offset 0)
template <int WC, bool TRACE>
__device__ __forceinline__ void qfold_half(const float (&v)[WC], const int (&sv)[WC], int col0, float& best,
                                           int& bestcol, int& beststart) {
    float m = v[0];
#pragma unroll
    for (int w = 1; w < WC; ++w) m = fminf(m, v[w]);
    if (m < best) {
        best = m;
#pragma unroll
        for (int w = WC - 1; w >= 0; --w)
            if (v[w] == m) {
                bestcol = col0 + w;
                beststart = TRACE ? sv[w] : 0;
            }
    }
}

// row samples of a query pair: row r stores (xA_r, xB_r); rows split by residue mod C
template <int C>
__device__ __forceinline__ unsigned long long qx(const float* xs, int r, int Pd) {
    return reinterpret_cast<const unsigned long long*>(xs)[xrow_index(r, Pd, C)];
}

__host__ __device__ inline SmemLayout smem_layout_q(int C, int WC, bool trace, int GW, int Pd, int RS) {
    SmemLayout L;
    const int ent = trace ? 16 : 8;
    int o = 0;
    L.off_ctr = o;  o += 3 * 32 * 4;
    L.off_red = o;  o += 32 * 32;                       // per-warp Partial2
    L.off_inf = o;  o += 32 * 16;
    o = (o + 15) & ~15;
    L.off_x = o;    o += xrow_stride(Pd, C) * C * 8;
    o = (o + 15) & ~15;
    L.off_bnd = o;  o += Pd * ent;
    o = (o + 15) & ~15;
    L.off_ring = o; o += GW * RS * ent;
    o = (o + 15) & ~15;
    L.off_stage = o; o += GW * 32 * C * WC * 4;
    L.bytes = (o + 15) & ~15;
    return L;
}

// ============================================================================ kernel
// P.Z = number of query PAIRS; P.X = [2*P.Z][N] (the host pads an odd batch);
// outputs / candidates are indexed by query (2*pair + half).
template <int C, int WC, bool FMA, bool TRACE>
__global__ void __launch_bounds__(384) sdtw_dpq_kernel(const DpParams P) {
    static_assert(C == 1 || C == 2, "chains per lane");
    static_assert(((WC + 1) & WC) == 0 && (32 * C) % (WC + 1) == 0 && (WC + 1) % C == 0, "rotation period");
    extern __shared__ __align__(16) unsigned char smem[];
    using E = Entry2<TRACE>;
    using RowT = QRow<C, WC, TRACE>;
    constexpr int U = RowT::U;

    const int GW = blockDim.x >> 5;
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int G = GW;
    const int gw = warp;
    const int V = 32 * C * G;
    const int Pd = P.Pd, N = P.N, K = P.K, RS = P.RS;
    const SmemLayout L = smem_layout_q(C, WC, TRACE, GW, Pd, RS);

    int* pp = reinterpret_cast<int*>(smem + L.off_ctr);
    int* cp = pp + 32;
    int* unit_sh = pp + 64;
    float* xs = reinterpret_cast<float*>(smem + L.off_x);
    E* bnd = reinterpret_cast<E*>(smem + L.off_bnd);
    E* ring = reinterpret_cast<E*>(smem + L.off_ring);
    Partial2* red = reinterpret_cast<Partial2*>(smem + L.off_red);
    E* infs = reinterpret_cast<E*>(smem + L.off_inf);
    float* ystage = reinterpret_cast<float*>(smem + L.off_stage) + warp * (32 * C * WC);

    const bool has_succ_ring = (gw < G - 1);
    E* succ_ring = has_succ_ring ? ring + (warp + 1) * RS : bnd;
    int* succ_pp = has_succ_ring ? pp + warp + 1 : pp;
    int* pred_cp = (gw > 0) ? cp + warp - 1 : nullptr;
    const E* my_in = (gw == 0) ? bnd : ring + warp * RS;
    const int u_min = 32 * C * gw;
    const int u_max = u_min + 32 * C - 1;
    const int u0 = C * (32 * gw + lane);
    const int u_last = V - 1;
    const unsigned FULL = 0xffffffffu;

    for (int unit_iter = 0;; ++unit_iter) {
        // ---- which unit: (query pair qp, rounds [pa, pb))
        int qp, seg = 0, pa = 0, pb = P.Pr;
        if (P.persistent) {
            if (threadIdx.x == 0) {
                const int raw = atomicAdd(P.counter, 1);
                *unit_sh = (P.order && raw < P.Z * P.S) ? P.order[raw] : raw;
            }
            __syncthreads();
            const int u = *unit_sh;
            __syncthreads();
            if (u >= P.Z * P.S) break;
            qp = u % P.Z;
            seg = u / P.Z;
            pa = (int)((long)seg * P.Pr / P.S);
            pb = (int)((long)(seg + 1) * P.Pr / P.S);
            if (seg > 0) {                                  // every thread polls: no split warps
                long n = 0;
                while (ld_acquire_gpu(P.seg_done + qp) < seg) {
                    __nanosleep(256);
                    if (++n == (1LL << 26)) { printf("sdtw watchdog: unit %d waits segment\n", u); __trap(); }
                }
            }
            __syncthreads();
        } else {
            if (unit_iter > 0) break;
            qp = blockIdx.x;
        }
        const int Pl = pb - pa;
        const int Mtot_bands = Pl * Pd;

        // ---- prologue: (xA, xB) rows -> smem, boundary ring, counters
        const float* xa = P.X + (long)(2 * qp) * N;
        const float* xb2 = xa + N;
        const E* bg = reinterpret_cast<const E*>(P.bnd_g) + (long)qp * Pd;
        for (int r = threadIdx.x; r < Pd; r += blockDim.x) {
            float* dst = xs + (long)xrow_index(r, Pd, C) * 2;
            dst[0] = (r < N) ? xa[r] : 0.0f;
            dst[1] = (r < N) ? xb2[r] : 0.0f;
            E e;
            if (pa > 0) {
                e = bg[r];
            } else {
                e.a = INFINITY; e.b = INFINITY;
                if constexpr (TRACE) { e.sa = 0; e.sb = 0; }
            }
            bnd[r] = e;
        }
        if (threadIdx.x < 32) {
            E e;
            e.a = INFINITY; e.b = INFINITY;
            if constexpr (TRACE) { e.sa = 0; e.sb = 0; }
            infs[threadIdx.x] = e;
            pp[threadIdx.x] = 0;
            cp[threadIdx.x] = 32 * C * (threadIdx.x + 1);
        }
        __syncthreads();

        // ---- per-lane state
        RowT R;
        float Y[C][WC];
        QLane<C> ls;
        float best[C][2];
        int bestcol[C][2], beststart[C][2];
        const unsigned long long INF2 = pk(INFINITY, INFINITY);
#pragma unroll
        for (int c = 0; c < C; ++c) {
#pragma unroll
            for (int k = 0; k < U; ++k) {
                R.D[c][k] = INF2;
                if constexpr (TRACE) { R.SA[c][k] = 0; R.SB[c][k] = 0; }
            }
#pragma unroll
            for (int w = 0; w < WC; ++w) Y[c][w] = INFINITY;
            ls.prevleft[c] = INF2; ls.right[c] = INF2;
            ls.pls_a[c] = ls.pls_b[c] = ls.rs_a[c] = ls.rs_b[c] = 0;
            best[c][0] = best[c][1] = INFINITY;
            bestcol[c][0] = bestcol[c][1] = 0x7fffffff;
            beststart[c][0] = beststart[c][1] = 0;
        }
        int b0 = -C * lane;
        int p0 = (b0 < 0) ? -1 : 0;
        int r0 = (b0 < 0) ? b0 + Pd : 0;
        const int span = (32 * C - 1 + Mtot_bands + K - 1) / K * K;
        const int t_begin = u_min;
        const int t_end = t_begin + span;
        const int pred_end = t_end - 32 * C;
        const int last_end = 32 * C * (G - 1) + span;

        int pf_round = 0;
        stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa, lane);

        auto slow_step = [&](int t) {
            unsigned long long lin;
            int lsa = 0, lsb = 0;
            {
                const float la = __shfl_up_sync(FULL, lo32(ls.right[C - 1]), 1);
                const float lb = __shfl_up_sync(FULL, hi32(ls.right[C - 1]), 1);
                lin = pk(la, lb);
                if constexpr (TRACE) {
                    lsa = __shfl_up_sync(FULL, ls.rs_a[C - 1], 1);
                    lsb = __shfl_up_sync(FULL, ls.rs_b[C - 1], 1);
                }
            }
            if (lane == 0) {
                E e;
                if (gw == 0) {
                    if (p0 >= 1 || pa > 0) e = my_in[r0];
                    else { e.a = INFINITY; e.b = INFINITY; if constexpr (TRACE) { e.sa = 0; e.sb = 0; } }
                } else {
                    e = my_in[(t - 1) & (RS - 1)];
                }
                lin = pk(e.a, e.b);
                if constexpr (TRACE) { lsa = e.sa; lsb = e.sb; }
            }
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int rc = (r0 >= c) ? r0 - c : r0 - c + Pd;
                const int pc = (r0 >= c) ? p0 : p0 - 1;
                if (rc == 0) {            // round transition of chain c (both queries)
                    const long strip = (long)(pa + pc) * V + u0 + c;
                    const bool live = pc < Pl;
                    const float* ys = ystage + (lane * C + c) * WC;
#pragma unroll
                    for (int w = 0; w < WC; ++w) Y[c][w] = live ? ys[w] : INFINITY;
#pragma unroll
                    for (int k = 0; k < U; ++k) {
                        R.D[c][k] = 0ull;      // (0.0f, 0.0f): virtual row -1
                        if constexpr (TRACE) { R.SA[c][k] = R.SB[c][k] = (int)(strip * WC) + k + 1; }
                    }
                    ls.prevleft[c] = 0ull;
                    ls.pls_a[c] = ls.pls_b[c] = (int)(strip * WC);
                }
            }
            unsigned long long x[C];
#pragma unroll
            for (int c = 0; c < C; ++c) x[c] = qx<C>(xs, (r0 >= c) ? r0 - c : r0 - c + Pd, Pd);
            qrow_cells<C, WC, FMA, TRACE, 0>(R, Y, x, lin, lsa, lsb, ls);
            qunrotate1<C, WC, TRACE>(R);
#pragma unroll
            for (int c = 0; c < C; ++c) {
                const int rc = (r0 >= c) ? r0 - c : r0 - c + Pd;
                const int pc = (r0 >= c) ? p0 : p0 - 1;
                if (rc == N - 1 && pc >= 0 && pc < Pl) {
                    const int col0 = (int)(((long)(pa + pc) * V + u0 + c) * WC);
                    float va[WC], vb[WC];
                    int sa[WC], sb[WC];
#pragma unroll
                    for (int w = 0; w < WC; ++w) {
                        va[w] = lo32(R.D[c][w]);
                        vb[w] = hi32(R.D[c][w]);
                        sa[w] = TRACE ? R.SA[TRACE ? c : 0][TRACE ? w : 0] : 0;
                        sb[w] = TRACE ? R.SB[TRACE ? c : 0][TRACE ? w : 0] : 0;
                    }
                    qfold_half<WC, TRACE>(va, sa, col0, best[c][0], bestcol[c][0], beststart[c][0]);
                    qfold_half<WC, TRACE>(vb, sb, col0, best[c][1], bestcol[c][1], beststart[c][1]);
                }
            }
            if (lane == 31) {
                E o;
                o.a = lo32(ls.right[C - 1]);
                o.b = hi32(ls.right[C - 1]);
                if constexpr (TRACE) { o.sa = ls.rs_a[C - 1]; o.sb = ls.rs_b[C - 1]; }
                if (has_succ_ring) {
                    succ_ring[t & (RS - 1)] = o;
                } else {
                    const int bl = b0 - (C - 1);
                    if (bl >= 0 && bl < Mtot_bands) succ_ring[fmod_pos(bl, Pd)] = o;
                }
            }
            ++b0;
            if (++r0 == Pd) { r0 = 0; ++p0; }
            __syncwarp();
        };

        for (int t0 = t_begin; t0 < t_end; t0 += K) {
            {   // warp-uniform flow control (see wait_uniform)
                const int np = gw > 0 ? min(t0 + K - 1, pred_end)
                                      : (t0 + K - 1 >= Pd ? min(t0 + K - Pd + u_last, last_end) : INT_MIN);
                const int ns = has_succ_ring ? t0 + K - RS + 1 : INT_MIN;
                wait_uniform(pp + warp, np, false, cp + warp, ns, false);
            }
#pragma unroll 1
            for (int s = 0; s < K; s += U) {
                const int tg = t0 + s;
                const int blo = tg - u_max, blen = U + 32 * C - 1;
                const bool fast = !hits_row(blo, blen, 0, Pd) && !hits_row(blo, blen, N - 1, Pd);
                if (fast) {
                    const E* ib0;
                    const E* ib1;
                    if (gw == 0) {
                        ib0 = (tg < Pd && pa == 0) ? infs : bnd + fmod_pos(tg - u_min, Pd);
                        ib1 = ib0 + 1;
                    } else {
                        ib0 = my_in + ((tg - 1) & (RS - 1));
                        ib1 = my_in + (tg & (RS - 1));
                    }
                    E* ob = has_succ_ring ? succ_ring + (tg & (RS - 1)) : succ_ring + fmod_pos(tg - u_max, Pd);
                    // chain c at step h reads row r0+h-c: class (r0+h-c) mod C
                    const unsigned long long* xb[C];
#pragma unroll
                    for (int j = 0; j < C; ++j)
                        xb[j] = reinterpret_cast<const unsigned long long*>(xs) + xrow_index(r0 + j, Pd, C);
                    static_for<0, U>([&](auto hc) {
                        constexpr int h = decltype(hc)::value;
                        const float la = __shfl_up_sync(FULL, lo32(ls.right[C - 1]), 1);
                        const float lb = __shfl_up_sync(FULL, hi32(ls.right[C - 1]), 1);
                        unsigned long long lin = pk(la, lb);
                        int lsa = 0, lsb = 0;
                        if constexpr (TRACE) {
                            lsa = __shfl_up_sync(FULL, ls.rs_a[C - 1], 1);
                            lsb = __shfl_up_sync(FULL, ls.rs_b[C - 1], 1);
                        }
                        const E e = (h == 0) ? ib0[0] : ib1[h - 1];
                        if (lane == 0) {
                            lin = pk(e.a, e.b);
                            if constexpr (TRACE) { lsa = e.sa; lsb = e.sb; }
                        }
                        unsigned long long x[C];
#pragma unroll
                        for (int c = 0; c < C; ++c) {
                            const int k = h - c, j = ((k % C) + C) % C, o = (k - j) / C;
                            x[c] = xb[j][o];
                        }
                        qrow_cells<C, WC, FMA, TRACE, h>(R, Y, x, lin, lsa, lsb, ls);
                        if (lane == 31) {
                            E o;
                            o.a = lo32(ls.right[C - 1]);
                            o.b = hi32(ls.right[C - 1]);
                            if constexpr (TRACE) { o.sa = ls.rs_a[C - 1]; o.sb = ls.rs_b[C - 1]; }
                            ob[h] = o;
                        }
                    });
                    b0 += U;
                    r0 += U;
                    if (r0 >= Pd) { r0 -= Pd; ++p0; }
                } else {
                    if (hits_row(blo, blen, 0, Pd)) {
                        asm volatile("cp.async.wait_all;" ::: "memory");
                        __syncwarp();
                    }
#pragma unroll 1
                    for (int h = 0; h < U; ++h) slow_step(tg + h);
                }
                if (tg + U > pf_round * Pd + u_max + 1 && pf_round + 1 < Pl) {
                    ++pf_round;
                    __syncwarp();
                    stage_round<C, WC>(ystage, P.Y, P.Malloc, P.Pr, V, u_min, pa + pf_round, lane);
                }
            }
            __syncwarp();
            if (lane == 31) st_release<false>(succ_pp, t0 + K);
            if (lane == 0 && gw > 0) st_release<false>(pred_cp, t0 + K);
        }

        // ---- reduction per query half over chains, lanes, warps
        Partial2 pr;
        {
            float bca = best[0][0], bcb = best[0][1];
            int bja = bestcol[0][0], bjb = bestcol[0][1], bsa = beststart[0][0], bsb = beststart[0][1];
#pragma unroll
            for (int c = 1; c < C; ++c) {
                if (better(best[c][0], bestcol[c][0], bca, bja)) { bca = best[c][0]; bja = bestcol[c][0]; bsa = beststart[c][0]; }
                if (better(best[c][1], bestcol[c][1], bcb, bjb)) { bcb = best[c][1]; bjb = bestcol[c][1]; bsb = beststart[c][1]; }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const float oca = __shfl_xor_sync(FULL, bca, o), ocb = __shfl_xor_sync(FULL, bcb, o);
                const int oja = __shfl_xor_sync(FULL, bja, o), ojb = __shfl_xor_sync(FULL, bjb, o);
                const int osa = __shfl_xor_sync(FULL, bsa, o), osb = __shfl_xor_sync(FULL, bsb, o);
                if (better(oca, oja, bca, bja)) { bca = oca; bja = oja; bsa = osa; }
                if (better(ocb, ojb, bcb, bjb)) { bcb = ocb; bjb = ojb; bsb = osb; }
            }
            pr.a = Partial{bca, bja, bsa, 0};
            pr.b = Partial{bcb, bjb, bsb, 0};
        }
        if (lane == 0) red[warp] = pr;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < GW; ++w) {
                if (better(red[w].a.cost, red[w].a.col, pr.a.cost, pr.a.col)) pr.a = red[w].a;
                if (better(red[w].b.cost, red[w].b.col, pr.b.cost, pr.b.col)) pr.b = red[w].b;
            }
            const Partial halves[2] = {pr.a, pr.b};
            for (int hq = 0; hq < 2; ++hq) {
                const int q = 2 * qp + hq;
                if (q >= P.Zq) continue;           // the dummy half of an odd batch
                Partial b = halves[hq];
                if (P.persistent) {
                    reinterpret_cast<Partial*>(P.cand)[(long)q * P.S + seg] = b;
                } else if (*P.err_flag == 0) {
                    if (b.col == 0x7fffffff) { b.col = 0; b.start = 0; }
                    P.out_cost[q] = b.cost;
                    P.out_end[q] = b.col;
                    if (TRACE && P.out_start) P.out_start[q] = b.start;
                }
            }
        }
        if (P.persistent) {
            if (seg + 1 < P.S) {
                E* bo = reinterpret_cast<E*>(P.bnd_g) + (long)qp * Pd;
                for (int r = threadIdx.x; r < Pd; r += blockDim.x) bo[r] = bnd[r];
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                __threadfence();
                st_release_gpu(P.seg_done + qp, seg + 1);
            }
        }
        asm volatile("cp.async.wait_all;" ::: "memory");
        __syncthreads();
    }
}

}  // namespace sdtw
