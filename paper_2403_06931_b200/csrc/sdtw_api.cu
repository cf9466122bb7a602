// sdtw_api.cu -- host side of the C ABI declared in include/sdtw.h.
//
// Per-device context (reference buffer, workspaces, flags), option handling,
// pointer-kind detection, launch-configuration choice and kernel dispatch.
// Every step of the hot path runs in the kernels of sdtw_prep.cuh / sdtw_dp.cuh;
// there is no CPU fallback: without a CUDA device every call returns SDTW_E_CUDA.
#include "../../include/sdtw.h"
#include "sdtw_dp.cuh"
#include "sdtw_dp_pick.h"
#include "sdtw_dpq.cuh"
#include "sdtw_q8.cuh"
#include "sdtw_path.cuh"
#include "sdtw_prep.cuh"
#include "sdtw_start.cuh"

#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <algorithm>
#include <vector>
#include <queue>

namespace {

thread_local std::string g_err;

struct Options {
    int normalize = 1;
    int fma = 1;
    int segment_w = 0;
    int lanes = 0;      // warps per CTA
    int cluster = 0;
    int packed = -1;
    int chunk = 0;
    int profile = 0;
    int ring = 0;
    int sched = 0;       // 0 auto, 1 one CTA (or cluster) per query, 2 persistent segments
    int segments = 0;
    int workers = 0;     // resident CTAs per SM under persistent scheduling (0 = auto)
    int precision = 32;  // 32 fp32 cells; 16 packed half; 8 uint8 codebook (sdtw_dp2.cuh, sdtw_q8.cuh)
    int q8_prune = -1;   // uint8 codebook: INF-pruning threshold tau in code units (-1 = off)
    int q8_clip = 1000;  // uint8 codebook: clipped tail mass per side, parts per million
    int q8_codes_in = 0; // (internal) the batch already holds codes (speculative recomputation)
    int q8_int_out = 0;  // (internal) sdtw_batch_q8: leave the integer costs
    int query_rows = 0;  // 0 auto, 1 shared memory, 2 global memory (two-chain fp32 cost/end kernels)
    int pad = 0;         // extra idle rows per round period (0 = auto)
    int spec_rounds = 0; // speculative segments: rounds per correction pass (0 = auto)
    int start = 0;       // start index: 0 auto, 1 forward propagation, 2 checkpoints + walk-back
    cudaStream_t stream = 0;
};
Options g_opt;
std::mutex g_mu;
std::atomic<int64_t> g_launches{0};

struct Ctx {
    bool init = false;
    int sms = 0;
    float* ref = nullptr;
    int64_t M = 0, Malloc = 0;
    int ref_normalized = 0;
    float* ws_q = nullptr;   size_t ws_q_n = 0;     // staged host queries
    float* ws_x = nullptr;   size_t ws_x_n = 0;     // normalised queries
    unsigned char* ws_out = nullptr; size_t ws_out_n = 0;
    double* ws_part = nullptr;                      // reference partial sums + stats
    unsigned char* ws_sched = nullptr; size_t ws_sched_n = 0;   // persistent scheduling state
    unsigned char* ws_path = nullptr; size_t ws_path_n = 0;     // sdtw_path codes / row buffers / outputs
    unsigned char* ws_rag = nullptr; size_t ws_rag_n = 0;       // ragged-batch offsets + lengths
    int* order_d = nullptr; size_t order_n = 0;     // unit grab order (device) and its key
    int4* utab_d = nullptr; size_t utab_n = 0;      // speculative segments: unit-kind table
    // speculative segments: recomputed queries and their round checkpoints, one workspace per
    // recursion depth (a recomputation runs the speculative schedule again and may recompute
    // some of ITS queries: the inner level must not overwrite the outer level's rows/results)
    static constexpr int kFixDepth = 8;
    float* ws_fix[kFixDepth] = {};  size_t ws_fix_n[kFixDepth] = {};
    float* ws_fixck[kFixDepth] = {}; size_t ws_fixck_n[kFixDepth] = {};
    int fix_depth = 0;
    int last_fix_depth = 0;                         // deepest recomputation level of the last call
    float* ws_ck = nullptr; size_t ws_ck_n = 0;     // round checkpoints [Z][Pr][Pd] (checkpointed start index)
    float* ws_ckc = nullptr; size_t ws_ckc_n = 0;   // speculative correction units' checkpoints
    unsigned char* ws_win = nullptr; size_t ws_win_n = 0;   // start windows: codes, rows, query lists
    unsigned char* ws_start = nullptr; size_t ws_start_n = 0;   // start windows: starts (+ paths)
    double last_win_ms = 0.0;                       // checkpointed start index: window phase time
    int last_start_iters = 0;                       // ... and its window-widening iterations
    int64_t last_fixups = 0;                        // queries recomputed by the last call
    // grab order / unit table of the last persistent launch, reused while the plan is the
    // same (a per-call host simulation + synchronous copies left the GPU idle ~0.1-0.5 ms)
    int64_t order_key[7] = {-1, -1, -1, -1, -1, -1, -1};
    int64_t utab_key[3] = {-1, -1, -1};
    // uint8 codebook (NEXT-3, sdtw_q8.cuh): codes of the reference as fp32 0..255 (Malloc,
    // padded 0), the codebook {lo, hi} on the device and host, radix-select workspace
    float* ref_q8 = nullptr;
    unsigned char* q8_ws = nullptr;                 // 2 x 65536 counters + selections + codebook
    int q8_clip = -1;                               // clip of the current codes (-1: none built)
    float q8_lo = 0.f, q8_hi = 0.f;
    float* ws_xq = nullptr;  size_t ws_xq_n = 0;    // query codes
    float* ws_xg = nullptr;  size_t ws_xg_n = 0;    // query rows in the global pair layout (XG kernels)
    int* flag_d = nullptr;
    int* flag_h = nullptr;
    cudaEvent_t ev0 = nullptr, ev1 = nullptr;
    cudaEvent_t ev_sched = nullptr;   // after the last launch that read order_d / utab_d
    double last_dp_ms = 0.0;
    int64_t last_launches = 0;
};
constexpr int kMaxDev = 64;
Ctx g_ctx[kMaxDev];

sdtw_status fail(sdtw_status s, const std::string& msg) {
    g_err = msg;
    return s;
}
sdtw_status cuda_fail(cudaError_t e, const char* where) {
    cudaGetLastError();
    return fail(e == cudaErrorMemoryAllocation ? SDTW_E_NOMEM : SDTW_E_CUDA,
                std::string(where) + ": " + cudaGetErrorString(e));
}
#define CK(call)                                          \
    do {                                                  \
        cudaError_t _e = (call);                          \
        if (_e != cudaSuccess) return cuda_fail(_e, #call); \
    } while (0)

sdtw_status get_ctx(Ctx** out) {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDevice");
    if (dev < 0 || dev >= kMaxDev) return fail(SDTW_E_CUDA, "device index out of range");
    Ctx& c = g_ctx[dev];
    if (!c.init) {
        CK(cudaDeviceGetAttribute(&c.sms, cudaDevAttrMultiProcessorCount, dev));
        CK(cudaMalloc(&c.flag_d, 16));
        CK(cudaHostAlloc(&c.flag_h, 16, cudaHostAllocDefault));
        CK(cudaMalloc(&c.ws_part, sizeof(double) * (4 * 4096 + 8)));   // 4 doubles per partial
        CK(cudaEventCreate(&c.ev0));
        CK(cudaEventCreate(&c.ev1));
        CK(cudaEventCreateWithFlags(&c.ev_sched, cudaEventDisableTiming));
        c.init = true;
    }
    *out = &c;
    return SDTW_OK;
}

template <class T>
sdtw_status grow(T** p, size_t* have, size_t need_elems) {
    if (*have >= need_elems) return SDTW_OK;
    if (*p) cudaFree(*p);
    *p = nullptr;
    *have = 0;
    cudaError_t e = cudaMalloc(p, need_elems * sizeof(T));
    if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc(workspace)");
    *have = need_elems;
    return SDTW_OK;
}

// 1 = device pointer on the current device, 0 = host pointer, -1 = device pointer elsewhere
int ptr_kind(const void* p) {
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
        int dev = 0;
        cudaGetDevice(&dev);
        return a.device == dev ? 1 : -1;
    }
    return 0;
}

// ------------------------------------------------------------------ DP dispatch
using sdtw::DpParams;
using sdtw::DpKernel;

// dual: the dual-query kernel (two queries per lane, C chains of scalar-y strips)
// half: 0 fp32; 16 packed half; 8 / 9 uint8 codebook without / with INF pruning
DpKernel pick_kernel(int C, int WC, bool fma, bool trace, bool cl, bool dual = false, int half = 0,
                     int xs = 0) {
    if (half) {
        if (C != 2 || trace || cl || dual) return nullptr;
        return half == 16 ? sdtw::pick_dp16(WC) : sdtw::pick_dp8(WC, half == 9);
    }
    if (xs) return (C == 2 && !trace && !cl && !dual) ? (xs == 2 ? sdtw::pick_dp_c2xg(WC, fma) : sdtw::pick_dp_c2xs(WC, fma))
                                                      : nullptr;
    if (dual) {
        if (cl) return nullptr;
        return C == 1 ? sdtw::pick_dpq_c1(WC, fma, trace) : (C == 2 ? sdtw::pick_dpq_c2(WC, fma, trace) : nullptr);
    }
    return sdtw::pick_dp(C, WC, fma, trace, cl);
}

struct LaunchCfg {
    int C, WC, GW, CL, K, RS, Pd, Pr, smem;
    int persistent, S, workers;
    int dual;        // two queries per lane (chains per lane = C)
    int64_t units;   // rings per batch: queries, or query pairs when dual
    int need;        // V + (G+1)K: smallest ring-safe round period (ragged batches: per query)
    int half;        // two-chain reduced-precision kernel: 16 packed half, 8 / 9 uint8 codebook (9: INF pruning)
    int xs;          // query rows: 0 shared-memory pairs, 1 single-row layout, 2 global memory (long queries)
    int spec = 0;    // speculative segments: Sseg segments, correction passes of Rc rounds
    int Sseg = 0, Rc = 0;
    int ck = 0;      // round checkpoints (the CKPT kernel)
};

// Ragged batch descriptor (host): offsets[Z+1], the longest and shortest query.
struct Ragged {
    const std::vector<int64_t>* off = nullptr;
    int64_t nmin = 0;
};

int smem2_bytes(int half, int WC, int GW, int Pd, int RS) {
    return half == 16 ? sdtw::smem_layout2<sdtw::Half2Arith>(WC, GW, Pd, RS).bytes
                      : sdtw::smem_layout2<sdtw::Q8Arith<false>>(WC, GW, Pd, RS).bytes;
}

// Schedule choice.  OPT_PACKED: 0 scalar (C=1), 1 two packed chains (C=2), 2 four
// chains (C=4), 3 dual-query x 2 chains, 4 dual-query x 1 chain; -1 auto.
sdtw_status plan(const Ctx& ctx, int64_t Z, int64_t N, bool trace, LaunchCfg* cfg, const Ragged* rg = nullptr) {
    const Options& o = g_opt;
    // auto: two packed chains (f32x2) for cost/end; scalar strips for the start-index
    // variant, whose per-cell start selects double the registers per slot (r01 sweep at
    // N=1000: scalar W=15 3.00, packed W=14 2.89, packed W=30 1.80 TCUPS)
    const int half = o.precision == 16 ? 16 : (o.precision == 8 ? (o.q8_prune >= 0 && o.q8_prune < 255 ? 9 : 8) : 0);
    if (half && trace) return fail(SDTW_E_ARG, "the packed-half and uint8 precisions have no start index (OPT_PRECISION=32)");
    if (half && o.cluster > 1) return fail(SDTW_E_ARG, "the packed-half and uint8 precisions run without clusters");
    if (half && half != 16 && N > sdtw::kQ8MaxN) return fail(SDTW_E_ARG, "the uint8 precision takes queries of <= 12,000 samples");
    if (half == 9 && N > sdtw::kQ8PruneMaxN)
        return fail(SDTW_E_ARG, "the uint8 precision with INF pruning takes queries of <= 8,000 samples");
    const int packed = half ? 1 : (o.packed < 0 ? (trace ? 0 : 1) : o.packed);
    const bool dual = packed >= 3;
    int C = dual ? (packed == 3 ? 2 : 1) : (packed == 0 ? 1 : (packed == 1 ? 2 : 4));
    // uint8 codebook: W = 14 (r02u sweep at config 3: 6.77 vs 6.32 TCUPS unpruned, 4.39 vs 2.60
    // pruned -- the int32 chains' 30-column loop overflows the instruction footprint and spills)
    int W = o.segment_w > 0 ? o.segment_w : (C == 4 ? 28 : (C == 2 ? ((half == 8 || half == 9) ? 14 : 30) : 15));
    if (W % C != 0) return fail(SDTW_E_ARG, "segment width must be a multiple of the chains per lane");
    int WC = W / C;
    if (!pick_kernel(C, WC, true, false, false, dual, half))
        return fail(SDTW_E_ARG, "unsupported segment width " + std::to_string(W) + " for this chain layout" +
                                    (C == 4 ? " (28)" : C == 2 ? " (14, 30)" : " (7, 15)"));
    const int64_t units = dual ? (Z + 1) / 2 : Z;
    // Warps per ring.  Short fixed-length queries: 2-warp rings (round 2, speculative schedule,
    // 512 queries vs 1M, profiles/r02az_lanes.jsonl, r02ba_*: N = 500 5.40 -> 6.82 TCUPS, N =
    // 1,000 6.65 -> 7.48; the ring's fill of V steps per unit weighs less against a short round
    // period); N >= 1,500 keeps 4 (N = 1,500 7.99 vs 7.65, N = 2,000 8.18 vs 7.28).  Ragged
    // batches: 4 (the round-1 rule of 8-warp rings for short reads, measured under sequential
    // segments, lost under the speculative schedule: reads 500..8,000 7.52 -> 7.76 with 4,
    // 500..2,000 5.16 -> 7.14).
    int GW = o.lanes > 0 ? o.lanes : ((!rg && !half && C == 2 && N <= 1000) ? 2 : 4);
    int CL = o.cluster > 0 ? o.cluster : 1;
    if (GW < 1 || GW > (dual ? 12 : (C == 4 ? 4 : 8)) || CL < 1 || CL > 16 || (dual && CL != 1))
        return fail(SDTW_E_ARG, "lanes / cluster out of range for this kernel");
    // chunk = whole rotation periods (U = WC+1 steps), about the requested size
    const int U = WC + 1;
    const int G = GW * CL;
    const int64_t V = 32LL * C * G;
    // chunk: 64 steps when the query is long enough that the round period stays N
    // (Pd >= V + (G+1)K), else 32 (r01 sweep: K=64 +1.5% over 32, K=128 -12%)
    const int64_t Nk = rg ? rg->nmin : N;                // ragged: the shortest query decides
    // (with fast runs, r01: K=128 +1.5 % over 64 at 10M, +1 % at 1M; 256 -10 %)
    // Start-index runs are ALU-pipe bound and their units are short: smaller chunks
    // measured better there (r01 C5 sweep: N=500 K=32 2.86 vs K=64 2.43; N=1000 K=64 3.14 vs
    // K=128 2.80; N>=4000 K=128 ~ K=64).
    int Kauto = Nk >= V + (int64_t)(G + 1) * 128 ? 128 : (Nk >= V + (int64_t)(G + 1) * 64 ? 64 : 32);
    if (trace) Kauto = std::min(Kauto, Nk <= 600 ? 32 : (Nk <= 2000 ? 64 : 128));
    const int Kreq = o.chunk > 0 ? o.chunk : Kauto;
    const int KU = (dual ? 1 : SDTW_FAST_PERIODS) * U;   // chunk = whole fast/slow decision windows
    int K = KU * std::max(1, (Kreq + KU / 2) / KU);
    // long queries: rows and boundary ring fill the shared memory; a shorter chunk allows a
    // shallower ring (>= 4K) -- take it when that keeps more CTAs resident
    if (o.chunk <= 0 && o.ring <= 0 && !dual) {
        auto bytes_for = [&](int k) {
            const int64_t nd = V + (int64_t)(G + 1) * k;
            const int pd = (int)(N > nd ? N : nd);
            int rs = 1;
            while (rs < std::max(4 * k, 64)) rs <<= 1;
            return half ? smem2_bytes(half, WC, GW, pd, rs) : sdtw::smem_layout(C, WC, trace, GW, pd, rs).bytes;
        };
        auto ctas = [&](int bytes) { return (int)((228 * 1024) / (bytes + 1024)); };
        const int base = ctas(bytes_for(K));
        for (int k = K / 2; base < 3 && k >= 2 * KU; k /= 2)
            if (ctas(bytes_for(k)) > base) { K = k; break; }
    }
    const int64_t need = V + (int64_t)(G + 1) * K;
    const int64_t Pd = std::max<int64_t>(N + o.pad, need);
    const int64_t Pr = (ctx.M + V * WC - 1) / (V * WC);
    if (Pr * Pd + V + 2 * K >= (1LL << 31) || Pr * V * WC >= (1LL << 31))
        return fail(SDTW_E_ARG, "problem too large for 32-bit step/column counters");
    // inter-warp ring depth: deep enough to absorb one warp's round-transition
    // (slow) chunks without stalling its neighbours
    int RS = 1;
    const int RSmin = std::max(o.ring > 0 ? 4 * K : 8 * K, o.ring > 0 ? (int)o.ring : 512);
    while (RS < RSmin) RS <<= 1;
    auto layout = [&](int rs) {
        if (half) {
            sdtw::SmemLayout r;
            r.bytes = smem2_bytes(half, WC, GW, (int)Pd, rs);
            return r;
        }
        return dual ? sdtw::smem_layout_q(C, WC, trace, GW, (int)Pd, rs) : sdtw::smem_layout(C, WC, trace, GW, (int)Pd, rs);
    };
    sdtw::SmemLayout L = layout(RS);
    // long queries: the query rows and the boundary ring grow with N; shallower inter-warp
    // rings (down to 4K) when that keeps one more CTA resident per SM
    if (o.ring <= 0) {
        auto ctas = [&](int bytes) { return (int)((228 * 1024) / (bytes + 1024)); };
        for (int rs = RS / 2; rs >= std::max(4 * K, 64); rs /= 2) {
            const sdtw::SmemLayout L2 = layout(rs);
            // (2-warp rings: up to the register limit of 8 CTAs -- config 5 N = 1,000: RS 1024 -> 512
            // takes 7 -> 8 CTAs per SM, 6.88 -> 7.12 TCUPS, profiles/r02bl_*)
            const bool want = ctas(L.bytes) < 3 || (GW <= 2 && ctas(L.bytes) < 16 / GW);
            if (ctas(L2.bytes) > ctas(L.bytes) && want) { RS = rs; L = L2; }
        }
    }
    if (L.bytes > 227 * 1024) return fail(SDTW_E_ARG, "query too long for shared memory at this config");
    // long queries: the single-row layout halves the rows' bytes; take it when that keeps
    // one more CTA resident (C == 2, cost/end, no cluster)
    // Even longer: the rows in global memory (read through L1: a warp's lanes sweep a window of
    // a few hundred rows, so they stay L1-resident), the CTA keeps only the rings -- taken when
    // that allows more resident CTAs than either shared-memory layout (up to the register
    // limit of 4), or when forced by SDTW_OPT_QUERY_ROWS.
    int xs = 0;
    const bool xs_ok = !half && !dual && !trace && C == 2 && CL == 1;
    if (xs_ok && o.query_rows != 1 && pick_kernel(C, WC, true, false, false, false, 0, 1)) {
        auto ctas = [&](int bytes) { return (int)((228 * 1024) / (bytes + 1024)); };
        const sdtw::SmemLayout Lx = sdtw::smem_layout(C, WC, trace, GW, (int)Pd, RS, true);
        if (ctas(L.bytes) < 3 && ctas(Lx.bytes) > ctas(L.bytes)) { L = Lx; xs = 1; }
        const sdtw::SmemLayout Lg = sdtw::smem_layout(C, WC, trace, GW, (int)Pd, RS, false, true);
        if (o.query_rows == 2 || (ctas(L.bytes) < 4 && std::min(ctas(Lg.bytes), 4) > ctas(L.bytes))) { L = Lg; xs = 2; }
    } else if (o.query_rows == 2) {
        return fail(SDTW_E_ARG, "query rows in global memory need the two-chain fp32 cost/end kernel (no clusters)");
    }
    *cfg = LaunchCfg{C, WC, GW, CL, K, RS, (int)Pd, (int)Pr, L.bytes, 0, 1, 0, dual ? 1 : 0, units, (int)need,
                     half, xs};
    if (getenv("SDTW_DEBUG_PLAN"))                      // diagnostics only
        fprintf(stderr, "[sdtw plan] Z=%lld N=%lld C=%d WC=%d GW=%d K=%d RS=%d Pd=%lld Pr=%lld smem=%d rows=%d\n",
                (long long)Z, (long long)N, C, WC, GW, K, RS, (long long)Pd, (long long)Pr, L.bytes, xs);
    // Persistent scheduling (default when a cluster is not requested): k resident CTAs
    // per SM, k = min(occupancy, rings / SMs), pull (ring, round-segment) units, so every
    // SM carries the same load whatever the batch size mod #SMs is.
    const int sched = o.sched;
    // Speculative segments: small batches (fewer rings than SMs) cannot
    // fill the GPU with sequential segments; every segment then starts at once and a
    // correction pass of Rc rounds per segment boundary restores the exact result.
    const int64_t cols = V * WC;
    // correction length: the query's length in columns plus half a round, rounded up
    // (a slope-1 path from the boundary is dominated about N columns later).  Round-2 sweep
    // (profiles/r02aw_*): config 2 best at 2 rounds, config 5 N = 4,000 at 2 (7.51 vs 7.28
    // TCUPS with the earlier 3N rule's 4), N = 8,000 at 3 (7.27 vs 6.85 with 7); N <= 1,000: 1.
    // Any length is exact (failed corrections are recomputed); this only moves work.
    const int Rc = o.spec_rounds > 0 ? o.spec_rounds
                                     : (int)std::max<int64_t>(1, (N + cols / 2 + cols - 1) / cols);
    const bool spec_ok = !dual && CL == 1 && Pr >= 4 * (int64_t)(Rc + 1);
    if (sched == 3 && !spec_ok)
        return fail(SDTW_E_ARG, "speculative segments need no clusters, OPT_PACKED <= 2 and >= 4 "
                                "segments of more than OPT_SPEC_ROUNDS rounds");
    int occ = 0;
    if (sched == 3 || (sched == 0 && spec_ok)) {
        DpKernel k = pick_kernel(C, WC, o.fma != 0, trace, false, dual, half, xs);
        cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * GW, L.bytes) != cudaSuccess || occ < 1) {
            cudaGetLastError();
            return fail(SDTW_E_CUDA, "occupancy query failed");
        }
    }
    // auto whenever it applies (r01 sweeps, 10M x 2000, TCUPS sequential -> speculative:
    // Z=64 1.88 -> 8.15, Z=200 4.24 -> 8.54, Z=512 (config 3) 8.40 -> 8.78; 1M x 2000:
    // 8.13 -> 8.13; 100K: 7.05 -> 7.05; start index Z=512 equal): every SM runs all its
    // resident CTA slots (4 here, vs 3 rings' worth of chains) and no unit waits for a
    // long predecessor segment.
    if (sched == 3 || (sched == 0 && spec_ok)) {
        const int per_sm = o.workers > 0 ? std::min(o.workers, occ) : occ;
        const int64_t W = (int64_t)per_sm * ctx.sms;
        // segments: about five long (B) units per worker (Z=512: 5 segments 8.40, 6 8.78,
        // 8 8.74, 12 8.65; Z=64: 28 7.91, 40 8.15, 65 8.02; Z=200: 10 8.32, 16 8.54, 24 8.48),
        // each > Rc rounds and long enough that the correction passes stay a small share
        // (Rc / segment length)
        // (ragged batches, with the round-period-weighted grab order: c6 sweep 3 segments
        // 7.40, 4 7.14, 5 6.90, 8 6.67 TCUPS; sequential segments 5.63)
        int64_t Sg = o.segments > 0 ? o.segments : (10 * W + units) / (2 * units);
        Sg = std::min<int64_t>(Sg, Pr / std::max<int64_t>(4 * (Rc + 1), 8));
        Sg = std::max<int64_t>(Sg, 2);
        for (int sg = 0; sg < (int)Sg; ++sg)
            if (sdtw::spec_seg_start(sg + 1, (int)Pr, (int)Sg) - sdtw::spec_seg_start(sg, (int)Pr, (int)Sg) <= Rc)
                return fail(SDTW_E_ARG, "speculative segments shorter than the correction pass");
        cfg->spec = 1;
        cfg->Sseg = (int)Sg;
        cfg->Rc = Rc;
        cfg->persistent = 1;
        cfg->S = 3 * (int)Sg - 1;                           // unit kinds per ring (A_s, B_s, C_s)
        cfg->workers = (int)std::min<int64_t>(W, units * cfg->S);
        return SDTW_OK;
    }
    if (sched == 2 || (sched == 0 && CL == 1 && units >= ctx.sms && Pr >= 8)) {
        if (CL != 1) return fail(SDTW_E_ARG, "persistent scheduling needs cluster = 1");
        int occ = 0;
        DpKernel k = pick_kernel(C, WC, o.fma != 0, trace, false, dual, half, xs);
        cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, L.bytes);
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 32 * GW, L.bytes) != cudaSuccess || occ < 1) {
            cudaGetLastError();
            return fail(SDTW_E_CUDA, "occupancy query failed");
        }
        const int per_sm = o.workers > 0 ? std::min(o.workers, occ)
                                         : (int)std::max<int64_t>(1, std::min<int64_t>(occ, units / ctx.sms));
        // round-segments per ring: enough units to fill the last wave, long enough that the
        // per-unit fill/drain (~V steps) stays small (r01 sweep: 10M S=32 > 16 > 8; 1M S=16;
        // 100K S=6 > 8)
        int S = o.segments > 0 ? o.segments
                               : (int)std::min<int64_t>(32, std::max<int64_t>(Pr / 16, std::max<int64_t>(1, std::min<int64_t>(16, Pr / 4))));
        if (S > Pr) S = (int)Pr;
        cfg->persistent = 1;
        cfg->S = S;
        cfg->workers = (int)std::min<int64_t>((int64_t)per_sm * ctx.sms, units * S);
    }
    return SDTW_OK;
}

sdtw_status launch_dp(const LaunchCfg& c, bool fma, bool trace, const DpParams& p, cudaStream_t st) {
    DpKernel k = c.ck ? sdtw::pick_dp_c2ck(c.WC, fma, c.xs)
                      : pick_kernel(c.C, c.WC, fma, trace, c.CL > 1, c.dual != 0, c.half, c.xs);
    if (!k) return fail(SDTW_E_ARG, "no kernel for this configuration");
    CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeMaxDynamicSharedMemorySize, c.smem));
    if (c.CL > 8) CK(cudaFuncSetAttribute((const void*)k, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    cudaLaunchConfig_t lc;
    memset(&lc, 0, sizeof(lc));
    lc.gridDim = dim3((unsigned)(c.persistent ? c.workers : c.units * c.CL));
    lc.blockDim = dim3((unsigned)(32 * c.GW));
    lc.dynamicSmemBytes = (size_t)c.smem;
    lc.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)c.CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    CK(cudaLaunchKernelEx(&lc, k, p));
    g_launches++;
    return SDTW_OK;
}

// Grab order of the persistent units u = seg*R + q (R rings, S round-segments each,
// W resident workers).  Segments of one ring are sequential (segment s starts from
// segment s-1's boundary column), so a fixed seg-major order makes a worker that grabs
// (q, s) while (q, s-1) is still running wait for it -- a whole unit when R is not a
// multiple of W.  Instead simulate list scheduling with equal unit durations, one wave
// of W units at a time, longest remaining chain first: every unit is grabbed one wave
// after its predecessor, and every wave is as full as the chains allow.
std::vector<int> unit_order(int64_t R, int S, int64_t W) {
    std::vector<int> order;
    order.reserve((size_t)(R * S));
    std::vector<int> next(R, 0);
    std::vector<int64_t> idx(R);
    for (int64_t q = 0; q < R; ++q) idx[q] = q;
    int64_t left = R * S;
    while (left > 0) {
        // chains with the most segments left first (stable: lower q on ties)
        std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) { return next[a] < next[b]; });
        int64_t taken = 0;
        for (int64_t k = 0; k < R && taken < W; ++k) {
            const int64_t q = idx[k];
            if (next[q] >= S) continue;
            order.push_back((int)((int64_t)next[q] * R + q));
            ++next[q];
            ++taken;
            --left;
        }
    }
    return order;
}

// Device-side views of a finished batch (for sdtw_path): the query samples the DP
// used and the per-query results, valid until the next call.
struct BatchDev {
    const float* x = nullptr;
    const float* cost = nullptr;
    const int64_t* end = nullptr;
    const int64_t* start = nullptr;
};

// Ragged batches: units of one ring take time ~ its round period, so the wave model
// above no longer holds.  Event simulation of W workers with per-ring unit durations
// w[q]: a free worker takes the ready chain (predecessor segment finished) with the most
// remaining work, else waits for the earliest chain to become ready.
std::vector<int> unit_order_weighted(int64_t R, int S, int64_t W, const std::vector<double>& w) {
    std::vector<int> order;
    order.reserve((size_t)(R * S));
    std::vector<int> next(R, 0);
    typedef std::pair<double, int64_t> Item;
    std::priority_queue<Item> ready;                                              // (remaining work, q)
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pending;       // (ready time, q)
    std::priority_queue<double, std::vector<double>, std::greater<double>> workers;  // free times
    for (int64_t q = 0; q < R; ++q) ready.push(Item(w[q] * S, q));
    for (int64_t k = 0; k < W; ++k) workers.push(0.0);
    for (int64_t left = R * S; left > 0; --left) {
        double t = workers.top();
        workers.pop();
        while (!pending.empty() && pending.top().first <= t) {
            const int64_t q = pending.top().second;
            pending.pop();
            ready.push(Item(w[q] * (S - next[q]), q));
        }
        if (ready.empty()) {                       // idle until the earliest chain is ready
            t = pending.top().first;
            const int64_t q = pending.top().second;
            pending.pop();
            ready.push(Item(w[q] * (S - next[q]), q));
        }
        const int64_t q = ready.top().second;
        ready.pop();
        order.push_back((int)((int64_t)next[q] * R + q));
        const double fin = t + w[q];
        ++next[q];
        if (next[q] < S) pending.push(Item(fin, q));
        workers.push(fin);
    }
    return order;
}

// Reference-split requests (sdtw_batch_columns / sdtw_boundary_dp).
struct SegReq {
    int mode = 0;                  // 1: speculative batch + column copies; 2: one-unit boundary DP
    float* col_check = nullptr;    // mode 1: free-DP column at the end of the first Rc rounds [Z][N]
    float* col_last = nullptr;     // mode 1: last column of the reference [Z][N]
    int64_t* check_cols = nullptr; // mode 1: Rc * columns per round
    const float* bnd = nullptr;    // mode 2: left boundary column [Z][N] (device; nullptr = +inf)
    int free_start = 1;            // mode 2: 0 = virtual row -1 is +inf
    int64_t cols = 0;              // mode 2: reference columns to run (multiple of the round width; 0 = all)
    float* col_out = nullptr;      // mode 2: end column [Z][N] (device) or nullptr
    float* ck = nullptr;           // mode 3: round checkpoints [Z][Pr][Pd] (device), exact after the call
    int ck_Pr = 0, ck_Pd = 0;      // mode 3: the layout the caller allocated (must match the plan)
};

// The uint8 codebook of the current reference: two exact order statistics
// by radix select, then the reference codes.  Rebuilt when the reference or the clip
// option changed.  Untimed setup (once per reference).
constexpr size_t kQ8Hist = 2 * 65536 * sizeof(unsigned);
sdtw_status ensure_q8(Ctx* ctx, cudaStream_t st) {
    const int clip = g_opt.q8_clip;
    if (ctx->ref_q8 && ctx->q8_clip == clip) return SDTW_OK;
    if (!ctx->q8_ws) CK(cudaMalloc(&ctx->q8_ws, kQ8Hist + 256));
    if (!ctx->ref_q8) CK(cudaMalloc(&ctx->ref_q8, ctx->Malloc * sizeof(float)));
    unsigned* hist = reinterpret_cast<unsigned*>(ctx->q8_ws);
    sdtw::Q8Sel* sel = reinterpret_cast<sdtw::Q8Sel*>(ctx->q8_ws + kQ8Hist);
    float* cb = reinterpret_cast<float*>(ctx->q8_ws + kQ8Hist + 2 * sizeof(sdtw::Q8Sel));
    const int64_t M = ctx->M;
    const unsigned k_lo = (unsigned)(((int64_t)clip * (M - 1)) / 1000000);
    const unsigned k_hi = (unsigned)(M - 1 - k_lo);
    const int grid = 4 * ctx->sms;
    for (int pass = 0; pass < 2; ++pass) {
        CK(cudaMemsetAsync(hist, 0, kQ8Hist, st));
        sdtw::q8_hist_kernel<<<grid, 256, 0, st>>>(ctx->ref, M, hist, sel, pass);
        sdtw::q8_select_kernel<<<1, 1024, 0, st>>>(hist, sel, pass, k_lo, k_hi);
        g_launches += 2;
    }
    sdtw::q8_codebook_kernel<<<1, 32, 0, st>>>(sel, cb);
    sdtw::q8_quantize_kernel<<<grid, 256, 0, st>>>(ctx->ref, M, ctx->Malloc, cb, ctx->ref_q8);
    g_launches += 2;
    CK(cudaGetLastError());
    float h[2];
    CK(cudaMemcpyAsync(h, cb, sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ctx->q8_lo = h[0];
    ctx->q8_hi = h[1];
    ctx->q8_clip = clip;
    return SDTW_OK;
}
const float* q8_codebook_dev(const Ctx* ctx) {
    return reinterpret_cast<const float*>(ctx->q8_ws + kQ8Hist + 2 * sizeof(sdtw::Q8Sel));
}

sdtw_status run_batch(const float* Q, int64_t Z, int64_t N, float* out_cost, int64_t* out_end,
                      int64_t* out_start, bool trace, BatchDev* dev_out = nullptr, Ragged rg = Ragged(),
                      const SegReq* sr = nullptr);

// Speculative segments: queries whose correction pass was not overtaken within Rc rounds
// (fix[q] != 0) are recomputed with sequential segments from their normalised rows and
// their results replace the speculative ones.
#ifndef SDTW_FIXUP_SEQ
#define SDTW_FIXUP_SEQ 0    // A/B only: 1 recomputes failed queries with one CTA each (the r01 fixup)
#endif
sdtw_status spec_fixup(Ctx* ctx, const float* xd, int64_t Z, int64_t N, const std::vector<int64_t>* off,
                       const int* fix_d, float* dc, int64_t* de, int64_t* ds, cudaStream_t st, int Rc,
                       float* col_last = nullptr, const SegReq* ckr = nullptr) {
    std::vector<int> fix((size_t)Z);
    CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(fix.data(), fix_d, (size_t)Z * sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*ctx->flag_h) return SDTW_OK;                  // non-finite input: no results (reported by the caller)
    std::vector<int64_t> idx;
    for (int64_t q = 0; q < Z; ++q)
        if (fix[q]) idx.push_back(q);
    if (idx.empty()) return SDTW_OK;
    const int64_t F = (int64_t)idx.size();
    // the recomputed queries' rows, packed (ragged batches: with their own offsets)
    std::vector<int64_t> off2((size_t)F + 1, 0);
    int64_t nmin2 = INT64_MAX, nmax2 = 0;
    for (int64_t k = 0; k < F; ++k) {
        const int64_t n = off ? (*off)[idx[k] + 1] - (*off)[idx[k]] : N;
        off2[k + 1] = off2[k] + n;
        nmin2 = std::min(nmin2, n);
        nmax2 = std::max(nmax2, n);
    }
    const size_t need = 5 * (size_t)F + (size_t)off2[F] * (col_last ? 2 : 1);   // (end, start, cost) + rows (+ columns)
    const int depth = ctx->fix_depth;
    if (depth >= Ctx::kFixDepth) return fail(SDTW_E_CUDA, "internal: speculative recomputation nested too deep");
    sdtw_status s = grow(&ctx->ws_fix[depth], &ctx->ws_fix_n[depth], need);
    if (s != SDTW_OK) return s;
    int64_t* fe = reinterpret_cast<int64_t*>(ctx->ws_fix[depth]);
    int64_t* fs = fe + F;
    float* fc = ctx->ws_fix[depth] + 4 * F;
    float* rows = fc + F;
    for (int64_t k = 0; k < F; ++k) {
        const int64_t src = off ? (*off)[idx[k]] : idx[k] * N;
        CK(cudaMemcpyAsync(rows + off2[k], xd + src, (size_t)(off2[k + 1] - off2[k]) * sizeof(float),
                           cudaMemcpyDeviceToDevice, st));
    }
    Ragged rg2;
    if (off) {
        rg2.off = &off2;
        rg2.nmin = nmin2;
    }
    const Options saved = g_opt;
    g_opt.normalize = 0;
    g_opt.profile = 0;
    g_opt.q8_codes_in = 1;                            // uint8 codebook: rows are codes already
    g_opt.sched = 1;                                  // one CTA per ring (the column-returning paths)
    g_opt.stream = st;
    const int64_t fixed_before = F;
    ++ctx->fix_depth;                                 // nested recomputations use the next workspace
    ctx->last_fix_depth = std::max(ctx->last_fix_depth, ctx->fix_depth);
    float* fcol = rows + off2[F];
    float* fck = nullptr;
    if (ckr) {                                        // round checkpoints of the recomputed queries
        const size_t per = (size_t)ckr->ck_Pr * ckr->ck_Pd;
        s = grow(&ctx->ws_fixck[depth], &ctx->ws_fixck_n[depth], (size_t)F * per);
        if (s == SDTW_OK) {
            fck = ctx->ws_fixck[depth];
            SegReq r3 = *ckr;
            r3.ck = fck;
#if !SDTW_FIXUP_SEQ
            // as below: the recomputed queries as their own speculative batch, corrections x4
            // (the checkpoint layout depends only on N and the ring, not on the schedule)
            g_opt.sched = 0;
            g_opt.spec_rounds = 4 * std::max(Rc, 1);
            g_opt.segments = 0;
            g_opt.workers = 0;
#endif
            s = run_batch(rows, F, N, fc, fe, nullptr, false, nullptr, Ragged(), &r3);
        }
        for (int64_t k = 0; s == SDTW_OK && k < F; ++k) {   // (no early return: options restored below)
            const cudaError_t e = cudaMemcpyAsync(ckr->ck + idx[k] * per, fck + k * per, per * sizeof(float),
                                                  cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) s = cuda_fail(e, "cudaMemcpyAsync(recomputed checkpoints)");
        }
    } else if (col_last) {                            // also the true last column: one-unit DP per query
        g_opt.sched = 3;
        SegReq r2;
        r2.mode = 2;
        r2.col_out = fcol;
        s = run_batch(rows, F, N, fc, fe, nullptr, false, nullptr, Ragged(), &r2);
    } else {
        // The recomputed queries run through the speculative schedule again, with corrections
        // four times as long (a match that straddled a segment boundary for more than Rc
        // rounds); all SMs share the few queries instead of one CTA each (one CTA per query:
        // ~1.4 s per 10M-sample query, a cliff on top of a 1.2 s batch).  Queries that fail
        // again recurse with 16 Rc, ...; once the corrections no longer fit (Pr < 4(Rc+1))
        // the plan falls back to sequential segments, so the recursion ends.
#if !SDTW_FIXUP_SEQ
        g_opt.sched = 0;
        g_opt.spec_rounds = 4 * std::max(Rc, 1);
        g_opt.segments = 0;
        g_opt.workers = 0;
#endif
        s = run_batch(rows, F, off ? nmax2 : N, fc, fe, ds ? fs : nullptr, ds != nullptr, nullptr, rg2);
    }
    g_opt = saved;
    --ctx->fix_depth;
    if (s != SDTW_OK) return s;
    if (col_last)
        for (int64_t k = 0; k < F; ++k)
            CK(cudaMemcpyAsync(col_last + idx[k] * N, fcol + k * N, (size_t)N * 4, cudaMemcpyDeviceToDevice, st));
    for (int64_t k = 0; k < F; ++k) {
        CK(cudaMemcpyAsync(dc + idx[k], fc + k, sizeof(float), cudaMemcpyDeviceToDevice, st));
        CK(cudaMemcpyAsync(de + idx[k], fe + k, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
        if (ds) CK(cudaMemcpyAsync(ds + idx[k], fs + k, sizeof(int64_t), cudaMemcpyDeviceToDevice, st));
    }
    ctx->last_fixups = fixed_before;
    return SDTW_OK;
}

// Speculative segments: the unit-kind table {pa, pb, in_k, db} of one
// ring -- A_s (k = s): rounds [a_s, +Rc) from a +inf boundary (a_s = spec_seg_start); B_s (k = Sg + s): the
// rest of segment s after A_s; C_s (k = 2Sg + s - 1, s >= 1): A_s's rounds again from
// B_{s-1}'s end column with no free start.
std::vector<int4> spec_table(int Pr, int Sg, int Rc) {
    std::vector<int4> t(3 * Sg - 1);
    for (int s = 0; s < Sg; ++s) {
        const int a = sdtw::spec_seg_start(s, Pr, Sg), e = sdtw::spec_seg_start(s + 1, Pr, Sg);
        t[s] = make_int4(a, a + Rc, -1, 0);
        t[Sg + s] = make_int4(a + Rc, e, s, 0);
        if (s > 0) t[2 * Sg + s - 1] = make_int4(a, a + Rc, Sg + s - 1, 1);
    }
    return t;
}

// Grab order of the speculative units u = k*R + q: list scheduling of W workers over
// units with durations pb - pa and one predecessor each (in_k), highest remaining
// chain (own + successors' rounds) first among the ready units.
std::vector<int> spec_order(int64_t R, const std::vector<int4>& t, int64_t W, const std::vector<double>* wq = nullptr) {
    // wq: per-ring weight (ragged batches: round period of the query), 1 otherwise
    auto wt = [&](int64_t q) { return wq ? (*wq)[q] : 1.0; };
    const int S = (int)t.size(), Sg = (S + 1) / 3;
    std::vector<double> dur(S), prio(S);
    for (int k = 0; k < S; ++k) dur[k] = t[k].y - t[k].x;
    for (int s = 0; s < Sg; ++s) {
        const double c = (s + 1 < Sg) ? dur[2 * Sg + s] : 0.0;     // C_{s+1} follows B_s
        prio[Sg + s] = dur[Sg + s] + c;
        prio[s] = dur[s] + prio[Sg + s];
        if (s > 0) prio[2 * Sg + s - 1] = dur[2 * Sg + s - 1];
    }
    typedef std::pair<double, int64_t> Item;                      // (priority or time, unit)
    std::priority_queue<Item> ready;
    std::priority_queue<Item, std::vector<Item>, std::greater<Item>> pending;
    std::priority_queue<double, std::vector<double>, std::greater<double>> workers;
    std::vector<std::vector<int>> succ(S);
    for (int k = 0; k < S; ++k)
        if (t[k].z >= 0) succ[t[k].z].push_back(k);
    for (int64_t q = 0; q < R; ++q)
        for (int k = 0; k < S; ++k)
            if (t[k].z < 0) ready.push(Item(prio[k] * wt(q) - 1e-9 * (double)q, (int64_t)k * R + q));
    for (int64_t w = 0; w < W; ++w) workers.push(0.0);
    std::vector<int> order;
    order.reserve((size_t)(R * S));
    while ((int64_t)order.size() < R * S) {
        double now = workers.top();
        workers.pop();
        auto release = [&](double upto) {
            while (!pending.empty() && pending.top().first <= upto) {
                const int64_t u = pending.top().second;
                pending.pop();
                ready.push(Item(prio[u / R] * wt(u % R) - 1e-9 * (double)(u % R), u));
            }
        };
        release(now);
        if (ready.empty()) {
            now = pending.top().first;
            release(now);
        }
        const int64_t u = ready.top().second;
        ready.pop();
        order.push_back((int)u);
        const double fin = now + dur[u / R] * wt(u % R);
        for (int k2 : succ[u / R]) pending.push(Item(fin, (int64_t)k2 * R + u % R));
        workers.push(fin);
    }
    return order;
}

sdtw_status run_batch(const float* Q, int64_t Z, int64_t N, float* out_cost, int64_t* out_end,
                      int64_t* out_start, bool trace, BatchDev* dev_out, Ragged rg, const SegReq* sr) {
    if (N < 1 || Z < 0) return fail(SDTW_E_ARG, "N must be >= 1 and n_queries >= 0");
    if (Z > 0 && (!Q || !out_cost || !out_end || (trace && !out_start)))
        return fail(SDTW_E_ARG, "NULL pointer");
    if (Z > 0x7fffffff || N > 0x7fffffff) return fail(SDTW_E_ARG, "sizes exceed int32");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (!ctx->ref) return fail(SDTW_E_NOREF, "no reference set on this device");
    ctx->last_launches = 0;
    ctx->last_dp_ms = 0.0;
    if (Z == 0) return SDTW_OK;
    const Options o = g_opt;
    cudaStream_t st = o.stream;
    const int64_t launches0 = g_launches.load();

    LaunchCfg cfg;
    s = plan(*ctx, Z, N, trace, &cfg, rg.off ? &rg : nullptr);
    if (s != SDTW_OK) return s;
    if (rg.off && cfg.dual) return fail(SDTW_E_ARG, "ragged batches need OPT_PACKED in {0, 1, 2}");
    const int smode = sr ? sr->mode : 0;
    if (smode == 3) {                                   // round checkpoints
        if (trace || rg.off || cfg.half || cfg.dual || cfg.CL != 1 || cfg.C != 2 || !sdtw::pick_dp_c2ck(cfg.WC, true, false))
            return fail(SDTW_E_ARG, "round checkpoints need the two-chain fp32 cost/end kernel (no clusters, "
                                    "fixed-length queries)");
        if (cfg.Pr != sr->ck_Pr || cfg.Pd != sr->ck_Pd)
            return fail(SDTW_E_CUDA, "internal: checkpoint layout does not match the launch plan");
        cfg.ck = 1;
    } else if (smode) {
        if (!cfg.spec || trace || rg.off || cfg.half)
            return fail(SDTW_E_ARG, "reference-split calls need fp32 cost/end, fixed-length queries and the "
                                    "speculative schedule (no clusters, OPT_SCHED 0 or 3, >= 4(Rc+1) rounds)");
        const int64_t cpr = 32LL * cfg.C * cfg.GW * cfg.WC;
        if (smode == 1 && sr->col_last && ctx->M % cpr != 0)
            return fail(SDTW_E_ARG, "the last column needs a reference length that is a multiple of the round width");
        if (smode == 2) {
            const int64_t cols = sr->cols > 0 ? sr->cols : cfg.Pr * cpr;
            if (cols % cpr != 0 || cols > cfg.Pr * cpr)
                return fail(SDTW_E_ARG, "n_cols must be a multiple of the round width and <= the reference");
            cfg.Sseg = 0;
            cfg.Rc = (int)(cols / cpr);                     // rounds of the single unit
            cfg.S = 1;
            cfg.workers = (int)std::min<int64_t>(cfg.workers, cfg.units);
        }
    }

    const int kq = ptr_kind(Q), kc = ptr_kind(out_cost), ke = ptr_kind(out_end);
    const int ks = trace ? ptr_kind(out_start) : 1;
    if (kq < 0 || kc < 0 || ke < 0 || ks < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    const size_t nel = rg.off ? (size_t)(*rg.off)[Z] : (size_t)Z * (size_t)N;
    // ragged: offsets and lengths on the device (one small H2D)
    const int64_t* qoff_d = nullptr;
    const int* qlen_d = nullptr;
    if (rg.off) {
        const size_t bytes = (size_t)(Z + 1) * 8 + (size_t)Z * 4;
        if (bytes > ctx->ws_rag_n) {
            if (ctx->ws_rag) cudaFree(ctx->ws_rag);
            ctx->ws_rag = nullptr;
            ctx->ws_rag_n = 0;
            CK(cudaMalloc(&ctx->ws_rag, bytes));
            ctx->ws_rag_n = bytes;
        }
        std::vector<unsigned char> hb(bytes);
        memcpy(hb.data(), rg.off->data(), (size_t)(Z + 1) * 8);
        int* hl = reinterpret_cast<int*>(hb.data() + (size_t)(Z + 1) * 8);
        for (int64_t q = 0; q < Z; ++q) hl[q] = (int)((*rg.off)[q + 1] - (*rg.off)[q]);
        CK(cudaMemcpy(ctx->ws_rag, hb.data(), bytes, cudaMemcpyHostToDevice));
        qoff_d = reinterpret_cast<const int64_t*>(ctx->ws_rag);
        qlen_d = reinterpret_cast<const int*>(ctx->ws_rag + (size_t)(Z + 1) * 8);
    }

    const float* qd = Q;
    if (kq == 0) {
        s = grow(&ctx->ws_q, &ctx->ws_q_n, nel);
        if (s != SDTW_OK) return s;
        CK(cudaMemcpyAsync(ctx->ws_q, Q, nel * sizeof(float), cudaMemcpyHostToDevice, st));
        qd = ctx->ws_q;
    }
    CK(cudaMemsetAsync(ctx->flag_d, 0, sizeof(int), st));
    const float* xd = qd;
    const bool pad = cfg.dual && (Z & 1);       // odd batch: a zero dummy query completes the last pair
    if (o.normalize || pad) {
        s = grow(&ctx->ws_x, &ctx->ws_x_n, nel + (pad ? (size_t)N : 0));
        if (s != SDTW_OK) return s;
        if (pad) CK(cudaMemsetAsync(ctx->ws_x + nel, 0, (size_t)N * sizeof(float), st));
        sdtw::znorm_rows_kernel<<<(unsigned)Z, 256, 0, st>>>(qd, ctx->ws_x, N, o.normalize, ctx->flag_d, qoff_d);
        xd = ctx->ws_x;
    } else {
        sdtw::znorm_rows_kernel<<<(unsigned)Z, 256, 0, st>>>(qd, const_cast<float*>(qd), N, 0, ctx->flag_d, qoff_d);
    }
    CK(cudaGetLastError());
    g_launches++;
    if (cfg.half == 8 || cfg.half == 9) {                // uint8 codebook: query codes
        s = ensure_q8(ctx, st);
        if (s != SDTW_OK) return s;
        if (!o.q8_codes_in) {
            s = grow(&ctx->ws_xq, &ctx->ws_xq_n, nel);
            if (s != SDTW_OK) return s;
            sdtw::q8_quantize_kernel<<<4 * ctx->sms, 256, 0, st>>>(xd, (int64_t)nel, (int64_t)nel, q8_codebook_dev(ctx),
                                                                  ctx->ws_xq);
            CK(cudaGetLastError());
            g_launches++;
            xd = ctx->ws_xq;
        }
    }

    // outputs: direct when device pointers, else staged
    const bool host_out = (kc == 0 || ke == 0 || ks == 0);
    float* dc = out_cost;
    int64_t* de = out_end;
    int64_t* ds = out_start;
    if (host_out) {
        s = grow(&ctx->ws_out, &ctx->ws_out_n, (size_t)Z * 24 + 64);
        if (s != SDTW_OK) return s;
        de = reinterpret_cast<int64_t*>(ctx->ws_out);
        ds = de + Z;
        dc = reinterpret_cast<float*>(ds + Z);
    }
    DpParams p;
    p.X = xd;
    p.Y = (cfg.half == 8 || cfg.half == 9) ? ctx->ref_q8 : ctx->ref;
    p.q8_tau2 = cfg.half == 9 ? o.q8_prune * o.q8_prune : 0;
    p.xg = nullptr;
    if (cfg.xs == 2) {                                  // long queries: rows in global memory
        s = grow(&ctx->ws_xg, &ctx->ws_xg_n, (size_t)Z * cfg.Pd * 2);
        if (s != SDTW_OK) return s;
        sdtw::xg_layout_kernel<<<(unsigned)Z, 256, 0, st>>>(xd, (int)N, cfg.Pd, cfg.need, qoff_d, qlen_d, ctx->ws_xg);
        CK(cudaGetLastError());
        g_launches++;
        p.xg = ctx->ws_xg;
    }
    p.Malloc = (int)ctx->Malloc;
    p.Z = (int)cfg.units;
    p.Zq = (int)Z;
    p.N = (int)N;
    p.M = (int)ctx->M;
    p.Pd = cfg.Pd;
    p.Pr = cfg.Pr;
    p.K = cfg.K;
    p.RS = cfg.RS;
    p.out_cost = dc;
    p.out_end = de;
    p.out_start = trace ? ds : nullptr;
    p.err_flag = ctx->flag_d;
    p.persistent = cfg.persistent;
    p.S = cfg.S;
    p.counter = nullptr;
    p.order = nullptr;
    p.qoff = qoff_d;
    p.qlen = qlen_d;
    p.need = cfg.need;
    p.seg_done = nullptr;
    p.bnd_g = nullptr;
    p.cand = nullptr;
    p.utab = nullptr;
    p.bnd_user = nullptr;
    p.col_out = nullptr;
    p.negzero = -0.0f;
    // plain cost/end calls consume no end column of the last round (tail skip)
    p.unit_log = nullptr;
    p.tail_skip = (smode == 0 && !cfg.ck && getenv("SDTW_NO_TAIL_SKIP") == nullptr) ? 1 : 0;
    p.ckpt = nullptr;
    p.ckpt_c = nullptr;
    p.ck_sg = 0;
    p.ck_rc = 0;
    if (cfg.ck) {
        p.ckpt = sr->ck;
        if (cfg.spec && cfg.Sseg > 1) {
            s = grow(&ctx->ws_ckc, &ctx->ws_ckc_n, (size_t)Z * (cfg.Sseg - 1) * cfg.Rc * cfg.Pd);
            if (s != SDTW_OK) return s;
            p.ckpt_c = ctx->ws_ckc;
        }
        p.ck_sg = cfg.Sseg;
        p.ck_rc = cfg.Rc;
    }
    int* fix_d = nullptr;
    ctx->last_fixups = 0;
    if (ctx->fix_depth == 0) ctx->last_fix_depth = 0;
    if (cfg.persistent) {
        const size_t ent = cfg.half == 16 ? 2 : (trace ? 8 : 4) * (cfg.dual ? 2 : 1);
        const size_t R = (size_t)cfg.units;
        // done flags: per ring (sequential segments: a counter) or per unit (speculative)
        const size_t done_b = ((sizeof(int) * R * (cfg.spec ? cfg.S : 1) + 255) / 256) * 256;
        const size_t fix_b = cfg.spec ? ((sizeof(int) * R + 255) / 256) * 256 : 0;
        const size_t bnd_units = cfg.spec ? R * cfg.S : R;
        const size_t nb = 256 + done_b + fix_b + 16 * (size_t)Z * cfg.S + ent * bnd_units * cfg.Pd;
        s = grow(&ctx->ws_sched, &ctx->ws_sched_n, nb);
        if (s != SDTW_OK) return s;
        unsigned char* b = ctx->ws_sched;
        p.counter = reinterpret_cast<int*>(b);
        p.seg_done = reinterpret_cast<int*>(b + 256);
        if (cfg.spec) fix_d = reinterpret_cast<int*>(b + 256 + done_b);
        p.cand = b + 256 + done_b + fix_b;
        p.bnd_g = static_cast<unsigned char*>(p.cand) + 16 * (size_t)Z * cfg.S;
        CK(cudaMemsetAsync(b, 0, 256 + done_b, st));
        const bool utab_hit = cfg.spec && smode != 2 && ctx->utab_key[0] == cfg.Pr &&
                              ctx->utab_key[1] == cfg.Sseg && ctx->utab_key[2] == cfg.Rc;
        if (cfg.spec && utab_hit) {
            p.utab = ctx->utab_d;
        } else if (cfg.spec) {
            const std::vector<int4> tab = smode == 2
                ? std::vector<int4>{make_int4(0, cfg.Rc, sr->bnd ? -2 : -1, sr->free_start ? 0 : 1)}
                : spec_table(cfg.Pr, cfg.Sseg, cfg.Rc);
            ctx->utab_key[0] = -1;
            if (tab.size() > ctx->utab_n) {
                if (ctx->utab_d) cudaFree(ctx->utab_d);
                ctx->utab_d = nullptr;
                ctx->utab_n = 0;
                CK(cudaMalloc(&ctx->utab_d, tab.size() * sizeof(int4)));
                ctx->utab_n = tab.size();
            }
            // the previous launch that read the table may still run (on this or another stream)
            CK(cudaStreamWaitEvent(st, ctx->ev_sched, 0));
            CK(cudaMemcpyAsync(ctx->utab_d, tab.data(), tab.size() * sizeof(int4), cudaMemcpyHostToDevice, st));
            p.utab = ctx->utab_d;
            if (smode != 2) {
                ctx->utab_key[0] = cfg.Pr;
                ctx->utab_key[1] = cfg.Sseg;
                ctx->utab_key[2] = cfg.Rc;
            }
        }
        const int64_t okey[7] = {(int64_t)R, cfg.S, cfg.workers, cfg.spec, cfg.spec ? cfg.Pr : 0,
                                 cfg.spec ? cfg.Sseg : 0, cfg.spec ? cfg.Rc : 0};
        bool order_hit = !rg.off && smode != 2;
        for (int k = 0; k < 7; ++k) order_hit = order_hit && ctx->order_key[k] == okey[k];
        if (!order_hit) {
            std::vector<int> ord;
            if (smode == 2) {
                ord.resize(R);
                for (size_t k = 0; k < R; ++k) ord[k] = (int)k;
            } else if (cfg.spec) {
                std::vector<double> w;
                if (rg.off) {
                    w.resize(R);
                    for (int64_t q = 0; q < (int64_t)R; ++q)
                        w[q] = (double)std::max<int64_t>((*rg.off)[q + 1] - (*rg.off)[q], cfg.need);
                }
                ord = spec_order((int64_t)R, spec_table(cfg.Pr, cfg.Sseg, cfg.Rc), cfg.workers, rg.off ? &w : nullptr);
            } else if (rg.off) {
                std::vector<double> w(R);
                for (int64_t q = 0; q < (int64_t)R; ++q)
                    w[q] = (double)std::max<int64_t>((*rg.off)[q + 1] - (*rg.off)[q], cfg.need);
                ord = unit_order_weighted((int64_t)R, cfg.S, cfg.workers, w);
            } else {
                ord = unit_order((int64_t)R, cfg.S, cfg.workers);
            }
            if (ord.size() > ctx->order_n) {
                if (ctx->order_d) cudaFree(ctx->order_d);
                ctx->order_d = nullptr;
                ctx->order_n = 0;
                CK(cudaMalloc(&ctx->order_d, ord.size() * sizeof(int)));
                ctx->order_n = ord.size();
            }
            CK(cudaStreamWaitEvent(st, ctx->ev_sched, 0));
            CK(cudaMemcpyAsync(ctx->order_d, ord.data(), ord.size() * sizeof(int), cudaMemcpyHostToDevice, st));
            for (int k = 0; k < 7; ++k) ctx->order_key[k] = okey[k];
            if (rg.off || smode == 2) ctx->order_key[0] = -1;       // ragged / boundary DP: not cached
        }
        p.order = ctx->order_d;
    }
    p.bnd_user = smode == 2 ? sr->bnd : nullptr;
    p.col_out = smode == 2 ? sr->col_out : nullptr;
    // diagnostics: SDTW_UNIT_LOG=<file> appends one line per grabbed unit of this launch
    // (unit, SM, block, grab / start / end ns) -- scripts/unit_timeline.py reads it
    const char* ulog_path = cfg.persistent ? getenv("SDTW_UNIT_LOG") : nullptr;
    long long* ulog_d = nullptr;
    const size_t ulog_n = ulog_path ? (size_t)cfg.units * cfg.S : 0;
    if (ulog_path) {
        CK(cudaMalloc(&ulog_d, ulog_n * 4 * sizeof(long long)));
        CK(cudaMemsetAsync(ulog_d, 0, ulog_n * 4 * sizeof(long long), st));
        p.unit_log = ulog_d;
    }
    if (o.profile) CK(cudaEventRecord(ctx->ev0, st));
    s = launch_dp(cfg, o.fma != 0, trace, p, st);
    if (s != SDTW_OK) return s;
    if (cfg.persistent) CK(cudaEventRecord(ctx->ev_sched, st));
    if (ulog_path) {
        std::vector<long long> h(ulog_n * 4);
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(h.data(), ulog_d, h.size() * sizeof(long long), cudaMemcpyDeviceToHost));
        cudaFree(ulog_d);
        if (FILE* f = fopen(ulog_path, "a")) {
            fprintf(f, "# launch Z=%lld S=%d Sseg=%d Rc=%d Pr=%d workers=%d\n", (long long)cfg.units, cfg.S, cfg.Sseg,
                    cfg.Rc, cfg.Pr, cfg.workers);
            for (size_t i = 0; i < ulog_n; ++i)
                fprintf(f, "%zu %lld %lld %lld %lld %lld %lld\n", i, h[4 * i] & 0xfffff, (h[4 * i] >> 20) & 0xfffff,
                        h[4 * i] >> 40, h[4 * i + 1], h[4 * i + 2], h[4 * i + 3]);
            fclose(f);
        }
    }
    if (smode == 2) {
        sdtw::finalize_kernel<<<(unsigned)((Z + 127) / 128), 128, 0, st>>>(
            static_cast<const sdtw::Partial*>(p.cand), (int)Z, 1, ctx->flag_d, dc, de, nullptr);
        CK(cudaGetLastError());
        g_launches++;
    } else if (cfg.spec) {
        sdtw::finalize_spec_kernel<<<(unsigned)Z, 128, 0, st>>>(
            static_cast<const sdtw::Partial*>(p.cand), p.bnd_g, (int)Z, cfg.S, cfg.Sseg,
            cfg.Pd, (int)N, qlen_d, ctx->flag_d, dc, de, trace ? ds : nullptr, fix_d, cfg.half == 16);
        CK(cudaGetLastError());
        g_launches++;
        if (smode == 1) {                                   // free-DP columns of kinds A_0 and B_{Sg-1}
            // (copied only when no sample was non-finite: no partial results on error)
            CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
            CK(cudaStreamSynchronize(st));
            const size_t pitch = (size_t)cfg.S * cfg.Pd * sizeof(float);
            const float* bg = static_cast<const float*>(p.bnd_g);
            if (sr->col_check && !*ctx->flag_h)
                CK(cudaMemcpy2DAsync(sr->col_check, (size_t)N * 4, bg, pitch, (size_t)N * 4, (size_t)Z,
                                     cudaMemcpyDeviceToDevice, st));
            if (sr->col_last && !*ctx->flag_h)
                CK(cudaMemcpy2DAsync(sr->col_last, (size_t)N * 4, bg + (size_t)(2 * cfg.Sseg - 1) * cfg.Pd, pitch,
                                     (size_t)N * 4, (size_t)Z, cudaMemcpyDeviceToDevice, st));
            if (sr->check_cols) *sr->check_cols = (int64_t)cfg.Rc * 32LL * cfg.C * cfg.GW * cfg.WC;
        }
        if (cfg.ck && cfg.Sseg > 1) {                       // exact columns inside the correction rounds
            sdtw::merge_ckpt_kernel<<<dim3((unsigned)(cfg.Sseg - 1), (unsigned)Z), 256, 0, st>>>(
                p.ckpt, p.ckpt_c, fix_d, cfg.Pr, cfg.Pd, (int)N, cfg.Sseg, cfg.Rc);
            CK(cudaGetLastError());
            g_launches++;
        }
        s = spec_fixup(ctx, xd, Z, N, rg.off, fix_d, dc, de, trace ? ds : nullptr, st, cfg.Rc,
                       smode == 1 ? sr->col_last : nullptr, cfg.ck ? sr : nullptr);
        if (s != SDTW_OK) return s;
    } else if (cfg.persistent) {
        sdtw::finalize_kernel<<<(unsigned)((Z + 127) / 128), 128, 0, st>>>(
            static_cast<const sdtw::Partial*>(p.cand), (int)Z, cfg.S, ctx->flag_d, dc, de, trace ? ds : nullptr);
        CK(cudaGetLastError());
        g_launches++;
    }
    if (o.profile) CK(cudaEventRecord(ctx->ev1, st));
    if (cfg.half == 9 && !o.q8_codes_in) {              // pruning: (>= 2^29) -> (INF, end 0)
        sdtw::q8_canon_kernel<<<(unsigned)((Z + 255) / 256), 256, 0, st>>>(dc, de, Z, ctx->flag_d);
        CK(cudaGetLastError());
        g_launches++;
    }
    if ((cfg.half == 8 || cfg.half == 9) && !o.q8_int_out && !o.q8_codes_in) {   // sdtw_batch: normalised units
        sdtw::q8_scale_kernel<<<(unsigned)((Z + 255) / 256), 256, 0, st>>>(dc, Z, q8_codebook_dev(ctx), ctx->flag_d);
        CK(cudaGetLastError());
        g_launches++;
    }
    CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (o.profile) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_dp_ms = ms;
    }
    ctx->last_launches = g_launches.load() - launches0;
    if (*ctx->flag_h) return fail(SDTW_E_NONFINITE, "query batch contains a non-finite sample");
    if (dev_out) {
        dev_out->x = xd;
        dev_out->cost = dc;
        dev_out->end = de;
        dev_out->start = ds;
    }
    if (host_out) {
        // copy each output to wherever it lives
        auto cp = [&](void* dst, const void* src, size_t bytes, int kind) -> cudaError_t {
            return cudaMemcpyAsync(dst, src, bytes, kind ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st);
        };
        if (dc != out_cost) CK(cp(out_cost, dc, Z * sizeof(float), kc));
        if (de != out_end) CK(cp(out_end, de, Z * sizeof(int64_t), ke));
        if (trace && ds != out_start) CK(cp(out_start, ds, Z * sizeof(int64_t), ks));
        CK(cudaStreamSynchronize(st));
    }
    return SDTW_OK;
}

// Checkpointed start index: the cost/end DP with round checkpoints at the
// full cost/end speed, then per query a window DP from the checkpoint left of its end and
// the walk-back (sdtw_start.cuh), widening the window for the few queries whose chain
// starts further left.  Returns SDTW_E_ARG (before touching any output) when the launch
// does not qualify, so that the caller can fall back to forward propagation.
constexpr size_t kWinBudget = size_t(8) << 30;   // codes of one launch (all queries of a batch, normally)

sdtw_status run_traceback_ckpt(const float* Q, int64_t Z, int64_t N, float* out_cost, int64_t* out_end,
                               int64_t* out_start, int32_t* path_lo = nullptr, int32_t* path_hi = nullptr) {
    if (N < 1 || Z < 0) return fail(SDTW_E_ARG, "N must be >= 1 and n_queries >= 0");
    if (Z > 0 && (!Q || !out_cost || !out_end || !out_start)) return fail(SDTW_E_ARG, "NULL pointer");
    if (Z > 0x7fffffff || N > 0x7fffffff) return fail(SDTW_E_ARG, "sizes exceed int32");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (!ctx->ref) return fail(SDTW_E_NOREF, "no reference set on this device");
    if (Z == 0) return run_batch(Q, 0, N, out_cost, out_end, out_start, true);
    if (ctx->M >= (1LL << 31) - (1LL << 23)) return fail(SDTW_E_ARG, "reference too long for checkpoints");
    LaunchCfg cfg;
    s = plan(*ctx, Z, N, false, &cfg);
    if (s != SDTW_OK) return s;
    if (cfg.half || cfg.dual || cfg.CL != 1 || cfg.C != 2 || !sdtw::pick_dp_c2ck(cfg.WC, true, false))
        return fail(SDTW_E_ARG, "checkpointed start index needs the two-chain fp32 cost/end kernel");
    const size_t per = (size_t)cfg.Pr * cfg.Pd;
    const size_t ck_bytes = (size_t)Z * per * sizeof(float);
    const bool dbg = getenv("SDTW_DEBUG_PLAN") != nullptr;
    auto now_ms = []() { return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count(); };
    const double t_a = dbg ? now_ms() : 0.0;
    // (cudaMemGetInfo only when the checkpoints must grow: it stalled 8-40 ms now and then,
    // r02 probe at config 5)
    const size_t have_b = ctx->ws_ck_n * sizeof(float);
    if (ck_bytes > have_b) {
        size_t free_b = 0, total_b = 0;
        if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess) { cudaGetLastError(); free_b = 0; }
        if (ck_bytes > (free_b + have_b) / 2)
            return fail(SDTW_E_ARG, "round checkpoints exceed half the free device memory");
    }
    s = grow(&ctx->ws_ck, &ctx->ws_ck_n, (size_t)Z * per);
    if (s != SDTW_OK) return s;
    const int64_t launches0 = g_launches.load();
    // 1) cost/end with round checkpoints (device-side results in bd)
    SegReq r;
    r.mode = 3;
    r.ck = ctx->ws_ck;
    r.ck_Pr = cfg.Pr;
    r.ck_Pd = cfg.Pd;
    BatchDev bd;
    const Options o = g_opt;
    cudaStream_t st = o.stream;
    float ms_dp = 0.0f;
    const double t_b = dbg ? now_ms() : 0.0;
    s = run_batch(Q, Z, N, out_cost, out_end, nullptr, false, &bd, Ragged(), &r);
    const double t_c = dbg ? now_ms() : 0.0;
    if (s != SDTW_OK) return s;
    ms_dp = (float)ctx->last_dp_ms;
    const int ks = ptr_kind(out_start);
    const int kl = path_lo ? ptr_kind(path_lo) : 1, kh = path_hi ? ptr_kind(path_hi) : 1;
    if (ks < 0 || kl < 0 || kh < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    if (o.profile) CK(cudaEventRecord(ctx->ev0, st));
    // 2) windows: per query the round of its end and the previous one first
    std::vector<int64_t> he(Z);
    std::vector<float> hc(Z);
    CK(cudaMemcpyAsync(he.data(), bd.end, Z * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), bd.cost, Z * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t cpr = 32LL * cfg.C * cfg.GW * cfg.WC;
    const bool want_path = path_lo != nullptr;
    // results: start [Z] (+ path [Z][N] x 2), kept across iterations; the per-launch scratch
    // (query lists, codes, row buffers) lives in ws_win and may grow between launches
    const size_t fixed = (size_t)Z * 8 + (want_path ? (size_t)Z * N * 8 : 0);
    if (fixed > ctx->ws_start_n) {
        if (ctx->ws_start) cudaFree(ctx->ws_start);
        ctx->ws_start = nullptr;
        ctx->ws_start_n = 0;
        CK(cudaMalloc(&ctx->ws_start, fixed));
        ctx->ws_start_n = fixed;
    }
    int64_t* ds = reinterpret_cast<int64_t*>(ctx->ws_start);
    int32_t* dlo = want_path ? reinterpret_cast<int32_t*>(ds + Z) : nullptr;
    int32_t* dhi = want_path ? dlo + (size_t)Z * N : nullptr;
    std::vector<int> act, k0(Z, 0), kend(Z, 0);
    for (int64_t q = 0; q < Z; ++q) {
        kend[q] = (int)(he[q] / cpr);
        k0[q] = kend[q];                     // the end's own round first (most chains start in it)
        act.push_back((int)q);               // +inf costs: the walk writes start 0 (and -1 paths)
    }
    std::vector<int64_t> hs(Z, -1);
    int iters = 0;
    while (!act.empty()) {
        if (++iters > 64) return fail(SDTW_E_CUDA, "internal: start windows did not converge");
        // chunks of queries whose codes fit the budget
        size_t pos = 0;
        while (pos < act.size()) {
            int64_t Lmax = 1;
            size_t n = 0;
            size_t bytes = 0;
            while (pos + n < act.size()) {
                const int q = act[pos + n];
                const int64_t L = std::max<int64_t>(1, he[q] - (int64_t)k0[q] * cpr + 1);
                const int64_t Lm = std::max(Lmax, L);
                const size_t W = (size_t)((Lm + 15) / 16);
                const size_t b = (n + 1) * ((size_t)N * W * 4 + (size_t)Lm * 4 + 8);
                if (n > 0 && b > kWinBudget) break;
                Lmax = Lm;
                bytes = b;
                ++n;
            }
            const int W = (int)((Lmax + 15) / 16);
            const size_t need = bytes + 256;
            if (need > ctx->ws_win_n) {
                CK(cudaStreamSynchronize(st));                 // earlier launches may still read it
                if (ctx->ws_win) cudaFree(ctx->ws_win);
                ctx->ws_win = nullptr;
                ctx->ws_win_n = 0;
                CK(cudaMalloc(&ctx->ws_win, need));
                ctx->ws_win_n = need;
            }
            unsigned char* b0 = ctx->ws_win;
            int* dq = reinterpret_cast<int*>(b0);
            int* dk = dq + n;
            uint32_t* codes = reinterpret_cast<uint32_t*>(((uintptr_t)(dk + n) + 15) & ~(uintptr_t)15);
            float* rowbuf = reinterpret_cast<float*>(codes + n * (size_t)N * W);
            std::vector<int> lists(2 * n);
            for (size_t t = 0; t < n; ++t) { lists[t] = act[pos + t]; lists[n + t] = k0[act[pos + t]]; }
            CK(cudaMemcpyAsync(dq, lists.data(), 2 * n * sizeof(int), cudaMemcpyHostToDevice, st));
            CK(cudaStreamSynchronize(st));                     // `lists` is pageable host memory
            sdtw::WinParams wp;
            wp.X = bd.x;
            wp.Y = ctx->ref;
            wp.cost = bd.cost;
            wp.end = bd.end;
            wp.ck = ctx->ws_ck;
            wp.qidx = dq;
            wp.k0 = dk;
            wp.cpr = cpr;
            wp.Pr = cfg.Pr;
            wp.Pd = cfg.Pd;
            wp.N = (int)N;
            wp.W = W;
            wp.Lmax = (int)Lmax;
            wp.codes = codes;
            wp.rowbuf = rowbuf;
            wp.out_start = ds;
            wp.path_lo = dlo;
            wp.path_hi = dhi;
            wp.err_flag = ctx->flag_d;
            const int T = (int)std::min<int64_t>(256, (N + 31) / 32 * 32);
            const size_t wsm = 2 * (size_t)T * sdtw::kWinStrip * sizeof(float);
            if (o.fma) sdtw::window_dp_kernel<true><<<(unsigned)n, T, wsm, st>>>(wp);
            else sdtw::window_dp_kernel<false><<<(unsigned)n, T, wsm, st>>>(wp);
            sdtw::window_walk_kernel<<<(unsigned)((n + 127) / 128), 128, 0, st>>>(wp, (int)n);
            CK(cudaGetLastError());
            g_launches += 2;
            pos += n;
        }
        CK(cudaMemcpyAsync(hs.data(), ds, Z * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        if (*ctx->flag_h) return fail(SDTW_E_CUDA, "internal: window recomputation did not reproduce the batch cost");
        std::vector<int> next;
        for (int q : act)
            if (hs[q] < 0) {                                  // the chain leaves the window: double it
                const int width = kend[q] - k0[q] + 1;
                k0[q] = std::max(0, k0[q] - width);
                next.push_back(q);
            }
        act.swap(next);
    }
    if (o.profile) {
        float ms = 0.f;
        CK(cudaEventRecord(ctx->ev1, st));
        CK(cudaEventSynchronize(ctx->ev1));
        CK(cudaEventElapsedTime(&ms, ctx->ev0, ctx->ev1));
        ctx->last_dp_ms = ms_dp;                          // the DP kernel alone
        ctx->last_win_ms = ms;
    }
    // 3) outputs: the starts (and paths) wherever they live
    CK(cudaMemcpyAsync(out_start, ds, Z * sizeof(int64_t), ks ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    if (want_path) {
        CK(cudaMemcpyAsync(path_lo, dlo, (size_t)Z * N * 4, kl ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(path_hi, dlo + (size_t)Z * N, (size_t)Z * N * 4,
                           kh ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
    ctx->last_launches = g_launches.load() - launches0;
    ctx->last_start_iters = iters;
    if (dbg)
        fprintf(stderr, "[sdtw start] setup %.2f ms, cost/end+checkpoints %.2f ms, windows %.2f ms (%d iterations)\n",
                t_b - t_a, t_c - t_b, now_ms() - t_c, iters);
    return SDTW_OK;
}

// sdtw_path: the batch with start propagation, then per query the window DP with
// predecessor codes and the walk-back (sdtw_path.cuh), in chunks of queries whose codes
// fit the workspace budget.
constexpr size_t kPathBudget = size_t(1) << 30;

sdtw_status run_path(const float* Q, int64_t Z, int64_t N, float* out_cost, int64_t* out_end,
                     int64_t* out_start, int32_t* path_lo, int32_t* path_hi) {
    if (Z > 0 && (!path_lo || !path_hi)) return fail(SDTW_E_ARG, "NULL pointer");
    BatchDev bd;
    sdtw_status s = run_batch(Q, Z, N, out_cost, out_end, out_start, true, &bd);
    if (s != SDTW_OK || Z == 0) return s;
    Ctx* ctx;
    s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    const Options o = g_opt;
    cudaStream_t st = o.stream;
    const int kl = ptr_kind(path_lo), kh = ptr_kind(path_hi);
    if (kl < 0 || kh < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    // window widths (host): one small D2H of the per-query results
    std::vector<int64_t> hs(Z), he(Z);
    std::vector<float> hc(Z);
    CK(cudaMemcpyAsync(hs.data(), bd.start, Z * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(he.data(), bd.end, Z * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(hc.data(), bd.cost, Z * sizeof(float), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    int64_t Lmax = 1;
    for (int64_t q = 0; q < Z; ++q)
        if (hc[q] < INFINITY) Lmax = std::max<int64_t>(Lmax, he[q] - hs[q] + 1);
    const int64_t W = (Lmax + 15) / 16;
    const bool stage_out = (kl == 0 || kh == 0);
    const size_t per_q = (size_t)N * W * 4 + (size_t)Lmax * 4 + (stage_out ? (size_t)N * 8 : 0);
    const int64_t chunk = std::min<int64_t>(Z, (int64_t)(kPathBudget / per_q));
    if (chunk < 1) return fail(SDTW_E_NOMEM, "path window too large for the workspace budget");
    const size_t need = (size_t)chunk * per_q + 256;
    if (need > ctx->ws_path_n) {
        if (ctx->ws_path) cudaFree(ctx->ws_path);
        ctx->ws_path = nullptr;
        ctx->ws_path_n = 0;
        CK(cudaMalloc(&ctx->ws_path, need));
        ctx->ws_path_n = need;
    }
    uint32_t* codes = reinterpret_cast<uint32_t*>(ctx->ws_path);
    float* rowbuf = reinterpret_cast<float*>(codes + (size_t)chunk * N * W);
    int32_t* slo = reinterpret_cast<int32_t*>(rowbuf + (size_t)chunk * Lmax);
    int32_t* shi = slo + (size_t)chunk * N;
    CK(cudaMemsetAsync(ctx->flag_d, 0, sizeof(int), st));
    const int T = (int)std::min<int64_t>(256, (N + 31) / 32 * 32);
    for (int64_t q0 = 0; q0 < Z; q0 += chunk) {
        const int zc = (int)std::min<int64_t>(chunk, Z - q0);
        sdtw::PathParams p;
        p.X = bd.x + q0 * N;
        p.Y = ctx->ref;
        p.cost = bd.cost + q0;
        p.start = bd.start + q0;
        p.end = bd.end + q0;
        p.N = (int)N;
        p.W = (int)W;
        p.Lmax = (int)Lmax;
        p.codes = codes;
        p.rowbuf = rowbuf;
        p.path_lo = stage_out ? slo : path_lo + q0 * N;
        p.path_hi = stage_out ? shi : path_hi + q0 * N;
        p.err_flag = ctx->flag_d;
        if (o.fma) sdtw::path_dp_kernel<true><<<zc, T, 2 * T * sizeof(float), st>>>(p);
        else sdtw::path_dp_kernel<false><<<zc, T, 2 * T * sizeof(float), st>>>(p);
        sdtw::path_walk_kernel<<<(zc + 127) / 128, 128, 0, st>>>(p, zc);
        CK(cudaGetLastError());
        g_launches += 2;
        if (stage_out) {
            CK(cudaMemcpyAsync(path_lo + q0 * N, slo, (size_t)zc * N * 4,
                               kl ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
            CK(cudaMemcpyAsync(path_hi + q0 * N, shi, (size_t)zc * N * 4,
                               kh ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
        }
    }
    CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*ctx->flag_h) return fail(SDTW_E_CUDA, "internal: path recomputation did not reproduce the batch result");
    ctx->last_launches += 2 * ((Z + chunk - 1) / chunk);
    return SDTW_OK;
}

// ------------------------------------------------------------------ reference split
// Overtaking test of a correction (DESIGN.md §13/§14): flag[q] = all rows B >= F.
__global__ void dominate_kernel(const float* __restrict__ B, const float* __restrict__ F, int64_t N,
                                int32_t* flag) {
    const int64_t q = blockIdx.x;
    int lt = 0;
    for (int64_t i = threadIdx.x; i < N; i += blockDim.x) lt |= !(B[q * N + i] >= F[q * N + i]);
    lt = __syncthreads_or(lt);
    if (threadIdx.x == 0) flag[q] = lt ? 0 : 1;
}

// Lexicographic (cost, end) minimum over the valid candidate sets of each query.
__global__ void merge_kernel(const float* __restrict__ cost, const int64_t* __restrict__ end,
                             const int32_t* __restrict__ valid, int64_t n_sets, int64_t Z, float* out_cost,
                             int64_t* out_end, int32_t* out_invalid) {
    const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= Z) return;
    float bc = INFINITY;
    int64_t be = INT64_MAX;
    int inv = 0;
    for (int64_t k = 0; k < n_sets; ++k) {
        if (valid && !valid[k * Z + q]) { inv = 1; continue; }
        const float c = cost[k * Z + q];
        const int64_t e = end[k * Z + q];
        if (c < bc || (c == bc && e < be)) { bc = c; be = e; }
    }
    if (!(bc < INFINITY)) be = 0;                      // no path reaches the last row (or overflow)
    out_cost[q] = bc;
    out_end[q] = be;
    if (out_invalid) out_invalid[q] = inv;
}

}  // namespace

extern "C" {

sdtw_status sdtw_set_reference(const float* Y, int64_t M) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (M < 1 || !Y) return fail(SDTW_E_ARG, "M must be >= 1 and Y non-NULL");
    if (M > 0x7fffffffLL - 4096) return fail(SDTW_E_ARG, "M exceeds int32 range");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    cudaStream_t st = g_opt.stream;
    const int64_t Malloc = (M + 63) / 64 * 64 + 64;
    float* buf = nullptr;
    CK(cudaMalloc(&buf, Malloc * sizeof(float)));
    const int kind = ptr_kind(Y);
    if (kind < 0) { cudaFree(buf); return fail(SDTW_E_ARG, "device pointer on another device"); }
    cudaError_t e = cudaMemcpyAsync(buf, Y, M * sizeof(float),
                                    kind ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st);
    if (e != cudaSuccess) { cudaFree(buf); return cuda_fail(e, "cudaMemcpyAsync(reference)"); }
    const int nparts = 1184;
    e = cudaMemsetAsync(ctx->flag_d, 0, sizeof(int), st);
    if (e != cudaSuccess) { cudaFree(buf); return cuda_fail(e, "cudaMemsetAsync(flag)"); }
    sdtw::ref_partials_kernel<<<nparts, 256, 0, st>>>(buf, M, ctx->ws_part, ctx->flag_d);
    sdtw::ref_stats_kernel<<<1, 256, 0, st>>>(ctx->ws_part, nparts, M, ctx->ws_part + 4 * 4096);
    const int norm = g_opt.normalize;
    sdtw::ref_apply_kernel<<<1184, 256, 0, st>>>(buf, M, Malloc, ctx->ws_part + 4 * 4096, norm);   // in place
    g_launches += 3;
    e = cudaGetLastError();
    if (e == cudaSuccess) e = cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { cudaFree(buf); return cuda_fail(e, "set_reference kernels"); }
    if (*ctx->flag_h) { cudaFree(buf); return fail(SDTW_E_NONFINITE, "reference contains a non-finite sample"); }
    if (ctx->ref) cudaFree(ctx->ref);
    ctx->ref = buf;
    if (ctx->ref_q8) cudaFree(ctx->ref_q8);          // uint8 codes: rebuilt for the new reference
    ctx->ref_q8 = nullptr;
    ctx->q8_clip = -1;
    ctx->M = M;
    ctx->Malloc = Malloc;
    ctx->ref_normalized = norm;
    return SDTW_OK;
}

sdtw_status sdtw_batch(const float* Q, int64_t n_queries, int64_t N, float* out_cost, int64_t* out_end) {
    std::lock_guard<std::mutex> lk(g_mu);
    return run_batch(Q, n_queries, N, out_cost, out_end, nullptr, false);
}

sdtw_status sdtw_batch_columns(const float* Q, int64_t n_queries, int64_t N, float* out_cost, int64_t* out_end,
                               float* col_check, float* col_last, int64_t* check_cols) {
    std::lock_guard<std::mutex> lk(g_mu);
    if ((col_check && ptr_kind(col_check) != 1) || (col_last && ptr_kind(col_last) != 1))
        return fail(SDTW_E_ARG, "column outputs must be device pointers on the current device");
    SegReq r;
    r.mode = 1;
    r.col_check = col_check;
    r.col_last = col_last;
    r.check_cols = check_cols;
    return run_batch(Q, n_queries, N, out_cost, out_end, nullptr, false, nullptr, Ragged(), &r);
}

sdtw_status sdtw_boundary_dp(const float* Q, int64_t n_queries, int64_t N, const float* boundary, int free_start,
                             int64_t n_cols, float* out_cost, int64_t* out_end, float* col_out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if ((boundary && ptr_kind(boundary) != 1) || (col_out && ptr_kind(col_out) != 1))
        return fail(SDTW_E_ARG, "boundary / column must be device pointers on the current device");
    if (n_cols < 0) return fail(SDTW_E_ARG, "n_cols must be >= 0");
    const Options saved = g_opt;
    if (g_opt.sched == 0) g_opt.sched = 3;               // one unit per query on the speculative path
    SegReq r;
    r.mode = 2;
    r.bnd = boundary;
    r.free_start = free_start ? 1 : 0;
    r.cols = n_cols;
    r.col_out = col_out;
    const sdtw_status s = run_batch(Q, n_queries, N, out_cost, out_end, nullptr, false, nullptr, Ragged(), &r);
    g_opt = saved;
    return s;
}

sdtw_status sdtw_round_columns(int64_t N, int64_t* cols) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!cols || N < 1) return fail(SDTW_E_ARG, "NULL pointer or N < 1");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    Ctx probe = *ctx;                                    // the width does not depend on the reference:
    probe.M = 1LL << 24;                                 // plan against a stand-in length
    LaunchCfg cfg;
    s = plan(probe, 1, N, false, &cfg);
    if (s != SDTW_OK) return s;
    *cols = 32LL * cfg.C * cfg.GW * cfg.WC;
    return SDTW_OK;
}

sdtw_status sdtw_traceback(const float* Q, int64_t n_queries, int64_t N, float* out_cost, int64_t* out_end,
                           int64_t* out_start) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_opt.start != 1) {
        // checkpointed start index; SDTW_E_ARG from it means "does not qualify" (no output
        // written yet) -- fall back to forward propagation unless it was forced
        const sdtw_status s = run_traceback_ckpt(Q, n_queries, N, out_cost, out_end, out_start);
        if (s != SDTW_E_ARG || g_opt.start == 2) return s;
    }
    return run_batch(Q, n_queries, N, out_cost, out_end, out_start, true);
}

sdtw_status sdtw_batch_ragged(const float* Q, const int64_t* offsets, int64_t n_queries, float* out_cost,
                              int64_t* out_end, int64_t* out_start) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n_queries < 0) return fail(SDTW_E_ARG, "n_queries must be >= 0");
    if (n_queries == 0) return run_batch(Q, 0, 1, out_cost, out_end, out_start, out_start != nullptr);
    if (!offsets) return fail(SDTW_E_ARG, "NULL pointer");
    if (n_queries > 0x7fffffff) return fail(SDTW_E_ARG, "sizes exceed int32");
    const int ko = ptr_kind(offsets);
    if (ko < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    std::vector<int64_t> off((size_t)n_queries + 1);
    if (ko) {
        const cudaError_t e = cudaMemcpy(off.data(), offsets, off.size() * 8, cudaMemcpyDeviceToHost);
        if (e != cudaSuccess) return cuda_fail(e, "cudaMemcpy(offsets)");
    } else {
        memcpy(off.data(), offsets, off.size() * 8);
    }
    if (off[0] != 0) return fail(SDTW_E_ARG, "offsets[0] must be 0");
    int64_t nmax = 0, nmin = INT64_MAX;
    for (int64_t q = 0; q < n_queries; ++q) {
        const int64_t n = off[q + 1] - off[q];
        if (n < 1) return fail(SDTW_E_ARG, "every query needs >= 1 sample (offsets strictly increasing)");
        nmax = std::max(nmax, n);
        nmin = std::min(nmin, n);
    }
    if (nmax > 0x7fffffff) return fail(SDTW_E_ARG, "query length exceeds int32");
    Ragged rg;
    rg.off = &off;
    rg.nmin = nmin;
    return run_batch(Q, n_queries, nmax, out_cost, out_end, out_start, out_start != nullptr, nullptr, rg);
}

sdtw_status sdtw_path(const float* Q, int64_t n_queries, int64_t N, float* out_cost, int64_t* out_end,
                      int64_t* out_start, int32_t* path_lo, int32_t* path_hi) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (g_opt.start != 1 && n_queries > 0 && path_lo && path_hi) {
        // the checkpointed start's walk-back IS the warp path (same window, same codes)
        const sdtw_status s = run_traceback_ckpt(Q, n_queries, N, out_cost, out_end, out_start, path_lo, path_hi);
        if (s != SDTW_E_ARG || g_opt.start == 2) return s;
    }
    return run_path(Q, n_queries, N, out_cost, out_end, out_start, path_lo, path_hi);
}

sdtw_status sdtw_batch_q8(const float* Q, int64_t n_queries, int64_t N, int32_t* out_cost, int64_t* out_end) {
    std::lock_guard<std::mutex> lk(g_mu);
    const Options saved = g_opt;
    g_opt.precision = 8;
    g_opt.q8_int_out = 1;
    // the integer cost travels as the fp32 bit pattern of the int32 through the pipeline
    const sdtw_status s = run_batch(Q, n_queries, N, reinterpret_cast<float*>(out_cost), out_end, nullptr, false);
    g_opt = saved;
    return s;
}

sdtw_status sdtw_q8_codebook(float* lo, float* hi) {
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (!ctx->ref) return fail(SDTW_E_NOREF, "no reference set on this device");
    s = ensure_q8(ctx, g_opt.stream);
    if (s != SDTW_OK) return s;
    if (lo) *lo = ctx->q8_lo;
    if (hi) *hi = ctx->q8_hi;
    return SDTW_OK;
}

sdtw_status sdtw_quantize(const float* in, int64_t n, uint8_t* out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n < 0 || (n > 0 && (!in || !out))) return fail(SDTW_E_ARG, "n must be >= 0 and pointers non-NULL");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (!ctx->ref) return fail(SDTW_E_NOREF, "no reference set on this device");
    if (n == 0) return SDTW_OK;
    cudaStream_t st = g_opt.stream;
    s = ensure_q8(ctx, st);
    if (s != SDTW_OK) return s;
    const int ki = ptr_kind(in), ko = ptr_kind(out);
    if (ki < 0 || ko < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    const float* id = in;
    if (ki == 0) {
        s = grow(&ctx->ws_q, &ctx->ws_q_n, (size_t)n);
        if (s != SDTW_OK) return s;
        CK(cudaMemcpyAsync(ctx->ws_q, in, (size_t)n * sizeof(float), cudaMemcpyHostToDevice, st));
        id = ctx->ws_q;
    }
    unsigned char* od = out;
    if (ko == 0) {
        s = grow(&ctx->ws_out, &ctx->ws_out_n, (size_t)n);
        if (s != SDTW_OK) return s;
        od = ctx->ws_out;
    }
    CK(cudaMemsetAsync(ctx->flag_d, 0, sizeof(int), st));
    sdtw::finite_check_kernel<<<4 * ctx->sms, 256, 0, st>>>(id, n, ctx->flag_d);
    sdtw::q8_codes_u8_kernel<<<4 * ctx->sms, 256, 0, st>>>(id, n, q8_codebook_dev(ctx), od);
    g_launches += 2;
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*ctx->flag_h) return fail(SDTW_E_NONFINITE, "input contains a non-finite sample");
    if (ko == 0) {
        CK(cudaMemcpyAsync(out, od, (size_t)n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
    }
    return SDTW_OK;
}

sdtw_status sdtw_znormalize(const float* in, int64_t n_series, int64_t len, float* out) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n_series < 0 || len < 1) return fail(SDTW_E_ARG, "len must be >= 1 and n_series >= 0");
    if (n_series > 0 && (!in || !out)) return fail(SDTW_E_ARG, "NULL pointer");
    if (n_series > 0x7fffffff) return fail(SDTW_E_ARG, "n_series exceeds int32");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (n_series == 0) return SDTW_OK;
    cudaStream_t st = g_opt.stream;
    const int ki = ptr_kind(in), ko = ptr_kind(out);
    if (ki < 0 || ko < 0) return fail(SDTW_E_ARG, "device pointer on another device");
    const size_t nel = (size_t)n_series * (size_t)len;
    const float* id = in;
    if (ki == 0) {
        s = grow(&ctx->ws_q, &ctx->ws_q_n, nel);
        if (s != SDTW_OK) return s;
        CK(cudaMemcpyAsync(ctx->ws_q, in, nel * sizeof(float), cudaMemcpyHostToDevice, st));
        id = ctx->ws_q;
    }
    float* od = out;
    if (ko == 0) {
        s = grow(&ctx->ws_x, &ctx->ws_x_n, nel);
        if (s != SDTW_OK) return s;
        od = ctx->ws_x;
    }
    // write to a staging buffer when output is device memory too, so that no
    // partial result is written if a sample is non-finite
    if (ko == 1) {
        s = grow(&ctx->ws_x, &ctx->ws_x_n, nel);
        if (s != SDTW_OK) return s;
        od = ctx->ws_x;
    }
    CK(cudaMemsetAsync(ctx->flag_d, 0, sizeof(int), st));
    sdtw::znorm_rows_kernel<<<(unsigned)n_series, 256, 0, st>>>(id, od, len, 1, ctx->flag_d);
    CK(cudaGetLastError());
    g_launches++;
    CK(cudaMemcpyAsync(ctx->flag_h, ctx->flag_d, sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (*ctx->flag_h) return fail(SDTW_E_NONFINITE, "input contains a non-finite sample");
    CK(cudaMemcpyAsync(out, od, nel * sizeof(float), ko ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    return SDTW_OK;
}

sdtw_status sdtw_set_option(int key, int64_t v) {
    std::lock_guard<std::mutex> lk(g_mu);
    switch (key) {
        case SDTW_OPT_NORMALIZE: if (v != 0 && v != 1) break; g_opt.normalize = (int)v; return SDTW_OK;
        case SDTW_OPT_FMA: if (v != 0 && v != 1) break; g_opt.fma = (int)v; return SDTW_OK;
        case SDTW_OPT_SEGMENT_W: if (v < 0 || v > 64) break; g_opt.segment_w = (int)v; return SDTW_OK;
        case SDTW_OPT_LANES: if (v < 0 || v > 12) break; g_opt.lanes = (int)v; return SDTW_OK;
        case SDTW_OPT_CLUSTER: if (v < 0 || v > 16) break; g_opt.cluster = (int)v; return SDTW_OK;
        case SDTW_OPT_STREAM: g_opt.stream = reinterpret_cast<cudaStream_t>(v); return SDTW_OK;
        case SDTW_OPT_PACKED: if (v < -1 || v > 4) break; g_opt.packed = (int)v; return SDTW_OK;
        case SDTW_OPT_CHUNK: if (v < 0 || v > 256) break; g_opt.chunk = (int)v; return SDTW_OK;
        case SDTW_OPT_PROFILE: if (v != 0 && v != 1) break; g_opt.profile = (int)v; return SDTW_OK;
        case SDTW_OPT_RING: if (v < 0 || v > 16384) break; g_opt.ring = (int)v; return SDTW_OK;
        case SDTW_OPT_SCHED: if (v < 0 || v > 3) break; g_opt.sched = (int)v; return SDTW_OK;
        case SDTW_OPT_SEGMENTS: if (v < 0 || v > 4096) break; g_opt.segments = (int)v; return SDTW_OK;
        case SDTW_OPT_WORKERS: if (v < 0 || v > 32) break; g_opt.workers = (int)v; return SDTW_OK;
        case SDTW_OPT_PRECISION: if (v != 8 && v != 16 && v != 32) break; g_opt.precision = (int)v; return SDTW_OK;
        case SDTW_OPT_Q8_PRUNE: if (v < -1 || v > 255) break; g_opt.q8_prune = (int)v; return SDTW_OK;
        case SDTW_OPT_Q8_CLIP: if (v < 0 || v >= 500000) break; g_opt.q8_clip = (int)v; return SDTW_OK;
        case SDTW_OPT_QUERY_ROWS: if (v < 0 || v > 2) break; g_opt.query_rows = (int)v; return SDTW_OK;
        case SDTW_OPT_PAD: if (v < 0 || v > (1 << 20)) break; g_opt.pad = (int)v; return SDTW_OK;
        case SDTW_OPT_SPEC_ROUNDS: if (v < 0 || v > 4096) break; g_opt.spec_rounds = (int)v; return SDTW_OK;
        case SDTW_OPT_START: if (v < 0 || v > 2) break; g_opt.start = (int)v; return SDTW_OK;
        default: return fail(SDTW_E_ARG, "unknown option key " + std::to_string(key));
    }
    return fail(SDTW_E_ARG, "bad value for option " + std::to_string(key));
}

sdtw_status sdtw_get_option(int key, int64_t* v) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!v) return fail(SDTW_E_ARG, "NULL pointer");
    switch (key) {
        case SDTW_OPT_NORMALIZE: *v = g_opt.normalize; return SDTW_OK;
        case SDTW_OPT_FMA: *v = g_opt.fma; return SDTW_OK;
        case SDTW_OPT_SEGMENT_W: *v = g_opt.segment_w; return SDTW_OK;
        case SDTW_OPT_LANES: *v = g_opt.lanes; return SDTW_OK;
        case SDTW_OPT_CLUSTER: *v = g_opt.cluster; return SDTW_OK;
        case SDTW_OPT_STREAM: *v = reinterpret_cast<int64_t>(g_opt.stream); return SDTW_OK;
        case SDTW_OPT_PACKED: *v = g_opt.packed; return SDTW_OK;
        case SDTW_OPT_CHUNK: *v = g_opt.chunk; return SDTW_OK;
        case SDTW_OPT_PROFILE: *v = g_opt.profile; return SDTW_OK;
        case SDTW_OPT_RING: *v = g_opt.ring; return SDTW_OK;
        case SDTW_OPT_SCHED: *v = g_opt.sched; return SDTW_OK;
        case SDTW_OPT_SEGMENTS: *v = g_opt.segments; return SDTW_OK;
        case SDTW_OPT_WORKERS: *v = g_opt.workers; return SDTW_OK;
        case SDTW_OPT_PRECISION: *v = g_opt.precision; return SDTW_OK;
        case SDTW_OPT_Q8_PRUNE: *v = g_opt.q8_prune; return SDTW_OK;
        case SDTW_OPT_Q8_CLIP: *v = g_opt.q8_clip; return SDTW_OK;
        case SDTW_OPT_QUERY_ROWS: *v = g_opt.query_rows; return SDTW_OK;
        case SDTW_OPT_STAT_FIXUP_DEPTH: {
            Ctx* ctx;
            const sdtw_status s = get_ctx(&ctx);
            if (s != SDTW_OK) return s;
            *v = ctx->last_fix_depth;
            return SDTW_OK;
        }
        case SDTW_OPT_PAD: *v = g_opt.pad; return SDTW_OK;
        case SDTW_OPT_SPEC_ROUNDS: *v = g_opt.spec_rounds; return SDTW_OK;
        case SDTW_OPT_START: *v = g_opt.start; return SDTW_OK;
        default: return fail(SDTW_E_ARG, "unknown option key " + std::to_string(key));
    }
}

sdtw_status sdtw_spec_recomputed(int64_t* n) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (!n) return fail(SDTW_E_ARG, "NULL pointer");
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    *n = ctx->last_fixups;
    return SDTW_OK;
}

sdtw_status sdtw_profile(double* dp_ms, int64_t* launches) {
    std::lock_guard<std::mutex> lk(g_mu);
    Ctx* ctx;
    sdtw_status s = get_ctx(&ctx);
    if (s != SDTW_OK) return s;
    if (dp_ms) *dp_ms = ctx->last_dp_ms;
    if (launches) *launches = ctx->last_launches;
    return SDTW_OK;
}

int64_t sdtw_launch_count(void) { return g_launches.load(); }

const char* sdtw_last_error(void) { return g_err.c_str(); }

void sdtw_release(void) {
    std::lock_guard<std::mutex> lk(g_mu);
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDev) return;
    Ctx& c = g_ctx[dev];
    if (!c.init) return;
    cudaDeviceSynchronize();
    cudaFree(c.ref);
    cudaFree(c.ws_q);
    cudaFree(c.ws_x);
    cudaFree(c.ws_out);
    cudaFree(c.ws_part);
    cudaFree(c.ws_sched);
    cudaFree(c.ws_path);
    cudaFree(c.ws_rag);
    cudaFree(c.order_d);
    cudaFree(c.utab_d);
    for (int k = 0; k < Ctx::kFixDepth; ++k) {
        cudaFree(c.ws_fix[k]);
        cudaFree(c.ws_fixck[k]);
    }
    cudaFree(c.ws_ck);
    cudaFree(c.ws_ckc);
    cudaFree(c.ws_win);
    cudaFree(c.ws_start);
    cudaFree(c.ref_q8);
    cudaFree(c.q8_ws);
    cudaFree(c.ws_xq);
    cudaFree(c.ws_xg);
    cudaFree(c.flag_d);
    cudaFreeHost(c.flag_h);
    cudaEventDestroy(c.ev0);
    cudaEventDestroy(c.ev_sched);
    cudaEventDestroy(c.ev1);
    c = Ctx();
}

sdtw_status sdtw_columns_dominate(const float* B, const float* F, int64_t n_queries, int64_t N, int32_t* out_flag) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n_queries < 0 || N < 1) return fail(SDTW_E_ARG, "N must be >= 1 and n_queries >= 0");
    if (n_queries == 0) return SDTW_OK;
    if (n_queries > 0x7fffffff) return fail(SDTW_E_ARG, "n_queries exceeds int32");
    if (ptr_kind(B) != 1 || ptr_kind(F) != 1 || ptr_kind(out_flag) != 1)
        return fail(SDTW_E_ARG, "B, F and out_flag must be device pointers on the current device");
    const cudaStream_t st = g_opt.stream;
    dominate_kernel<<<(unsigned)n_queries, 256, 0, st>>>(B, F, N, out_flag);
    CK(cudaGetLastError());
    g_launches++;
    CK(cudaStreamSynchronize(st));
    return SDTW_OK;
}

sdtw_status sdtw_merge_candidates(const float* cost, const int64_t* end, const int32_t* valid, int64_t n_sets,
                                  int64_t n_queries, float* out_cost, int64_t* out_end, int32_t* out_invalid) {
    std::lock_guard<std::mutex> lk(g_mu);
    if (n_sets < 1 || n_queries < 0) return fail(SDTW_E_ARG, "n_sets must be >= 1 and n_queries >= 0");
    if (n_queries == 0) return SDTW_OK;
    if (ptr_kind(cost) != 1 || ptr_kind(end) != 1 || ptr_kind(out_cost) != 1 || ptr_kind(out_end) != 1 ||
        (valid && ptr_kind(valid) != 1) || (out_invalid && ptr_kind(out_invalid) != 1))
        return fail(SDTW_E_ARG, "candidate and output arrays must be device pointers on the current device");
    const cudaStream_t st = g_opt.stream;
    merge_kernel<<<(unsigned)((n_queries + 127) / 128), 128, 0, st>>>(cost, end, valid, n_sets, n_queries, out_cost,
                                                                      out_end, out_invalid);
    CK(cudaGetLastError());
    g_launches++;
    CK(cudaStreamSynchronize(st));
    return SDTW_OK;
}

int sdtw_version(void) { return 2; }

#define SDTW_STR2(x) #x
#define SDTW_STR(x) SDTW_STR2(x)
const char* sdtw_build_info(void) {
    return "libsdtw " SDTW_STR(__CUDACC_VER_MAJOR__) "." SDTW_STR(__CUDACC_VER_MINOR__) "." SDTW_STR(
        __CUDACC_VER_BUILD__) " nvcc/ptxas, sm_100a, float-pair pack mode " SDTW_STR(SDTW_MOV_ASM);
}

}  // extern "C"
