// Exact-order (bit-identical to a left-to-right loop) fp64 summation on the GPU.
// Algorithm and invariants: seqsum_core.h. Two launches per sum (the look-back
// flags are left zeroed by the fused scan+chain; only the split path of row slabs
// clears them with a memset):
//
//   k_ss_walk       : one CTA of kSsWT = 128 threads per chunk of 128*EPT terms (EPT = 32; 8 for sums of
//                     <= 2^20 terms), chunk = blockIdx.x (in-order dispatch, so every
//                     look-back predecessor is resident). (1) load the chunk's terms
//                     (striped, coalesced) into shared memory; (2) publish its
//                     approximate sum and get the approximate prefix of all earlier
//                     chunks by a decoupled look-back on 16-byte value+status words:
//                     the speculated running sum at the chunk start; (3) each thread
//                     walks its EPT consecutive terms from its speculated state,
//                     splitting them into in-binade integer segments and break
//                     elements; (4) uniform chunks (every thread one segment in the
//                     same binade) merge by an int64 scan, others by a block
//                     segmented scan; each break emits one record (the merged run
//                     before it + the break value) into the chunk's record slots.
//   k_ss_scan_chain : a thread per chunk: segmented scan of the chunk aggregates with
//                     a look-back over CTA aggregates (the run carried into each
//                     chunk, its first record's position), record compaction; then
//                     the CTA that finishes last replays the records from the exact
//                     state 0.0: validate the run and apply it as one integer add,
//                     then one real IEEE add for the break. A run that fails
//                     validation (wrong speculation) is re-summed literally over its
//                     own element range. (k_ss_scan2 + k_ss_chain when row slabs chain
//                     across ranks.)
//
// Term generators: `double term(int s, long long k)` returns term k (in the
// reference's k = j*nx + i order) of sum s.
#pragma once

#include "common.cuh"
#include "seqsum_core.h"

namespace gmg_dev {

constexpr int kSsT = 256;             // threads of the chain / partial-sum kernels
constexpr int kSsWT = 128;            // threads per chunk in the walk (6 CTAs per SM)
#ifndef GMG_WALK_MINB
#define GMG_WALK_MINB 6  // walk CTAs per SM the register budget is sized for
#endif
constexpr int kSsEPT = 32;            // terms per thread
constexpr int kSsC = kSsWT * kSsEPT;  // terms per chunk (large sums)
constexpr int kSsPC = kSsT * kSsEPT;  // terms per CTA of the fast-mode partial sums
constexpr int kSsEPTs = 8;            // terms per thread for small sums
constexpr int kSsCs = kSsWT * kSsEPTs; // terms per chunk (small sums)
constexpr long long kSsSmallMax = 1ll << 20;  // sums up to this length walk in small chunks (GMG_SS_SMALL_MAX)
constexpr uint32_t kRecOpen = 1u << 16;  // Rec.meta: the carried-in run is still to be prepended
constexpr int kSsBatch = 1024;        // records staged per chain batch
constexpr int kSsMaxSums = 2;
constexpr int kSsRMax = 512;           // records a chunk may store; more -> exact re-walk
constexpr int kSsRunCap = 32;         // a merged run never spans more than this many chunks

// Per-sum look-back state. ticket (unused), total, flag[0] (completion counter of the fused
// scan+chain) and cflag are zero when a walk starts: set by the host's memset or left so by
// the previous fused scan+chain.
struct SsState {
    int* flag;       // [nch] approximate-sum look-back: 0 none, 1 aggregate, 2 inclusive
    int* cflag;      // [nch] run/count look-back flags
    int* ticket;     // [1]
    int* total;      // [1] records stored
    longlong2* lbw;  // [nch] approximate-sum look-back words {value bits, status 0/1/2};
                     //       zeroed at allocation and, after each walk, by k_ss_scan2
    unsigned char* cagg;   // [nch] ChunkAgg
    unsigned char* cincl;  // [nch] ChunkAgg
    gmg_ss::Rec* recs;   // [nch * kSsRMax] per-chunk record slots written by the walk
    gmg_ss::Rec* recs2;  // compacted records in order (k_ss_scan2), read by the chain
    unsigned long long* stats;  // [16] calls, records, chain cycles, re-walk cycles, break adds, re-walks,
                                //      re-walked terms, chunks; walk phase cycles [8..13]
};
struct SsPair {
    SsState s[kSsMaxSums];
};

__device__ __forceinline__ int ld_flag(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_flag(int* p, int v) {
    __threadfence();
    *reinterpret_cast<volatile int*>(p) = v;
}

// ---- segmented run values --------------------------------------------------
// f = "a break happened inside", g = run since the last break (or the whole
// span if none), cnt = records stored.
struct SegF {
    gmg_ss::Seg g;
    int f;
    int cnt;
};
__device__ __forceinline__ SegF segf_id() {
    SegF r;
    r.g = gmg_ss::seg_empty();
    r.f = 0;
    r.cnt = 0;
    return r;
}
// a then b (a older)
__device__ __forceinline__ SegF segf_combine(const SegF& a, const SegF& b) {
    SegF r;
    r.f = a.f | b.f;
    r.g = b.f ? b.g : gmg_ss::seg_merge(a.g, b.g);
    r.cnt = a.cnt + b.cnt;
    return r;
}
__device__ __forceinline__ SegF segf_shfl(const SegF& x, int src, bool up, int o) {
    SegF r;
    const uint32_t meta = static_cast<uint32_t>(x.g.E) | (static_cast<uint32_t>(x.g.neg) << 11) |
                          (static_cast<uint32_t>(x.g.bad) << 12) | (static_cast<uint32_t>(x.f) << 13);
    uint32_t m2;
    if (up) {
        m2 = __shfl_up_sync(0xffffffffu, meta, o);
        r.g.len = __shfl_up_sync(0xffffffffu, x.g.len, o);
        r.cnt = __shfl_up_sync(0xffffffffu, x.cnt, o);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            r.g.Q[p] = __shfl_up_sync(0xffffffffu, x.g.Q[p], o);
            r.g.mn[p] = __shfl_up_sync(0xffffffffu, x.g.mn[p], o);
            r.g.mx[p] = __shfl_up_sync(0xffffffffu, x.g.mx[p], o);
        }
    } else {
        m2 = __shfl_sync(0xffffffffu, meta, src);
        r.g.len = __shfl_sync(0xffffffffu, x.g.len, src);
        r.cnt = __shfl_sync(0xffffffffu, x.cnt, src);
#pragma unroll
        for (int p = 0; p < 2; ++p) {
            r.g.Q[p] = __shfl_sync(0xffffffffu, x.g.Q[p], src);
            r.g.mn[p] = __shfl_sync(0xffffffffu, x.g.mn[p], src);
            r.g.mx[p] = __shfl_sync(0xffffffffu, x.g.mx[p], src);
        }
    }
    r.g.E = m2 & 0x7ff;
    r.g.neg = (m2 >> 11) & 1;
    r.g.bad = (m2 >> 12) & 1;
    r.g.tied = 1;
    r.f = (m2 >> 13) & 1;
    return r;
}

// ChunkAgg: SegF as published between chunks (plain struct, read with __ldcg)
struct ChunkAgg {
    long long Q[2], mn[2], mx[2];
    int meta;  // E | neg<<11 | bad<<12 | f<<13
    int len;
    int cnt;
    int pad;
};
__device__ __forceinline__ void agg_store(unsigned char* base, int c, const SegF& v) {
    ChunkAgg a;
    for (int p = 0; p < 2; ++p) {
        a.Q[p] = v.g.Q[p];
        a.mn[p] = v.g.mn[p];
        a.mx[p] = v.g.mx[p];
    }
    a.meta = v.g.E | (v.g.neg << 11) | (v.g.bad << 12) | (v.f << 13);
    a.len = v.g.len;
    a.cnt = v.cnt;
    a.pad = 0;
    reinterpret_cast<ChunkAgg*>(base)[c] = a;
}
__device__ __forceinline__ SegF agg_load(const unsigned char* base, int c) {
    const ChunkAgg* p = reinterpret_cast<const ChunkAgg*>(base) + c;
    SegF v;
    for (int q = 0; q < 2; ++q) {
        v.g.Q[q] = __ldcg(&p->Q[q]);
        v.g.mn[q] = __ldcg(&p->mn[q]);
        v.g.mx[q] = __ldcg(&p->mx[q]);
    }
    const int meta = __ldcg(&p->meta);
    v.g.E = meta & 0x7ff;
    v.g.neg = (meta >> 11) & 1;
    v.g.bad = (meta >> 12) & 1;
    v.g.tied = 1;
    v.f = (meta >> 13) & 1;
    v.g.len = __ldcg(&p->len);
    v.cnt = __ldcg(&p->cnt);
    return v;
}

// Approximate-prefix look-back words: value and status in one 16-byte word
// (one relaxed vector store / load, no fences). The prefix only seeds the
// speculative walk — the chain validates every segment from the exact state —
// so nothing here can change a result, only the number of re-walks.
__device__ __forceinline__ void lbw_store(longlong2* p, double v, long long status) {
    asm volatile("st.relaxed.gpu.global.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(v)),
                 "l"(status)
                 : "memory");
}
__device__ __forceinline__ longlong2 lbw_load(const longlong2* p) {
    longlong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
    return r;
}

// Decoupled look-back (one warp) for chunk c: approximate double prefix.
__device__ double lookback_d(int c, const longlong2* lbw) {
    const int lane = threadIdx.x & 31;
    double acc = 0.0;
    int p = c - 1;
    while (p >= 0) {
        const int idx = p - lane;
        long long st = 2;
        double v = 0.0;
        if (idx >= 0) {
            longlong2 wd = lbw_load(lbw + idx);
            while (wd.y == 0) {
                __nanosleep(32);
                wd = lbw_load(lbw + idx);
            }
            st = wd.y;
            v = __longlong_as_double(wd.x);
        }
        const unsigned m2 = __ballot_sync(0xffffffffu, st == 2);
        const int stop = m2 ? __ffs(m2) - 1 : 32;
        if (lane > stop) v = 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc += v;
        if (stop < 32) break;
        p -= 32;
    }
    return acc;
}

// Decoupled look-back (one warp) for chunk c: exclusive ordered segmented
// combine of the chunk aggregates (lane l holds predecessor p - l; older
// chunks combine on the left).
__device__ SegF lookback_seg(int c, const int* flag, const unsigned char* agg, const unsigned char* incl) {
    const int lane = threadIdx.x & 31;
    SegF acc = segf_id();
    int p = c - 1;
    while (p >= 0) {
        const int idx = p - lane;
        int f = 2;
        if (idx >= 0) {
            while ((f = ld_flag(flag + idx)) == 0) __nanosleep(64);
        }
        __threadfence();
        const unsigned m2 = __ballot_sync(0xffffffffu, f == 2);
        const int stop = m2 ? __ffs(m2) - 1 : 32;
        SegF v = segf_id();
        if (idx >= 0) {
            if (lane < stop) v = agg_load(agg, idx);
            else if (lane == stop) v = agg_load(incl, idx);
        }
        // ordered reduction: result in lane 0 = v_31 o ... o v_0
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const SegF y = segf_shfl(v, (lane + o) & 31, false, 0);
            if ((lane & (2 * o - 1)) == 0) v = segf_combine(y, v);
        }
        v = segf_shfl(v, 0, false, 0);
        acc = segf_combine(v, acc);
        if (stop < 32) break;
        p -= 32;
    }
    return acc;
}

// ---- block helpers (256 threads) -------------------------------------------
__device__ __forceinline__ double block_sum_d(double x, double* sw /* [8] */) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
    if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = x;
    __syncthreads();
    double t = 0.0;
    for (int w = 0; w < 8; ++w) t += sw[w];
    __syncthreads();
    return t;
}

// Block exclusive sum (NW warps) and the block total, one barrier pair.
template <int NW>
__device__ __forceinline__ double block_excl_sum_tot_d(double x, double* sw /* [NW] */, double* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    double base = 0.0, t = 0.0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        if (q == w) base = t;
        t += sw[q];
    }
    __syncthreads();
    *total = t;
    return base + inc - x;
}

// One segment per thread, all in the same binade and sign (uniform chunk):
// the merged segment's total (returned) and its prefix extremes. P, mn, mx are
// the thread's exact integer total and prefix extremes as doubles.
template <int NW>
__device__ __forceinline__ long long block_seg_i64(double Pd, double mnd, double mxd, long long (*sw)[NW],
                                                   long long* lo, long long* hi) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    const long long P = (long long)Pd;
    long long inc = P;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sw[0][w] = inc;
    __syncthreads();
    long long base = 0, t = 0;
#pragma unroll
    for (int q = 0; q < NW; ++q) {
        if (q == w) base = t;
        t += sw[0][q];
    }
    const long long ex = base + inc - P;
    long long a = ex + (long long)mnd, b = ex + (long long)mxd;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        a = min(a, __shfl_xor_sync(0xffffffffu, a, o));
        b = max(b, __shfl_xor_sync(0xffffffffu, b, o));
    }
    if (lane == 0) {
        sw[1][w] = a;
        sw[2][w] = b;
    }
    __syncthreads();
    a = sw[1][0];
    b = sw[2][0];
#pragma unroll
    for (int q = 1; q < NW; ++q) {
        a = min(a, sw[1][q]);
        b = max(b, sw[2][q]);
    }
    *lo = a;
    *hi = b;
    return t;
}

// Block exclusive segmented scan (NW warps); returns the block inclusive total too.
template <int NW>
__device__ __forceinline__ SegF block_excl_segscan(const SegF& x, SegF* sw /* [NW + 1] */, SegF* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    SegF inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const SegF y = segf_shfl(inc, 0, true, o);
        if (lane >= o) inc = segf_combine(y, inc);
    }
    const SegF ex = segf_shfl(inc, 0, true, 1);
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    // one thread turns the NW warp totals into exclusive bases (in place, the
    // block total in sw[NW]); every thread then reads its warp's base
    if (threadIdx.x == 0) {
        SegF acc = segf_id();
        for (int q = 0; q < NW; ++q) {
            const SegF v = sw[q];
            sw[q] = acc;
            acc = segf_combine(acc, v);
        }
        sw[NW] = acc;
    }
    __syncthreads();
    const SegF base = sw[w];
    *total = sw[NW];
    __syncthreads();
    if (lane == 0) return base;
    return segf_combine(base, ex);
}

__device__ __forceinline__ int ss_pad(int e) { return e + (e >> 5); }

// ---- walk ---------------------------------------------------------------------
// One chunk of WT*EPT terms, already in shared memory (padded layout ss_pad, striped
// by WT): (2) approximate prefix by look-back, (3) thread walks, (4) merge across
// threads, (5) the chunk's aggregate and its records. Block-uniform; WT threads.
template <class TG, int EPT, int WT>
__device__ __forceinline__ void walk_chunk(long long n, int nch, const SsState& S, int s, int c,
                                           const double* __restrict__ tm, const double* __restrict__ pre0) {
    constexpr int NW = WT / 32;
    __shared__ double swd[NW];
    __shared__ SegF sws[NW + 1];
    __shared__ int s_key;
    __shared__ double s_pre;
    __shared__ long long s_i64[3][NW];
    const int t = threadIdx.x;
    constexpr int kC = WT * EPT;
    const long long base = (long long)c * kC;
    const int clen = (int)min((long long)kC, n - base);
    long long ph[7];
    ph[0] = clock64();
    const int e0 = t * EPT;
    const int ne = max(0, min(EPT, clen - e0));
    double ts = 0.0;  // approximate (tree-order) sum of this thread's terms
    if (ne == EPT) {
        double a4[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int m = 0; m < EPT; ++m) a4[m & 3] += tm[ss_pad(e0 + m)];
        ts = (a4[0] + a4[1]) + (a4[2] + a4[3]);
    } else {
        for (int m = 0; m < ne; ++m) ts += tm[ss_pad(e0 + m)];
    }
    ph[1] = clock64();

    // (2) approximate prefix by look-back
    double tot_approx;
    const double ex_approx = block_excl_sum_tot_d<NW>(ts, swd, &tot_approx);
    // pre0: approximate sum of the terms before this range (earlier row slabs)
    const double base_pre = pre0 ? pre0[s] : 0.0;
    if (t == 0) {
        if (c == 0) lbw_store(S.lbw, base_pre + tot_approx, 2);
        else lbw_store(S.lbw + c, tot_approx, 1);
    }
    if (t < 32) {
        const double pre = c == 0 ? base_pre : lookback_d(c, S.lbw);
        if (t == 0) {
            s_pre = pre;
            if (c > 0) lbw_store(S.lbw + c, pre + tot_approx, 2);
        }
    }
    __syncthreads();
    const double pred = s_pre + ex_approx;
    ph[2] = clock64();

    // (3) thread walk, pass 1: leading segment, trailing segment, break count
    gmg_ss::Walker wk;
    gmg_ss::walker_init(wk, pred);
    gmg_ss::Seg lead = gmg_ss::seg_empty();
    int r = 0;
    // Fast path: all EPT terms stay in the binade without ties. The increments
    // q_m = RN(p_m/u) are independent, only their prefix sums are a chain; the
    // range test on the prefix extremes equals the walker's per-step tests (the
    // sign cannot change: |q| < 2^52 <= |M|). Same state and segment as
    // walker_try would leave; otherwise the element-wise walk below.
    bool fast = false;
    if (ne == EPT && wk.E != 0) {
        double P = 0.0, mn = 0.0, mx = 0.0;
        bool ok = true;
#pragma unroll
        for (int m = 0; m < EPT; ++m) {
            const double x = tm[ss_pad(e0 + m)] * wk.inv_u;  // exact power-of-two scaling
            const double q = rint(x);
            ok = ok && (x < gmg_ss::kTwo52 && x > -gmg_ss::kTwo52) && fabs(x - q) != 0.5;
            P = P + q;
            mn = m == 0 ? P : fmin(mn, P);
            mx = m == 0 ? P : fmax(mx, P);
        }
        const double M = wk.M;
        const double lo = static_cast<double>(gmg_ss::kLo), hi = static_cast<double>(gmg_ss::kHi);
        ok = ok && (M >= 0.0 ? (M + mn >= lo && M + mx <= hi) : (M + mx <= -lo && M + mn >= -hi));
        if (ok) {
            wk.segE = wk.E;
            wk.segneg = M < 0.0;
            wk.Q[0] = P;
            wk.mn[0] = mn;
            wk.mx[0] = mx;
            wk.len = EPT;
            wk.M = M + P;
            fast = true;
        }
    }
    if (!fast) {
        for (int m = 0; m < ne; ++m) {
            const double p = tm[ss_pad(e0 + m)];
            if (!gmg_ss::walker_try(wk, p)) {
                if (r == 0) lead = gmg_ss::walker_seg(wk);
                ++r;
                gmg_ss::walker_open(wk);
                gmg_ss::walker_real_add(wk, p);
            }
        }
    }
    // Uniform chunk: every thread took the fast path in the same binade and sign
    // (the common case). The chunk is then one segment, and merging the threads'
    // segments is an int64 exclusive scan of their totals plus a min/max of
    // (prefix + extreme) — no segmented scan, no records unless the run closes.
    if (t == 0) s_key = fast ? wk.segE * 2 + wk.segneg : -1;
    __syncthreads();
    const bool uni = __syncthreads_and(fast && wk.segE * 2 + wk.segneg == s_key);
    ph[3] = clock64();

    // (4) merge runs across threads; records = breaks (+ the final record)
    SegF tot, carry;
    if (uni) {
        tot = segf_id();
        long long lo, hi;
        tot.g.Q[0] = tot.g.Q[1] = block_seg_i64<NW>(wk.Q[0], wk.mn[0], wk.mx[0], s_i64, &lo, &hi);
        tot.g.mn[0] = tot.g.mn[1] = lo;
        tot.g.mx[0] = tot.g.mx[1] = hi;
        tot.g.E = wk.segE;
        tot.g.neg = wk.segneg;
        tot.g.len = clen;
        carry = segf_id();
    } else {
        const gmg_ss::Seg cur = gmg_ss::walker_seg(wk);
        if (r == 0) lead = cur;
        SegF x = segf_id();
        x.f = r > 0;
        x.g = r > 0 ? cur : lead;
        x.cnt = r;
        carry = block_excl_segscan<NW>(x, sws, &tot);
    }
    ph[4] = clock64();
    const bool last = c == nch - 1;
    // every kSsRunCap-th chunk closes its run with a no-break record, so a
    // speculation failure never re-walks more than kSsRunCap chunks
    const bool close = last || (c % kSsRunCap) == kSsRunCap - 1;
    const int R = tot.cnt + (close ? 1 : 0);
    const bool literal = R > kSsRMax;

    // (5) the chunk's aggregate for k_ss_scan2 (the run it carries on, the
    //     records it stores). No look-back: the cross-chunk segmented scan runs
    //     as one small kernel after all walks, and the chunk's first record is
    //     stored "open" (kRecOpen) for k_ss_scan2 to prepend the run carried in.
    SegF mine = tot;
    mine.cnt = literal ? 1 : R;
    if (literal || close) {
        mine.f = 1;
        mine.g = gmg_ss::seg_empty();
    }
    if (t == 0) agg_store(S.cagg, c, mine);
    ph[5] = clock64();
    if (t == 0 && S.stats) {
        for (int q = 0; q < 5; ++q) atomicAdd(S.stats + 8 + q, (unsigned long long)(ph[q + 1] - ph[q]));
        atomicAdd(S.stats + 13, 1ull);
    }
    gmg_ss::Rec* out = S.recs + (long long)c * kSsRMax;
    if (literal) {
        if (t == 0) out[0] = gmg_ss::rec_literal((uint32_t)(base + clen - 1));
        return;
    }
    if (r > 0) {
        // pass 2: emit this thread's records; the first absorbs the run since the
        // last break inside the chunk (and, when there is none, the run carried in)
        const int pos = carry.cnt;
        const gmg_ss::Seg first = carry.g;
        gmg_ss::walker_init(wk, pred);
        int k = 0;
        for (int m = 0; m < ne; ++m) {
            const double p = tm[ss_pad(e0 + m)];
            if (!gmg_ss::walker_try(wk, p)) {
                const gmg_ss::Seg sg = gmg_ss::walker_seg(wk);
                const gmg_ss::Seg g = k == 0 ? gmg_ss::seg_merge(first, sg) : sg;
                gmg_ss::Rec rec = gmg_ss::rec_make(g, true, p, (uint32_t)(base + e0 + m));
                if (k == 0 && !carry.f) rec.meta |= kRecOpen;
                out[pos + k] = rec;
                ++k;
                gmg_ss::walker_open(wk);
                gmg_ss::walker_real_add(wk, p);
            }
        }
    }
    if (close && t == WT - 1) {
        gmg_ss::Rec rec = gmg_ss::rec_make(tot.g, false, 0.0, (uint32_t)(base + clen - 1));
        if (!tot.f) rec.meta |= kRecOpen;
        out[R - 1] = rec;
    }
}


// grid (nch, NS); block kSsWT; dynamic smem (C + C/32) doubles, C = kSsWT * EPT terms
// per chunk (EPT = 32, or 8 for small sums: 4x shorter serial thread walks).
template <class TG, int EPT>
__global__ void __launch_bounds__(kSsWT, GMG_WALK_MINB) k_ss_walk(TG tg, long long n, int nch, SsPair sts,
                                                       const double* __restrict__ pre0) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ double tm[];
    const int s = blockIdx.y, t = threadIdx.x;
    // chunk = blockIdx.x: CTAs are dispatched in increasing linear block order, so every
    // look-back predecessor is already resident (no ticket atomic on the critical path)
    const int c = blockIdx.x;
    constexpr int kC = kSsWT * EPT;
    const long long base = (long long)c * kC;
    const int clen = (int)min((long long)kC, n - base);
    {  // (1) terms: striped (coalesced) loads, all in flight before the smem stores
        double v[EPT];
        tg.template striped<EPT, kSsWT>(s, base + t, clen, v);
#pragma unroll
        for (int m = 0; m < EPT; ++m) tm[ss_pad(m * kSsWT + t)] = v[m];
    }
    __syncthreads();
    walk_chunk<TG, EPT, kSsWT>(n, nch, sts.s[s], s, c, tm, pre0);
}

// ---- cross-chunk scan and record compaction --------------------------------
// Cross-chunk segmented scan + record compaction, single pass. grid (ceil(nch/256), NS);
// 256 threads, a thread per chunk. Block exclusive segmented scan of the chunk
// aggregates, then a decoupled look-back over the CTA aggregates (CTA = blockIdx.x:
// in-order dispatch keeps every predecessor resident),
// giving the run carried into each chunk and its first record's position; the
// warps then copy each chunk's records into the ordered list, prepending the
// carried-in run to an open record (seg_merge is associative, so this equals
// merging in order). CTA aggregates live in cincl[0, nb), inclusive prefixes in
// cincl[nb, 2nb) (cincl is otherwise unused); flags in cflag.
constexpr int kSsScanB = 256;
__device__ __forceinline__ void ss_scan2_body(const SsPair& sts, int nch) {
    __shared__ SegF sws[9];
    __shared__ SegF s_cin[kSsScanB];
    __shared__ int s_cnt[kSsScanB];
    const SsState& S = sts.s[blockIdx.y];
    const int t = threadIdx.x, lane = t & 31, w = t >> 5;
    const int b = blockIdx.x, nb = (nch + kSsScanB - 1) / kSsScanB;
    const int c = b * kSsScanB + t;
    const SegF a = c < nch ? agg_load(S.cagg, c) : segf_id();
    SegF tot;
    const SegF ex = block_excl_segscan<kSsScanB / 32>(a, sws, &tot);
    unsigned char* bagg = S.cincl;
    unsigned char* bincl = S.cincl + (size_t)nb * sizeof(ChunkAgg);
    if (t == 0) {
        if (b == 0) {
            agg_store(bincl, 0, tot);
            st_flag(S.cflag, 2);
        } else {
            agg_store(bagg, b, tot);
            st_flag(S.cflag + b, 1);
        }
    }
    if (w == 0) {
        const SegF pre = b > 0 ? lookback_seg(b, S.cflag, bagg, bincl) : segf_id();
        if (t == 0) {
            const SegF inc = segf_combine(pre, tot);
            if (b > 0) {
                agg_store(bincl, b, inc);
                st_flag(S.cflag + b, 2);
            }
            if (b == nb - 1) *S.total = inc.cnt;
            sws[8] = pre;
        }
    }
    __syncthreads();
    s_cin[t] = segf_combine(sws[8], ex);
    s_cnt[t] = c < nch ? a.cnt : 0;
    if (c < nch) lbw_store(S.lbw + c, 0.0, 0);  // reset the walk's look-back word for the next sum
    __syncthreads();
    // compaction: warp w takes chunks w, w+8, ...; lanes copy a chunk's records
    for (int q = w; q < kSsScanB; q += 8) {
        const int cnt = s_cnt[q];
        if (cnt == 0) continue;
        const SegF& cin = s_cin[q];
        const gmg_ss::Rec* src = S.recs + (long long)(b * kSsScanB + q) * kSsRMax;
        gmg_ss::Rec* dst = S.recs2 + cin.cnt;
        for (int j = lane; j < cnt; j += 32) {
            gmg_ss::Rec r = src[j];
            if (r.meta & kRecOpen) {
                const bool brk = (r.meta >> 12) & 1u;
                r = gmg_ss::rec_make(gmg_ss::seg_merge(cin.g, gmg_ss::rec_seg(r)), brk, r.pb, r.kb);
            }
            dst[j] = r;
        }
    }
}
__global__ void __launch_bounds__(kSsScanB) k_ss_scan2(SsPair sts, int nch) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger(); ss_scan2_body(sts, nch); }

// ---- chain --------------------------------------------------------------------
// Both re-sum paths read terms through a register ring of kSsRing batches of 32
// (lane = term within a batch), so ~kSsRing*256 B per warp are in flight and the
// walk is not bound by one memory round trip per batch.
constexpr int kSsRing = 8;

// Literal left-to-right adds over terms [k0, k1) of sum s, by one warp. The
// adds are one dependent fp64 chain (8 cycles each on B200), so nothing else may
// sit on it: the warp stages kSsLitTile terms in shared memory (coalesced;
// the next tile's loads are in flight in registers meanwhile) and every lane
// runs the same chain from broadcast shared-memory reads.
constexpr int kSsLitTile = 1024;
template <class TG>
__device__ double literal_sum(const TG& tg, int s, double a, long long k0, long long k1, double* tile) {
    const int lane = threadIdx.x & 31;
    constexpr int PER = kSsLitTile / 32;
    double r[PER];
    auto load = [&](long long k) {
#pragma unroll
        for (int j = 0; j < PER; ++j) {
            const long long kk = k + j * 32 + lane;
            r[j] = kk < k1 ? tg.term(s, kk) : 0.0;
        }
    };
    load(k0);
    for (long long k = k0; k < k1; k += kSsLitTile) {
#pragma unroll
        for (int j = 0; j < PER; ++j) tile[j * 32 + lane] = r[j];
        __syncwarp();
        if (k + kSsLitTile < k1) load(k + kSsLitTile);
        const int m = (int)min((long long)kSsLitTile, k1 - k);
        int j = 0;
        for (; j + 8 <= m; j += 8) {
            double v[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) v[q] = tile[j + q];
#pragma unroll
            for (int q = 0; q < 8; ++q) a = a + v[q];
        }
        for (; j < m; ++j) a = a + tile[j];
        __syncwarp();
    }
    return a;
}

// Exact sum of terms [k0, k1) added to sv, by one warp with the integer model:
// 32 terms at a time, an inclusive prefix of q = RN(p/u) across lanes, commit
// up to the first lane that breaks (binade exit, tie, huge term), real add for
// that lane, restart after it. Bit-identical to literal adds, ~5 cycles/term
// when breaks are sparse.
template <class TG>
__device__ double warp_walk(const TG& tg, int s, double sv, long long k0, long long k1) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    double ring[kSsRing];
#pragma unroll
    for (int r = 0; r < kSsRing; ++r) {
        const long long k = k0 + r * 32 + lane;
        ring[r] = k < k1 ? tg.term(s, k) : 0.0;
    }
    for (long long kr = k0; kr < k1; kr += 32 * kSsRing) {
#pragma unroll
        for (int r = 0; r < kSsRing; ++r) {
            const long long k = kr + r * 32;
            if (k >= k1) break;
            const double p = ring[r];
            const long long kn = k + 32 * kSsRing + lane;
            ring[r] = kn < k1 ? tg.term(s, kn) : 0.0;
            const int m = (int)min(32LL, k1 - k);
            int start = 0;
            while (start < m) {
                const uint64_t bits = gmg_ss::dbits(sv);
                const int E = (int)((bits >> 52) & 0x7ff);
                if (E < gmg_ss::kEMin || E > gmg_ss::kEMax) {  // zero/subnormal/huge: one real add
                    sv = sv + __shfl_sync(full, p, start);
                    ++start;
                    continue;
                }
                const double inv_u = gmg_ss::bitsd((uint64_t)(2098 - E) << 52);
                const bool mine = lane >= start && lane < m;
                const double xv = p * inv_u;
                const double fl = floor(xv);
                const double fr = xv - fl;
                const bool bad = !(xv < gmg_ss::kTwo52 && xv > -gmg_ss::kTwo52) || fr == 0.5;
                long long q = (mine && !bad) ? (long long)fl + (fr > 0.5 ? 1 : 0) : 0;
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const long long y = __shfl_up_sync(full, q, o);
                    if (lane >= o) q += y;
                }
                const bool neg = bits >> 63;
                const long long mant = (long long)((bits & ((1ull << 52) - 1)) | (1ull << 52));
                const long long Mn = neg ? mant - q : mant + q;  // |M| after this lane
                const bool ok = !bad && Mn >= gmg_ss::kLo && Mn <= gmg_ss::kHi;
                const unsigned failm = __ballot_sync(full, mine && !ok);
                const int f = failm ? __ffs(failm) - 1 : m;
                if (f > start) {
                    const long long P = __shfl_sync(full, q, f - 1);
                    sv = gmg_ss::compose(neg ? -(mant - P) : mant + P, E);  // signed M + P
                }
                if (f < m) {
                    sv = sv + __shfl_sync(full, p, f);
                    start = f + 1;
                } else {
                    start = m;
                }
            }
        }
    }
    return sv;
}

// Shared memory of the chain (dynamic): two batches of records (the next batch is
// staged while the current one replays), the serial step's operands of both
// batches, and the state entering every record of the current batch.
struct ChainOps {
    long long d[kSsBatch];  // run step on the sum's bit pattern (see chain_decode)
    double pb[kSsBatch];    // break term (-0.0: none)
    int ft[kSsBatch];       // parity handling: bit 0 = f, bit 1 = t (see chain_decode)
};
struct ChainSmem {
    gmg_ss::Rec buf[2][kSsBatch];
    ChainOps op[2];
    double before[kSsBatch];
    double ltile[kSsLitTile];  // literal re-sum staging
};

// Operands of one record's serial step. In a valid run the sum keeps its binade
// and sign, so s + Q*u is the integer add of D = +-Q to the double's bit pattern
// (the magnitude grows by Q for a positive sum, by -Q for a negative one). Q has
// one value per parity of the state entering the run (ties, seqsum_core.h), at
// most one unit apart; the step is written branch-free as
//     bits += d + ((bits ^ f) & t),
// d = the smaller of the two steps, t = 1 if they differ, f = 1 if the even
// state takes the larger one. An empty run adds 0; a record without a break
// element adds -0.0 afterwards (the exact identity). `ok` = false (never seen;
// the variants would have to differ by more than a unit) forces the fallback.
__device__ __forceinline__ void chain_decode(const gmg_ss::Rec& r, long long& d, int& ft, double& pb, bool& ok) {
    const uint32_t meta = r.meta;
    const bool brk = (meta >> 12) & 1u, ne = (meta >> 15) & 1u, negr = (meta >> 11) & 1u;
    const long long D0 = ne ? (negr ? -r.Q[0] : r.Q[0]) : 0;
    const long long D1 = ne ? (negr ? -r.Q[1] : r.Q[1]) : 0;
    d = D0 < D1 ? D0 : D1;
    ft = (D0 != D1 ? 2 : 0) | (D0 > D1 ? 1 : 0);
    ok = D0 - D1 <= 1 && D1 - D0 <= 1;
    pb = brk ? r.pb : -0.0;
}

// Is record r valid from the exact state `before` entering it? (seg_valid on the
// double's bits; literal and bad records never are.)
__device__ __forceinline__ bool chain_valid(const gmg_ss::Rec& r, double before) {
    const uint32_t meta = r.meta;
    const bool lit = (meta >> 14) & 1u, ne = (meta >> 15) & 1u;
    const uint64_t Er = meta & 0x7ffu;
    const bool negr = (meta >> 11) & 1u, badr = (meta >> 13) & 1u;
    const uint64_t bits = gmg_ss::dbits(before);
    const uint64_t E = (bits >> 52) & 0x7ffu;
    const bool v = (bits & 1u) != 0;
    const long long mant = (long long)((bits & ((1ull << 52) - 1)) | (1ull << 52));
    const long long mni = v ? r.mn[1] : r.mn[0], mxi = v ? r.mx[1] : r.mx[0];
    const bool neg = bits >> 63;
    const long long lo_v = neg ? mant - mxi : mant + mni;
    const long long hi_v = neg ? mant - mni : mant + mxi;
    const bool ok_run = E >= (uint64_t)gmg_ss::kEMin && E <= (uint64_t)gmg_ss::kEMax && E == Er && neg == negr &&
                        lo_v >= gmg_ss::kLo && hi_v <= gmg_ss::kHi;
    return !lit && !badr && (!ne || ok_run);
}

// The serial replay of records [q0, cnt) of a decoded batch by one warp, from
// state sv: per record an integer add on the sum's bits (run step) and one fp64
// add (break term) — the only serial dependence is on the sum itself; the
// operands of 32 records sit one per lane and are broadcast by shuffles, off the
// chain. The state entering each record is kept for the validation that
// follows. Nothing is validated here: the caller checks every record against
// before[] afterwards and resumes from the first failure.
__device__ __forceinline__ double chain_serial(const ChainOps& op, double* before, int q0, int cnt, double sv) {
    const int lane = threadIdx.x & 31;
    const unsigned full = 0xffffffffu;
    for (int g = q0; g < cnt; g += 32) {
        const int gn = min(32, cnt - g);
        const int q = g + (lane < gn ? lane : 0);
        const long long d = op.d[q];
        const double pb = op.pb[q];
        const int ft = op.ft[q];
        double x = sv, bf = sv;
        auto step = [&](int k) {
            const long long dk = __shfl_sync(full, d, k);
            const double pk = __shfl_sync(full, pb, k);
            const unsigned ftk = (unsigned)__shfl_sync(full, ft, k);
            const unsigned tk = ftk >> 1;
            if (lane == k) bf = x;
            const uint64_t bits = gmg_ss::dbits(x);
            const unsigned e = ((unsigned)bits ^ ftk) & tk;
            x = gmg_ss::bitsd(bits + (uint64_t)dk + e) + pk;
        };
        if (gn == 32) {
#pragma unroll
            for (int k = 0; k < 32; ++k) step(k);
        } else {
            for (int k = 0; k < gn; ++k) step(k);
        }
        if (lane < gn) before[g + lane] = bf;
        sv = x;
    }
    return sv;
}

// grid (NS); block kSsT; dynamic smem ss_chain_smem(). Per batch of kSsBatch records:
// warp 0 replays the batch serially (chain_serial) while warps 1.. stage and decode the
// next one; then all threads validate the batch in parallel against the states warp 0
// recorded. From the first record that fails (a wrong speculation, a literal chunk) the
// results are discarded: that record's element range is re-summed literally from the
// true state, and the replay resumes after it.
template <class TG>
__device__ __forceinline__ void ss_chain_body(const TG& tg, long long n, const SsState& S, int s,
                                              double* __restrict__ out, const double* __restrict__ start,
                                              unsigned char* smraw) {
    ChainSmem& M = *reinterpret_cast<ChainSmem*>(smraw);
    __shared__ int s_fail;
    __shared__ double s_sv;
    __shared__ unsigned long long s_nbrk;
    const int t = threadIdx.x;
    const int total = *S.total;
    const int nb = (total + kSsBatch - 1) / kSsBatch;
    unsigned n_brk = 0;  // break records this thread staged (stats)
    auto stage_batch = [&](int b, int t0, int nt) {
        const int cn = min(kSsBatch, total - b * kSsBatch);
        const gmg_ss::Rec* src = S.recs2 + (long long)b * kSsBatch;
        gmg_ss::Rec* B = M.buf[b & 1];
        ChainOps& O = M.op[b & 1];
        for (int q = t0; q < cn; q += nt) {
            gmg_ss::Rec r = src[q];
            n_brk += (r.meta >> 12) & 1u;
            bool ok;
            chain_decode(r, O.d[q], O.ft[q], O.pb[q], ok);
            if (!ok) r.meta |= 1u << 13;  // bad: re-summed literally
            B[q] = r;
        }
    };
    if (nb > 0) stage_batch(0, t, kSsT);
    if (t == 0) s_nbrk = 0ull;
    __syncthreads();

    double sv = start ? start[s] : 0.0;  // exact state entering this range (earlier row slabs)
    long long prev = -1;                 // global index of the last element consumed
    unsigned long long n_lit = 0, n_litterms = 0, cyc_lit = 0, n_dense = 0, cyc_dense = 0;
    const long long cyc0 = clock64();
    for (int b = 0; b < nb; ++b) {
        const gmg_ss::Rec* A = M.buf[b & 1];
        const ChainOps& O = M.op[b & 1];
        const int cnt = min(kSsBatch, total - b * kSsBatch);
        int q0 = 0;
        bool staged = false;
        while (q0 < cnt) {
            if (t < 32) {
                const double r = chain_serial(O, M.before, q0, cnt, sv);
                if (t == 0) s_sv = r;
            } else if (!staged && b + 1 < nb) {
                stage_batch(b + 1, t - 32, kSsT - 32);
            }
            staged = true;
            if (t == 0) s_fail = cnt;
            __syncthreads();
            // validation of records [q0, cnt) against the states they were applied to
            int f = cnt;
            for (int q = q0 + t; q < cnt; q += kSsT)
                if (!chain_valid(A[q], M.before[q])) f = min(f, q);
            if (f < cnt) atomicMin(&s_fail, f);
            __syncthreads();
            f = s_fail;
            if (f == cnt) {
                sv = s_sv;
                prev = A[cnt - 1].kb;
                q0 = cnt;
            } else {
                // re-sum the failed record's range exactly from the true state (the break
                // element, if any, is applied after; otherwise kb is inclusive): plain
                // left-to-right adds — a failed record sits where the sum crosses binades
                // often, and there the literal chain (~6 cycles/term) beats an integer walk
                const gmg_ss::Rec& rf = A[f];
                const bool brk_f = (rf.meta >> 12) & 1u, lit_f = (rf.meta >> 14) & 1u;
                const long long kb_f = rf.kb;
                const long long pf = f > 0 ? (long long)A[f - 1].kb : prev;
                const long long k1 = min(brk_f ? kb_f : kb_f + 1, n);
                double s1 = M.before[f];
                if (t < 32) {
                    const long long c0 = clock64();
                    s1 = literal_sum(tg, s, s1, pf + 1, k1, M.ltile);
                    cyc_lit += clock64() - c0;
                    ++n_lit;
                    n_litterms += k1 - (pf + 1);
                    if (lit_f) {
                        ++n_dense;
                        cyc_dense += clock64() - c0;
                    }
                    if (t == 0) s_sv = brk_f ? s1 + rf.pb : s1;
                }
                __syncthreads();
                sv = s_sv;
                prev = kb_f;
                q0 = f + 1;
            }
            __syncthreads();  // s_fail / s_sv / before[] are rewritten by the next round
        }
    }
    if (S.stats) {
        n_brk = __reduce_add_sync(0xffffffffu, n_brk);
        if ((t & 31) == 0 && n_brk) atomicAdd(&s_nbrk, (unsigned long long)n_brk);
        __syncthreads();
    }
    if (t == 0) {
        out[s] = sv;
        if (S.stats) {
            atomicAdd(S.stats + 0, 1ull);
            atomicAdd(S.stats + 1, (unsigned long long)total);
            atomicAdd(S.stats + 2, (unsigned long long)(clock64() - cyc0));
            atomicAdd(S.stats + 3, cyc_lit);
            atomicAdd(S.stats + 4, s_nbrk);
            atomicAdd(S.stats + 5, n_lit);
            atomicAdd(S.stats + 6, n_litterms);
            atomicAdd(S.stats + 14, n_dense);
            atomicAdd(S.stats + 15, cyc_dense);
            atomicAdd(S.stats + 7, (unsigned long long)((n + kSsC - 1) / kSsC));
        }
    }
}

// grid (NS); block kSsT; dynamic smem ss_chain_smem(). One CTA per sum.
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_chain(TG tg, long long n, SsPair sts, double* __restrict__ out,
                                                 const double* __restrict__ start) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smraw[];
    ss_chain_body(tg, n, sts.s[blockIdx.x], (int)blockIdx.x, out, start, smraw);
}

// k_ss_scan2 with the chain fused: the CTA that finishes its sum's compaction
// last (completion counter, threadfence-reduction pattern) replays the records.
// Saves a launch per sum; used when no other range has to chain in first.
template <class TG>
__global__ void __launch_bounds__(kSsScanB) k_ss_scan_chain(TG tg, long long n, SsPair sts, int nch,
                                                           double* __restrict__ out,
                                                           const double* __restrict__ start) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ __align__(16) unsigned char smraw[];
    __shared__ int s_last;
    const SsState& S = sts.s[blockIdx.y];
    ss_scan2_body(sts, nch);
    __threadfence();
    __syncthreads();
    const int nb = (nch + kSsScanB - 1) / kSsScanB;
    if (threadIdx.x == 0) s_last = atomicAdd(S.flag, 1) == nb - 1;  // flag[0]: completion counter
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    ss_chain_body(tg, n, S, (int)blockIdx.y, out, start, smraw);
    // every other CTA of this sum is done with the flags: leave them zeroed for the
    // next sum on this workspace (the host then skips its memset)
    __syncthreads();
    for (int q = threadIdx.x; q < 2 + 2 * nch; q += blockDim.x) S.ticket[q] = 0;
}

// Small sums (n <= kSsDirect): the reference's loop literally. The CTA stages
// the terms in shared memory (coalesced, all loads in flight), then one thread
// adds them left to right from s = 0.0 (stencil.cpp:9-26). One launch instead of
// walk + chain: on the coarse levels the engine's phases are pure latency.
constexpr int kSsDirect = 4096;
template <class TG>
__global__ void __launch_bounds__(256) k_ss_direct(TG tg, int n, double* __restrict__ out,
                                                   const double* __restrict__ start) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ double tv[];
    const int s = blockIdx.x;
    for (int k = threadIdx.x; k < n; k += blockDim.x) tv[k] = tg.term(s, k);
    __syncthreads();
    if (threadIdx.x == 0) {
        double a = start ? start[s] : 0.0;
        int k = 0;
        for (; k + 8 <= n; k += 8) {
            double v[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) v[j] = tv[k + j];
#pragma unroll
            for (int j = 0; j < 8; ++j) a = a + v[j];
        }
        for (; k < n; ++k) a = a + tv[k];
        out[s] = a;
    }
}

// Fast mode: tree-order partial sums per chunk, then one CTA finishes.
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_partial(TG tg, long long n, double* __restrict__ csum, int nch) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    __shared__ double swd[8];
    const int s = blockIdx.y;
    const long long base = (long long)blockIdx.x * kSsPC;
    double acc = 0.0;
#pragma unroll 4
    for (int m = 0; m < kSsEPT; ++m) {
        const long long k = base + m * kSsT + threadIdx.x;
        if (k < n) acc += tg.term(s, k);
    }
    acc = block_sum_d(acc, swd);
    if (threadIdx.x == 0) csum[(long long)s * nch + blockIdx.x] = acc;
}

template <int EPT>
constexpr size_t ss_walk_smem() { return sizeof(double) * (kSsWT * EPT + kSsWT * EPT / 32); }
constexpr size_t ss_chain_smem() { return sizeof(ChainSmem); }

// ---- term generators ----------------------------------------------------------
// row index j = k / nx without an integer division: fp64 estimate + exact fix-up
__device__ __forceinline__ int row_of(long long k, int nx, double inv_nx) {
    int j = (int)((double)k * inv_nx);
    const long long r = k - (long long)j * nx;
    j += (r >= nx) - (r < 0);
    return j;
}

// Each generator also loads a chunk's terms for one thread of the walk:
// `striped(s, k0, clen, v)` fills v[m] = term k0 + m*kSsWT (0 past the chunk),
// where k0 = chunk base + threadIdx.x and clen = terms in the chunk.
#define GMG_SS_STRIPED_DEFAULT                                                              \
    template <int EPT, int WT>                                                               \
    __device__ __forceinline__ void striped(int s, long long k0, int clen, double (&v)[EPT]) const { \
        _Pragma("unroll") for (int m = 0; m < EPT; ++m) {                                   \
            const int kl = m * WT + (int)threadIdx.x;                                         \
            v[m] = kl < clen ? term(s, k0 + m * WT) : 0.0;                                    \
        }                                                                                    \
    }

struct NormTerms {  // r_k * r_k (norm_l2, stencil.cpp:9-13) on a pitched grid function
    static constexpr int NS = 1;
    static constexpr const char* kProfName = "ss_walk(norm)";
    static constexpr double kBytesPerTerm = 8.0;  // algorithmic bytes read per term (all sums)
    const double* r;
    Grid g;
    double inv_nx;
    __device__ __forceinline__ double term(int, long long k) const {
        const int j = row_of(k, g.nx, inv_nx), i = (int)(k - (long long)j * g.nx);
        const double v = __ldg(r + g.at(i, j));
        return v * v;
    }
    // row/column of the first term once, then stepped by kSsWT (no per-term division)
    template <int EPT, int WT>
    __device__ __forceinline__ void striped(int, long long k0, int clen, double (&v)[EPT]) const {
        int j = row_of(k0, g.nx, inv_nx), i = (int)(k0 - (long long)j * g.nx);
#pragma unroll
        for (int m = 0; m < EPT; ++m) {
            const int kl = m * WT + (int)threadIdx.x;
            double x = 0.0;
            if (kl < clen) x = __ldg(r + g.at(i, j));
            v[m] = x * x;
            i += WT;
            while (i >= g.nx) {
                i -= g.nx;
                ++j;
            }
        }
    }
};

struct DotTerms {  // a_k * b_k (dot, stencil.cpp:21-26) on flat arrays
    static constexpr int NS = 1;
    static constexpr const char* kProfName = "ss_walk(dot)";
    static constexpr double kBytesPerTerm = 16.0;  // algorithmic bytes read per term (all sums)
    const double *a, *b;
    __device__ __forceinline__ double term(int, long long k) const { return __ldg(a + k) * __ldg(b + k); }
    GMG_SS_STRIPED_DEFAULT
};

struct FlatNormTerms {  // v_k * v_k on a flat array
    static constexpr int NS = 1;
    static constexpr const char* kProfName = "ss_walk(norm)";
    static constexpr double kBytesPerTerm = 8.0;  // algorithmic bytes read per term (all sums)
    const double* a;
    __device__ __forceinline__ double term(int, long long k) const {
        const double v = __ldg(a + k);
        return v * v;
    }
    GMG_SS_STRIPED_DEFAULT
};

struct ArrTerms {  // materialised terms: sum s reads t[s][k]
    static constexpr int NS = 2;
    static constexpr const char* kProfName = "ss_walk(omega dots)";
    static constexpr double kBytesPerTerm = 16.0;  // algorithmic bytes read per term (all sums)
    const double* t0;
    const double* t1;
    __device__ __forceinline__ double term(int s, long long k) const { return __ldg((s ? t1 : t0) + k); }
    GMG_SS_STRIPED_DEFAULT
};

}  // namespace gmg_dev
