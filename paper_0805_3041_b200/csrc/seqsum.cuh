// Exact-order (bit-identical to a left-to-right loop) fp64 summation on the GPU.
// Algorithm and invariants: seqsum_core.h. Two launches per sum (+1 memset):
//
//   k_ss_walk  : one CTA per chunk of C = 8192 terms (chunks taken from an
//                atomic ticket, so every predecessor is already running).
//                (1) loads its terms, (2) publishes its approximate sum and
//                obtains the approximate prefix of all earlier chunks by
//                decoupled look-back — the speculated running sum at its start,
//                (3) each thread walks its 32 consecutive terms from the
//                speculated state, splitting them into in-binade integer
//                segments and break elements, (4) a block-wide segmented scan
//                merges segments across threads -> (#breaks + 1) records,
//                (5) a second look-back over record counts gives the chunk's
//                offset in one compact, chunk-ordered record array.
//   k_ss_chain : one CTA per sum replays the records in order from the exact
//                state 0.0 — validate+apply each segment (integer add), real
//                IEEE add for each break element — while the other warps
//                stream the next batch of records into shared memory. A
//                segment that fails validation (a wrong speculation) makes the
//                chain re-sum the rest of that chunk with literal adds.
//
// Term generators: `double term(int s, long long k)` returns term k (in the
// reference's k = j*nx + i order) of sum s.
#pragma once

#include "common.cuh"
#include "seqsum_core.h"

namespace gmg_dev {

constexpr int kSsT = 256;             // threads per chunk
constexpr int kSsEPT = 32;            // terms per thread
constexpr int kSsC = kSsT * kSsEPT;   // terms per chunk
constexpr int kSsBatch = 1024;        // records staged per chain batch
constexpr int kSsMaxSums = 2;
constexpr int kSsRMax = 512;         // records a chunk may store; more -> literal re-sum

// Per-sum look-back state (zeroed before each k_ss_walk: flags, counters).
struct SsState {
    int* flag;       // [nch] 0 none, 1 aggregate published, 2 inclusive published
    int* cflag;      // [nch] record-count look-back flags
    int* ticket;     // [1]
    int* total;      // [1] total records stored
    double* agg;     // [nch]
    double* incl;    // [nch]
    int* cagg;       // [nch]
    int* cincl;      // [nch]
    gmg_ss::Rec* recs;
    int cap;         // record capacity
};
struct SsPair {
    SsState s[kSsMaxSums];
};

__device__ __forceinline__ int ld_flag(const int* p) { return *reinterpret_cast<const volatile int*>(p); }
__device__ __forceinline__ void st_flag(int* p, int v) {
    __threadfence();
    *reinterpret_cast<volatile int*>(p) = v;
}

// Exclusive prefix for chunk c by decoupled look-back (one warp). T is double
// (approximate running sums) or int (record counts).
template <class T>
__device__ T lookback(int c, const int* flag, const T* agg, const T* incl) {
    const int lane = threadIdx.x & 31;
    T acc = T(0);
    int p = c - 1;
    while (p >= 0) {
        const int idx = p - lane;
        int f = 2;
        if (idx >= 0) {
            do {
                f = ld_flag(flag + idx);
            } while (f == 0);
        }
        __threadfence();
        const unsigned m2 = __ballot_sync(0xffffffffu, f == 2);
        const int stop = m2 ? __ffs(m2) - 1 : 32;  // nearest predecessor with an inclusive prefix
        T v = T(0);
        if (idx >= 0) {
            if (lane < stop) v = __ldcg(agg + idx);
            else if (lane == stop) v = __ldcg(incl + idx);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        acc += v;
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

__device__ __forceinline__ double block_excl_sum_d(double x, double* sw /* [8] */) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    double base = 0.0;
    for (int q = 0; q < w; ++q) base += sw[q];
    __syncthreads();
    return base + inc - x;
}

__device__ __forceinline__ int block_excl_sum_i(int x, int* sw /* [8] */, int* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    int base = 0, tot = 0;
    for (int q = 0; q < 8; ++q) {
        if (q < w) base += sw[q];
        tot += sw[q];
    }
    __syncthreads();
    *total = tot;
    return base + inc - x;
}

// segmented scan element: f = "a break closed the run inside this thread"
struct SegF {
    gmg_ss::Seg g;
    int f;
};
__device__ __forceinline__ SegF segf_combine(const SegF& a, const SegF& b) {
    SegF r;
    r.f = a.f | b.f;
    r.g = b.f ? b.g : gmg_ss::seg_merge(a.g, b.g);
    return r;
}
__device__ __forceinline__ SegF segf_shfl_up(const SegF& x, int o) {
    SegF r;
    const uint32_t meta = static_cast<uint32_t>(x.g.E) | (static_cast<uint32_t>(x.g.neg) << 11) |
                          (static_cast<uint32_t>(x.g.bad) << 12) | (static_cast<uint32_t>(x.f) << 13) |
                          (static_cast<uint32_t>(x.g.len) << 14);
    const uint32_t m2 = __shfl_up_sync(0xffffffffu, meta, o);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        r.g.Q[p] = __shfl_up_sync(0xffffffffu, x.g.Q[p], o);
        r.g.mn[p] = __shfl_up_sync(0xffffffffu, x.g.mn[p], o);
        r.g.mx[p] = __shfl_up_sync(0xffffffffu, x.g.mx[p], o);
    }
    r.g.E = m2 & 0x7ff;
    r.g.neg = (m2 >> 11) & 1;
    r.g.bad = (m2 >> 12) & 1;
    r.f = (m2 >> 13) & 1;
    r.g.len = static_cast<int>(m2 >> 14);
    return r;
}

// Block exclusive segmented scan; also returns the block inclusive total.
__device__ __forceinline__ SegF block_excl_segscan(const SegF& x, SegF* sw /* [8] */, SegF* total) {
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    SegF inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const SegF y = segf_shfl_up(inc, o);
        if (lane >= o) inc = segf_combine(y, inc);
    }
    const SegF ex = segf_shfl_up(inc, 1);
    if (lane == 31) sw[w] = inc;
    __syncthreads();
    SegF base;
    base.g = gmg_ss::seg_empty();
    base.f = 0;
    SegF tot = base;
    for (int q = 0; q < 8; ++q) {
        if (q < w) base = segf_combine(base, sw[q]);
        tot = segf_combine(tot, sw[q]);
    }
    __syncthreads();
    *total = tot;
    if (lane == 0) return base;
    return segf_combine(base, ex);
}

__device__ __forceinline__ int ss_pad(int e) { return e + (e >> 5); }

// ---- walk ---------------------------------------------------------------------
// grid (nch, NS); block kSsT; dynamic smem (kSsC + kSsC/32) doubles.
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_walk(TG tg, long long n, int nch, SsPair sts) {
    extern __shared__ double tm[];
    __shared__ double swd[8];
    __shared__ int swi[8];
    __shared__ SegF sws[8];
    __shared__ int s_chunk;
    __shared__ double s_pre;
    __shared__ int s_off;

    const int s = blockIdx.y;
    const SsState& S = sts.s[s];
    const int t = threadIdx.x;
    if (t == 0) s_chunk = atomicAdd(S.ticket, 1);
    __syncthreads();
    const int c = s_chunk;
    const long long base = (long long)c * kSsC;
    const int clen = (int)min((long long)kSsC, n - base);

    // (1) terms: striped (coalesced) loads into shared memory
#pragma unroll 8
    for (int m = 0; m < kSsEPT; ++m) {
        const int kl = m * kSsT + t;
        tm[ss_pad(kl)] = kl < clen ? tg.term(s, base + kl) : 0.0;
    }
    __syncthreads();
    const int e0 = t * kSsEPT;
    const int ne = max(0, min(kSsEPT, clen - e0));
    double ts = 0.0;
    for (int m = 0; m < ne; ++m) ts += tm[ss_pad(e0 + m)];

    // (2) approximate prefix by look-back
    const double tot_approx = block_sum_d(ts, swd);
    if (t == 0) {
        if (c == 0) {
            S.incl[0] = tot_approx;
            st_flag(S.flag, 2);
        } else {
            S.agg[c] = tot_approx;
            st_flag(S.flag + c, 1);
        }
    }
    if (t < 32) {
        const double pre = c == 0 ? 0.0 : lookback<double>(c, S.flag, S.agg, S.incl);
        if (t == 0) {
            s_pre = pre;
            if (c > 0) {
                S.incl[c] = pre + tot_approx;
                st_flag(S.flag + c, 2);
            }
        }
    }
    __syncthreads();
    const double pred = s_pre + block_excl_sum_d(ts, swd);

    // (3) thread walk, pass 1: leading segment, trailing segment, break count
    gmg_ss::State st = gmg_ss::make_state(pred);
    gmg_ss::Seg cur = gmg_ss::seg_empty(), lead = gmg_ss::seg_empty();
    int r = 0;
    double pb0 = 0.0;
    for (int m = 0; m < ne; ++m) {
        const double p = tm[ss_pad(e0 + m)];
        if (!gmg_ss::walk_try(st, cur, p)) {
            if (r == 0) {
                lead = cur;
                pb0 = p;
            }
            ++r;
            cur = gmg_ss::seg_empty();
            gmg_ss::real_add(st, p);
        }
    }
    if (r == 0) lead = cur;

    // (4) merge runs across threads
    SegF x;
    x.f = r > 0;
    x.g = r > 0 ? cur : lead;
    SegF tot;
    const SegF carry = block_excl_segscan(x, sws, &tot);
    int R;
    const int pos = block_excl_sum_i(r, swi, &R);
    R += 1;

    // (5) record offset by look-back over stored counts (aggregate published
    //     before looking back, so chunks never wait on a predecessor's look-back)
    const int stored = R <= kSsRMax ? R : 1;
    if (t == 0) {
        if (c == 0) {
            S.cincl[0] = stored;
            st_flag(S.cflag, 2);
        } else {
            S.cagg[c] = stored;
            st_flag(S.cflag + c, 1);
        }
    }
    if (t < 32) {
        const int o = c == 0 ? 0 : lookback<int>(c, S.cflag, S.cagg, S.cincl);
        if (t == 0) {
            if (c > 0) {
                S.cincl[c] = o + stored;
                st_flag(S.cflag + c, 2);
            }
            if (c == nch - 1) *S.total = o + stored;
            s_off = o;
        }
    }
    __syncthreads();
    const int off = s_off;
    if (stored != R) {  // too many breaks: the chain sums this chunk literally
        if (t == 0) S.recs[off] = gmg_ss::rec_literal(c);
        return;
    }
    gmg_ss::Rec* out = S.recs + off;
    if (r > 0) {
        // pass 2: emit records; the first one absorbs the run carried in
        out[pos] = gmg_ss::rec_make(gmg_ss::seg_merge(carry.g, lead), true, pb0, c);
        st = gmg_ss::make_state(pred);
        cur = gmg_ss::seg_empty();
        int k = 0;
        for (int m = 0; m < ne; ++m) {
            const double p = tm[ss_pad(e0 + m)];
            if (!gmg_ss::walk_try(st, cur, p)) {
                if (k > 0) out[pos + k] = gmg_ss::rec_make(cur, true, p, c);
                ++k;
                cur = gmg_ss::seg_empty();
                gmg_ss::real_add(st, p);
            }
        }
    }
    if (t == kSsT - 1) out[R - 1] = gmg_ss::rec_make(tot.g, false, 0.0, c);
}

// ---- chain --------------------------------------------------------------------
__device__ __forceinline__ gmg_ss::Seg seg_shfl(const gmg_ss::Seg& x, int src) {
    gmg_ss::Seg r;
    const uint32_t meta = static_cast<uint32_t>(x.E) | (static_cast<uint32_t>(x.neg) << 11) |
                          (static_cast<uint32_t>(x.bad) << 12) | (static_cast<uint32_t>(x.len) << 13);
    const uint32_t m2 = __shfl_sync(0xffffffffu, meta, src);
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        r.Q[p] = __shfl_sync(0xffffffffu, x.Q[p], src);
        r.mn[p] = __shfl_sync(0xffffffffu, x.mn[p], src);
        r.mx[p] = __shfl_sync(0xffffffffu, x.mx[p], src);
    }
    r.E = m2 & 0x7ff;
    r.neg = (m2 >> 11) & 1;
    r.bad = (m2 >> 12) & 1;
    r.len = static_cast<int>(m2 >> 13);
    return r;
}

// Literal left-to-right adds over terms [k0, k1) of sum s.
template <class TG>
__device__ double literal_sum(const TG& tg, int s, double a, long long k0, long long k1) {
    for (long long k = k0; k < k1; ++k) a = a + tg.term(s, k);
    return a;
}

// grid (NS); block kSsT; dynamic smem 2 * kSsBatch records. Warp 0 replays the
// records: in each window of 32 it merges the pure segments up to the first
// break record with a parity-aware merge-scan, validates the merged run once
// against the exact state and applies it, then performs that record's break
// add. Warps 1.. stream the next batch into shared memory meanwhile.
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_chain(TG tg, long long n, SsPair sts, double* __restrict__ out) {
    extern __shared__ unsigned char smraw[];
    gmg_ss::Rec* buf = reinterpret_cast<gmg_ss::Rec*>(smraw);
    const int s = blockIdx.x;
    const SsState& S = sts.s[s];
    const int t = threadIdx.x, lane = t & 31;
    const int total = *S.total;
    const int nb = (total + kSsBatch - 1) / kSsBatch;

    for (int q = t; q < min(total, kSsBatch); q += kSsT) buf[q] = S.recs[q];
    __syncthreads();

    gmg_ss::State st = gmg_ss::make_state(0.0);  // identical in every lane of warp 0
    long long cur_chunk = -1, skip = -1;
    int pos = 0;
    for (int b = 0; b < nb; ++b) {
        const gmg_ss::Rec* A = buf + (b & 1) * kSsBatch;
        const int cnt = min(kSsBatch, total - b * kSsBatch);
        if (t < 32) {
            int q = 0;
            while (q < cnt) {
                const int idx = q + lane;
                const bool have = idx < cnt;
                gmg_ss::Rec rec{};
                if (have) rec = A[idx];
                const long long c = have ? (long long)rec.chunk : -2;
                const bool lit = have && gmg_ss::rec_literal_flag(rec);
                const bool skipme = have && c == skip;
                const bool brk = have && !lit && !skipme && gmg_ss::rec_has_break(rec);
                const unsigned stopm = __ballot_sync(0xffffffffu, !have || brk || lit || skipme);
                const int f = stopm ? __ffs(stopm) - 1 : 32;  // lanes < f: pure segments
                // Runs of >= 3 pure segments are merged with a warp merge-scan; break
                // records (and short runs) take the cheap serial path below.
                if (f >= 3) {
                    const int run_end = f - 1;
                    gmg_ss::Seg g = (lane <= run_end) ? gmg_ss::rec_seg(rec) : gmg_ss::seg_empty();
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        const gmg_ss::Seg y = seg_shfl(g, lane >= o ? lane - o : lane);
                        if (lane >= o) g = gmg_ss::seg_merge(y, g);
                    }
                    const gmg_ss::Seg run = seg_shfl(g, run_end);
                    if (gmg_ss::seg_valid(run, st)) {
                        const long long c_end = __shfl_sync(0xffffffffu, c, run_end);
                        int my = (lane <= run_end && c == c_end) ? (int)(rec.meta >> 15) : 0;
#pragma unroll
                        for (int o = 16; o > 0; o >>= 1) my += __shfl_xor_sync(0xffffffffu, my, o);
                        pos = (c_end == cur_chunk ? pos : 0) + my;
                        cur_chunk = c_end;
                        gmg_ss::seg_apply(run, st);
                        q += run_end + 1;
                        continue;
                    }
                }
                // serial handling of the window's first record
                const gmg_ss::Rec r0 = A[q];
                const long long c0 = r0.chunk;
                ++q;
                if (c0 == skip) continue;
                if (c0 != cur_chunk) {
                    cur_chunk = c0;
                    pos = 0;
                }
                const gmg_ss::Seg g0 = gmg_ss::rec_seg(r0);
                if (gmg_ss::rec_literal_flag(r0) || !gmg_ss::seg_valid(g0, st)) {
                    double a = 0.0;
                    if (lane == 0) a = literal_sum(tg, s, st.s, c0 * kSsC + pos, min(n, (c0 + 1) * kSsC));
                    a = __shfl_sync(0xffffffffu, a, 0);
                    st = gmg_ss::make_state(a);
                    skip = c0;
                    continue;
                }
                gmg_ss::seg_apply(g0, st);
                pos += g0.len;
                if (gmg_ss::rec_has_break(r0)) {
                    gmg_ss::real_add(st, r0.pb);
                    pos += 1;
                }
            }
        } else if (b + 1 < nb) {
            gmg_ss::Rec* B = buf + ((b + 1) & 1) * kSsBatch;
            const int cn = min(kSsBatch, total - (b + 1) * kSsBatch);
            const gmg_ss::Rec* src = S.recs + (long long)(b + 1) * kSsBatch;
            for (int q = t - 32; q < cn; q += kSsT - 32) B[q] = src[q];
        }
        __syncthreads();
    }
    if (t == 0) out[s] = st.s;
}

// Fast mode: tree-order partial sums per chunk, then one CTA finishes.
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_partial(TG tg, long long n, double* __restrict__ csum, int nch) {
    __shared__ double swd[8];
    const int s = blockIdx.y;
    const long long base = (long long)blockIdx.x * kSsC;
    double acc = 0.0;
#pragma unroll 4
    for (int m = 0; m < kSsEPT; ++m) {
        const long long k = base + m * kSsT + threadIdx.x;
        if (k < n) acc += tg.term(s, k);
    }
    acc = block_sum_d(acc, swd);
    if (threadIdx.x == 0) csum[(long long)s * nch + blockIdx.x] = acc;
}

constexpr size_t ss_walk_smem() { return sizeof(double) * (kSsC + kSsC / 32); }
constexpr size_t ss_chain_smem() { return sizeof(gmg_ss::Rec) * 2 * kSsBatch; }

// ---- term generators ----------------------------------------------------------
// row index j = k / nx without an integer division: fp64 estimate + exact fix-up
__device__ __forceinline__ int row_of(long long k, int nx, double inv_nx) {
    int j = (int)((double)k * inv_nx);
    const long long r = k - (long long)j * nx;
    j += (r >= nx) - (r < 0);
    return j;
}

struct NormTerms {  // r_k * r_k (norm_l2, stencil.cpp:9-13) on a pitched grid function
    static constexpr int NS = 1;
    const double* r;
    Grid g;
    double inv_nx;
    __device__ __forceinline__ double term(int, long long k) const {
        const int j = row_of(k, g.nx, inv_nx), i = (int)(k - (long long)j * g.nx);
        const double v = __ldg(r + g.at(i, j));
        return v * v;
    }
};

struct DotTerms {  // a_k * b_k (dot, stencil.cpp:21-26) on flat arrays
    static constexpr int NS = 1;
    const double *a, *b;
    __device__ __forceinline__ double term(int, long long k) const { return __ldg(a + k) * __ldg(b + k); }
};

struct FlatNormTerms {  // v_k * v_k on a flat array
    static constexpr int NS = 1;
    const double* a;
    __device__ __forceinline__ double term(int, long long k) const {
        const double v = __ldg(a + k);
        return v * v;
    }
};

struct ArrTerms {  // materialised terms: sum s reads t[s][k]
    static constexpr int NS = 2;
    const double* t0;
    const double* t1;
    __device__ __forceinline__ double term(int s, long long k) const { return __ldg((s ? t1 : t0) + k); }
};

}  // namespace gmg_dev
