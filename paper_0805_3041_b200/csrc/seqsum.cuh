// Exact-order (bit-identical to a left-to-right loop) fp64 summation on the GPU.
// Algorithm and invariants: seqsum_core.h. Four launches per call:
//
//   S1 k_ss_partial : per chunk of C = 8192 terms, an approximate (tree) sum.
//   S2 k_ss_scan    : one CTA, approximate exclusive prefix over the chunks
//                     -> a speculated running sum at every chunk start.
//   S3 k_ss_walk    : per chunk, each thread walks its 32 consecutive terms from
//                     the speculated state (chunk prefix + in-chunk thread
//                     prefix), splitting them into in-binade integer segments
//                     and break elements; a block-wide segmented scan merges
//                     segments across threads, so a chunk yields
//                     (#breaks + 1) records.
//   S4 k_ss_chain   : one CTA per sum replays all records in order from the
//                     exact state 0.0: validate+apply each segment (integer
//                     add), real IEEE add for each break element. A segment
//                     that fails validation (speculation wrong) or a chunk
//                     with too many records falls back to literal sequential
//                     adds over that chunk's terms.
//
// Terms are produced by a generator TG (element k in the reference's k order)
// in S1, S3 and (rarely) S4, so the inputs are streamed from HBM twice; no
// term array is materialised.
#pragma once

#include "common.cuh"
#include "seqsum_core.h"

namespace gmg_dev {

constexpr int kSsT = 256;             // threads per chunk
constexpr int kSsEPT = 32;            // terms per thread
constexpr int kSsC = kSsT * kSsEPT;   // terms per chunk
constexpr int kSsRMax = 256;          // records stored per chunk
constexpr int kSsCap = 2048;          // records staged per chain batch
constexpr int kSsFT = 2048;           // fallback tile

// ---- block reductions / scans (256 threads) --------------------------------
template <int NS>
__device__ __forceinline__ void block_sum(double (&v)[NS], double* red /* [NS][8] */) {
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        double x = v[s];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
        if ((threadIdx.x & 31) == 0) red[s * 8 + (threadIdx.x >> 5)] = x;
    }
    __syncthreads();
#pragma unroll
    for (int s = 0; s < NS; ++s) {
        double x = 0.0;
        for (int w = 0; w < 8; ++w) x += red[s * 8 + w];
        v[s] = x;
    }
    __syncthreads();
}

// exclusive prefix sum of a double over the block (approximate order)
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
    for (int q = 0; q < (int)(blockDim.x >> 5); ++q) {
        if (q < w) base += sw[q];
        tot += sw[q];
    }
    __syncthreads();
    *total = tot;
    return base + inc - x;
}

// segmented scan element: flag = "a break closed the run before this thread"
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
                          (static_cast<uint32_t>(x.g.bad) << 12) | (static_cast<uint32_t>(x.f) << 13);
    const uint32_t m2 = __shfl_up_sync(0xffffffffu, meta, o);
    r.g.len = __shfl_up_sync(0xffffffffu, x.g.len, o);
    r.g.Q = __shfl_up_sync(0xffffffffu, x.g.Q, o);
    r.g.mn = __shfl_up_sync(0xffffffffu, x.g.mn, o);
    r.g.mx = __shfl_up_sync(0xffffffffu, x.g.mx, o);
    r.g.E = m2 & 0x7ff;
    r.g.neg = (m2 >> 11) & 1;
    r.g.bad = (m2 >> 12) & 1;
    r.f = (m2 >> 13) & 1;
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
    SegF ex = segf_shfl_up(inc, 1);
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

// ---- S1 --------------------------------------------------------------------
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_partial(TG tg, long long n, double* __restrict__ csum,
                                                     int nch, int* __restrict__ nzflag) {
    constexpr int NS = TG::NS;
    __shared__ double red[NS * 8];
    const long long base = (long long)blockIdx.x * kSsC;
    double acc[NS];
#pragma unroll
    for (int s = 0; s < NS; ++s) acc[s] = 0.0;
    int nz = 0;
#pragma unroll 4
    for (int m = 0; m < kSsEPT; ++m) {
        const long long k = base + m * kSsT + threadIdx.x;
        if (k < n) {
            double p[NS];
            int z = 0;
            tg.get(k, p, z);
#pragma unroll
            for (int s = 0; s < NS; ++s) acc[s] += p[s];
            nz |= z;
        }
    }
    const int anynz = __syncthreads_or(nz);
    block_sum<NS>(acc, red);
    if (threadIdx.x == 0) {
#pragma unroll
        for (int s = 0; s < NS; ++s) csum[(long long)s * nch + blockIdx.x] = acc[s];
        if (nzflag && anynz) atomicOr(nzflag, 1);
    }
}

// ---- S2 --------------------------------------------------------------------
template <int NS>
__global__ void __launch_bounds__(1024) k_ss_scan(const double* __restrict__ csum,
                                                  double* __restrict__ cpred, int nch) {
    __shared__ double sw[32];
    const int T = blockDim.x;
    const int per = (nch + T - 1) / T;
    const int c0 = threadIdx.x * per;
    const int c1 = min(c0 + per, nch);
    for (int s = 0; s < NS; ++s) {
        const double* cs = csum + (long long)s * nch;
        double loc = 0.0;
        for (int c = c0; c < c1; ++c) loc += cs[c];
        // block exclusive scan over 1024 threads
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        double inc = loc;
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
        double run = base + inc - loc;
        for (int c = c0; c < c1; ++c) {
            cpred[(long long)s * nch + c] = run;
            run += cs[c];
        }
    }
}

// ---- S3 --------------------------------------------------------------------
__device__ __forceinline__ int ss_pad(int e) { return e + (e >> 5); }

template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_walk(TG tg, long long n, const double* __restrict__ cpred,
                                                  int nch, int* __restrict__ counts,
                                                  gmg_ss::Rec* __restrict__ recs) {
    constexpr int NS = TG::NS;
    extern __shared__ double tm[];  // [NS][kSsC + kSsC/32]
    __shared__ double swd[8];
    __shared__ int swi[8];
    __shared__ SegF sws[8];
    constexpr int STRIDE = kSsC + kSsC / 32;

    const int c = blockIdx.x;
    const long long base = (long long)c * kSsC;
    const int clen = (int)min((long long)kSsC, n - base);
    const int t = threadIdx.x;

#pragma unroll 4
    for (int m = 0; m < kSsEPT; ++m) {
        const int kl = m * kSsT + t;
        double p[NS];
        int z = 0;
        if (kl < clen) {
            tg.get(base + kl, p, z);
        } else {
#pragma unroll
            for (int s = 0; s < NS; ++s) p[s] = 0.0;
        }
#pragma unroll
        for (int s = 0; s < NS; ++s) tm[s * STRIDE + ss_pad(kl)] = p[s];
    }
    __syncthreads();

    const int e0 = t * kSsEPT;
    const int ne = max(0, min(kSsEPT, clen - e0));

    for (int s = 0; s < NS; ++s) {
        const double* P = tm + s * STRIDE;
        double ts = 0.0;
        for (int m = 0; m < ne; ++m) ts += P[ss_pad(e0 + m)];
        const double pred = cpred[(long long)s * nch + c] + block_excl_sum_d(ts, swd);

        // pass 1: leading segment, trailing segment, break count
        gmg_ss::State st = gmg_ss::make_state(pred);
        gmg_ss::Seg cur = gmg_ss::seg_empty(), lead = gmg_ss::seg_empty();
        int r = 0;
        double pb0 = 0.0;
        for (int m = 0; m < ne; ++m) {
            const double p = P[ss_pad(e0 + m)];
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
        SegF x;
        x.f = r > 0;
        x.g = r > 0 ? cur : lead;
        SegF tot;
        const SegF carry = block_excl_segscan(x, sws, &tot);
        int R;
        const int pos = block_excl_sum_i(r, swi, &R);
        R += 1;
        int* cnt = counts + (long long)s * nch + c;
        gmg_ss::Rec* out = recs + ((long long)s * nch + c) * kSsRMax;
        if (R > kSsRMax) {
            if (t == 0) *cnt = -1;
            continue;
        }
        if (r > 0) {
            // pass 2: emit records; first one absorbs the run carried in
            out[pos] = gmg_ss::rec_make(gmg_ss::seg_merge(carry.g, lead), true, pb0);
            st = gmg_ss::make_state(pred);
            cur = gmg_ss::seg_empty();
            int k = 0;
            for (int m = 0; m < ne; ++m) {
                const double p = P[ss_pad(e0 + m)];
                if (!gmg_ss::walk_try(st, cur, p)) {
                    if (k > 0) out[pos + k] = gmg_ss::rec_make(cur, true, p);
                    ++k;
                    cur = gmg_ss::seg_empty();
                    gmg_ss::real_add(st, p);
                }
            }
        }
        if (t == kSsT - 1) {
            out[R - 1] = gmg_ss::rec_make(tot.g, false, 0.0);
            *cnt = R;
        }
    }
}

// ---- S4 --------------------------------------------------------------------
template <class TG>
__global__ void __launch_bounds__(kSsT) k_ss_chain(TG tg, long long n, int nch,
                                                   const int* __restrict__ counts,
                                                   const gmg_ss::Rec* __restrict__ recs,
                                                   double* __restrict__ out) {
    constexpr int NS = TG::NS;
    extern __shared__ unsigned char smraw[];
    gmg_ss::Rec* rb = reinterpret_cast<gmg_ss::Rec*>(smraw);                     // [kSsCap]
    double* ft = reinterpret_cast<double*>(smraw + sizeof(gmg_ss::Rec) * kSsCap);  // [kSsFT]
    __shared__ int off[kSsT + 1];
    __shared__ int cn[kSsT];
    __shared__ int swi[8];
    __shared__ int s_be, s_fb_chunk, s_fb_pos;
    __shared__ double s_state;

    const int s = blockIdx.x;
    const int t = threadIdx.x;
    const int* cnts = counts + (long long)s * nch;
    gmg_ss::State st = gmg_ss::make_state(0.0);  // thread 0's running state

    int c0 = 0;
    while (c0 < nch) {
        const int cc = c0 + t;
        const int craw = cc < nch ? cnts[cc] : 0;
        const int nrec = craw > 0 ? craw : 0;
        int total;
        const int o = block_excl_sum_i(nrec, swi, &total);
        off[t] = o;
        cn[t] = craw;
        if (t == 0) off[kSsT] = total;
        __syncthreads();
        // batch = longest prefix of chunks whose records fit the staging buffer
        if (t == 0) {
            int be = 0;
            while (be < kSsT && c0 + be < nch && off[be + 1] <= kSsCap) ++be;
            if (be == 0) be = 1;  // a single chunk always fits (kSsRMax <= kSsCap)
            s_be = be;
        }
        __syncthreads();
        const int be = s_be;
        const int nstage = off[be];
        for (int q = t; q < nstage; q += kSsT) {
            int lo = 0, hi = be - 1;  // find chunk owning staged record q
            while (lo < hi) {
                const int mid = (lo + hi + 1) >> 1;
                if (off[mid] <= q) lo = mid; else hi = mid - 1;
            }
            rb[q] = recs[((long long)s * nch + c0 + lo) * kSsRMax + (q - off[lo])];
        }
        __syncthreads();
        if (t == 0) {
            int fb_chunk = -1, fb_pos = 0;
            for (int b = 0; b < be && fb_chunk < 0; ++b) {
                if (cn[b] < 0) {
                    fb_chunk = b;
                    fb_pos = 0;
                    break;
                }
                int pos = 0;
                for (int r = 0; r < cn[b]; ++r) {
                    const gmg_ss::Rec& rec = rb[off[b] + r];
                    const gmg_ss::Seg g = gmg_ss::rec_seg(rec);
                    if (!gmg_ss::seg_valid(g, st)) {
                        fb_chunk = b;
                        fb_pos = pos;
                        break;
                    }
                    gmg_ss::seg_apply(g, st);
                    pos += g.len;
                    if (gmg_ss::rec_has_break(rec)) {
                        gmg_ss::real_add(st, rec.pb);
                        pos += 1;
                    }
                }
            }
            s_fb_chunk = fb_chunk;
            s_fb_pos = fb_pos;
            s_state = st.s;
        }
        __syncthreads();
        const int fbc = s_fb_chunk;
        if (fbc < 0) {
            c0 += be;
            continue;
        }
        // literal sequential adds over the rest of chunk c0+fbc
        const long long cbase = (long long)(c0 + fbc) * kSsC;
        const int clen = (int)min((long long)kSsC, n - cbase);
        for (int e = s_fb_pos; e < clen; e += kSsFT) {
            const int len = min(kSsFT, clen - e);
            for (int q = t; q < len; q += kSsT) {
                double p[NS];
                int z = 0;
                tg.get(cbase + e + q, p, z);
                ft[q] = p[s];
            }
            __syncthreads();
            if (t == 0) {
                double a = s_state;
                for (int q = 0; q < len; ++q) a = a + ft[q];
                s_state = a;
            }
            __syncthreads();
        }
        if (t == 0) st = gmg_ss::make_state(s_state);
        c0 += fbc + 1;
        __syncthreads();
    }
    if (t == 0) out[s] = st.s;
}

constexpr size_t ss_walk_smem(int ns) { return sizeof(double) * ns * (kSsC + kSsC / 32); }
constexpr size_t ss_chain_smem() { return sizeof(gmg_ss::Rec) * kSsCap + sizeof(double) * kSsFT; }

// ---- term generators -------------------------------------------------------
struct NormTerms {  // r_k * r_k (norm_l2, stencil.cpp:9-13)
    static constexpr int NS = 1;
    const double* r;
    Grid g;
    __device__ __forceinline__ void get(long long k, double (&p)[1], int& nz) const {
        const int j = (int)(k / g.nx), i = (int)(k - (long long)j * g.nx);
        const double v = __ldg(r + g.at(i, j));
        p[0] = v * v;
        nz = 0;
    }
};

struct DotTerms {  // a_k * b_k (dot, stencil.cpp:21-26)
    static constexpr int NS = 1;
    const double *a, *b;
    Grid g;
    __device__ __forceinline__ void get(long long k, double (&p)[1], int& nz) const {
        const int j = (int)(k / g.nx), i = (int)(k - (long long)j * g.nx);
        const long long o = g.at(i, j);
        p[0] = __ldg(a + o) * __ldg(b + o);
        nz = 0;
    }
};

// adaptive_omega (cycle.cpp:40-51) on corr = P uc computed on the fly:
// p[0] = (A corr)_k * corr_k, p[1] = d_k * corr_k, nz |= corr_k*corr_k != 0.
template <class Coef>
struct OmegaTerms {
    static constexpr int NS = 2;
    const double* d;
    Grid g;
    Coef A;
    Prolong P;
    __device__ __forceinline__ double corr(int i, int j) const {
        return g.inside(i, j) ? P.at(i, j) : 0.0;
    }
    __device__ __forceinline__ void get(long long k, double (&p)[2], int& nz) const {
        const int j = (int)(k / g.nx), i = (int)(k - (long long)j * g.nx);
        const double cc = corr(i, j);
        const double ac = stencil_apply(A, i, j, cc, corr(i - 1, j), corr(i + 1, j), corr(i, j - 1),
                                        corr(i, j + 1));
        p[0] = ac * cc;
        p[1] = __ldg(d + g.at(i, j)) * cc;
        nz = (cc * cc) != 0.0;
    }
};

}  // namespace gmg_dev
