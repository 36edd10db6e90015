// Exact emulation of the reference's left-to-right fp64 summation
//   double s = 0.0; for (k) s += p[k];      (stencil.cpp:9-13,21-26; cycle.cpp:44)
// split into parallel pieces. Shared by the CUDA kernels (seqsum.cuh) and the
// host emulation used by the CPU tests (host_setup.cpp).
//
// Idea: while the running sum s stays inside one binade
// [2^(e-1), 2^e) its representable neighbours are the multiples of
// u = ulp(s) = 2^(e-53), so fl(s + p) = s + u*RN(p/u) — the sum is an exact
// integer prefix sum M_k = s/u + sum q_j with q_j = RN(p_j/u) (an exact
// half-integer p/u rounds to the even total; see Seg). Only two situations need
// a real IEEE add ("break"): the state is zero/subnormal/huge or |p/u| >= 2^52,
// or the integer state would leave the open binade (|M| outside
// [2^52+1, 2^53-1]; the +1 keeps a result that lands just below 2^(e-1), where
// the spacing halves, out of the integer model).
//
// A *segment* is a run of elements summed in one binade; it is described by
// (E, sign, Q, minP, maxP) (two variants, see Seg): Q is the integer total in
// units of u, minP/maxP the extremes of its inclusive prefixes. Given the EXACT state M entering it, a
// segment is valid iff E and sign match and M+minP, M+maxP stay in range —
// then the exit state is exactly M+Q. Segments merge associatively when E and
// sign agree. A *record* is a segment optionally followed by one break element
// whose value is applied with a real add. The device walks every thread's
// elements from a speculated start (an approximate prefix) to discover where
// breaks happen; a short serial chain then replays the records from the exact
// state, validating each segment and falling back to real adds if a
// speculation was wrong. Correctness never depends on the speculation.
#pragma once

#include <stdint.h>
#include <string.h>

#ifdef __CUDACC__
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD inline
#endif

namespace gmg_ss {

constexpr int64_t kLo = (int64_t(1) << 52) + 1;  // smallest admissible |M| after a step
constexpr int64_t kHi = (int64_t(1) << 53) - 1;  // largest admissible |M|
constexpr double kTwo52 = 4503599627370496.0;
constexpr int kEMin = 64;    // usable biased exponents: u = 2^(E-1075) and
constexpr int kEMax = 2040;  // 2^(1075-E) both normal, far from overflow

SS_HD uint64_t dbits(double x) {
#ifdef __CUDA_ARCH__
    return static_cast<uint64_t>(__double_as_longlong(x));
#else
    uint64_t b;
    memcpy(&b, &x, 8);
    return b;
#endif
}
SS_HD double bitsd(uint64_t b) {
#ifdef __CUDA_ARCH__
    return __longlong_as_double(static_cast<long long>(b));
#else
    double x;
    memcpy(&x, &b, 8);
    return x;
#endif
}

// Decomposed running sum: E = biased exponent (0 if not usable), M = signed
// integer significand (s = M * 2^(E-1075)), inv_u = 2^(1075-E).
struct State {
    double s;
    int E;
    int64_t M;
    double inv_u;
};

SS_HD State make_state(double s) {
    State st;
    st.s = s;
    const uint64_t b = dbits(s);
    const int E = static_cast<int>((b >> 52) & 0x7ff);
    if (E < kEMin || E > kEMax) {
        st.E = 0;
        st.M = 0;
        st.inv_u = 0.0;
        return st;
    }
    int64_t m = static_cast<int64_t>((b & ((uint64_t(1) << 52) - 1)) | (uint64_t(1) << 52));
    st.E = E;
    st.M = (b >> 63) ? -m : m;
    st.inv_u = bitsd(static_cast<uint64_t>(1075 + 1023 - E) << 52);  // 2^(1075-E)
    return st;
}

// Value of integer state M in binade E (|M| in [2^52, 2^53)). Exact.
SS_HD double compose(int64_t M, int E) {
    const uint64_t neg = M < 0 ? 1u : 0u;
    const uint64_t a = static_cast<uint64_t>(M < 0 ? -M : M);
    return bitsd((neg << 63) | (static_cast<uint64_t>(E) << 52) | (a - (uint64_t(1) << 52)));
}

// A segment carries two variants, indexed by the parity of the exact integer
// state entering it: an exact tie (p/u = n + 1/2) rounds to the even total, so
// q = n + ((M + n) & 1) depends only on M's parity — and after the first tie
// the running state is even in both variants. Ties therefore stay inside the
// integer model instead of forcing a real add.
struct Seg {
    int E;     // binade of the segment (meaningless when len == 0)
    int neg;   // sign of the running sum inside the segment
    int len;   // number of elements; 0 = empty (identity for merge)
    int bad;   // 1 = produced by merging incompatible segments (forces a fallback)
    int tied;  // walking only: a tie occurred (variant 1 is tracked separately from then on)
    int64_t Q[2], mn[2], mx[2];
};

// Before a walked segment is merged or stored: without a tie both parity
// variants are identical, and only variant 0 was maintained.
SS_HD void seg_finish(Seg& g) {
    if (!g.tied) {
        g.Q[1] = g.Q[0];
        g.mn[1] = g.mn[0];
        g.mx[1] = g.mx[0];
    }
    g.tied = 1;
}

SS_HD Seg seg_empty() {
    Seg s;
    s.E = 0;
    s.neg = 0;
    s.len = 0;
    s.bad = 0;
    s.tied = 1;
    for (int p = 0; p < 2; ++p) s.Q[p] = s.mn[p] = s.mx[p] = 0;
    return s;
}

SS_HD Seg seg_merge(Seg a, Seg b) {
    seg_finish(a);
    seg_finish(b);
    if (a.len == 0 && !a.bad) return b;
    if (b.len == 0 && !b.bad) return a;
    Seg r;
    r.E = a.E;
    r.neg = a.neg;
    r.len = a.len + b.len;
    r.bad = a.bad | b.bad | (a.E != b.E) | (a.neg != b.neg);
    r.tied = 1;
    // (selects, not b.Q[pb]: a runtime index would force the struct to local memory)
#pragma unroll
    for (int p = 0; p < 2; ++p) {
        const int64_t qa = a.Q[p];
        const bool odd = ((p + qa) & 1) != 0;
        const int64_t bq = odd ? b.Q[1] : b.Q[0];
        const int64_t bmn = qa + (odd ? b.mn[1] : b.mn[0]);
        const int64_t bmx = qa + (odd ? b.mx[1] : b.mx[0]);
        r.Q[p] = qa + bq;
        r.mn[p] = a.mn[p] < bmn ? a.mn[p] : bmn;
        r.mx[p] = a.mx[p] > bmx ? a.mx[p] : bmx;
    }
    return r;
}

// Is the segment valid from exact state st? (len == 0 is always valid.)
SS_HD bool seg_valid(const Seg& g, const State& st) {
    if (g.len == 0) return !g.bad;
    if (g.bad || st.E == 0 || st.E != g.E || (st.M < 0) != (g.neg != 0)) return false;
    const bool odd = (st.M & 1) != 0;
    const int64_t mn = odd ? g.mn[1] : g.mn[0], mx = odd ? g.mx[1] : g.mx[0];
    if (!g.neg) return st.M + mn >= kLo && st.M + mx <= kHi;
    return st.M + mx <= -kLo && st.M + mn >= -kHi;
}

// Apply a valid segment.
SS_HD void seg_apply(const Seg& g, State& st) {
    if (g.len == 0) return;
    st.M += (st.M & 1) ? g.Q[1] : g.Q[0];
    st.s = compose(st.M, st.E);
}

// Sequential walker: advances a (speculated or exact) state element by element,
// accumulating the current segment. Returns true if element p was absorbed,
// false if it is a break (the caller closes the segment, then calls real_add).
SS_HD bool walk_try(State& st, Seg& cur, double p) {
    if (st.E == 0) return false;
    const double x = p * st.inv_u;  // exact power-of-two scaling
    if (!(x < kTwo52 && x > -kTwo52)) return false;
#ifdef __CUDA_ARCH__
    const double fl = floor(x);
#else
    const double fl = __builtin_floor(x);
#endif
    const double fr = x - fl;  // exact
    const int64_t n = static_cast<int64_t>(fl);
    const bool tie = fr == 0.5;
    const int64_t qr = n + (fr > 0.5 ? 1 : 0);  // non-tie rounding
    const int64_t qs = tie ? n + ((st.M + n) & 1) : qr;
    const int64_t Mn = st.M + qs;
    if (st.M >= 0) {
        if (Mn < kLo || Mn > kHi) return false;
    } else {
        if (Mn > -kLo || Mn < -kHi) return false;
    }
    if (cur.len == 0) {
        cur.E = st.E;
        cur.neg = st.M < 0;
        cur.tied = 0;
        for (int v = 0; v < 2; ++v) cur.Q[v] = cur.mn[v] = cur.mx[v] = 0;
    }
    if (!cur.tied && !tie) {
        // fast path: both variants identical so far, only variant 0 is kept
        const int64_t P = cur.Q[0] + qr;
        if (cur.len == 0) {
            cur.mn[0] = P;
            cur.mx[0] = P;
        } else {
            cur.mn[0] = P < cur.mn[0] ? P : cur.mn[0];
            cur.mx[0] = P > cur.mx[0] ? P : cur.mx[0];
        }
        cur.Q[0] = P;
    } else {
        if (!cur.tied) seg_finish(cur);  // first tie: variant 1 starts as a copy
        for (int v = 0; v < 2; ++v) {
            // variant v: segment entered with parity v; current parity (v + Q[v]) & 1
            const int64_t q = tie ? n + ((v + cur.Q[v] + n) & 1) : qr;
            const int64_t P = cur.Q[v] + q;
            if (cur.len == 0) {
                cur.mn[v] = P;
                cur.mx[v] = P;
            } else {
                cur.mn[v] = P < cur.mn[v] ? P : cur.mn[v];
                cur.mx[v] = P > cur.mx[v] ? P : cur.mx[v];
            }
            cur.Q[v] = P;
        }
    }
    st.M = Mn;
    cur.len += 1;
    return true;
}

// fp64 speculative walker: the same decisions as walk_try, with the integer
// state and the open segment kept as exactly-representable doubles (|M| < 2^53,
// |prefix| < 2^53 inside a valid segment), so the per-term fast path is a
// handful of fp64 ops instead of emulated 64-bit integer arithmetic. Ties and
// segment closing convert to int64 (exact).
struct Walker {
    double s;      // speculated running sum (exact; authoritative when E == 0)
    int E;         // binade of s (0 = unusable: zero/subnormal/huge)
    double inv_u;  // 2^(1075-E)
    double u;      // 2^(E-1075)
    double M;      // signed integer significand of s
    int len, tied, segE, segneg;  // open segment
    double Q[2], mn[2], mx[2];
};

SS_HD void walker_set(Walker& w, double s) {
    w.s = s;
    const uint64_t b = dbits(s);
    const int E = static_cast<int>((b >> 52) & 0x7ff);
    if (E < kEMin || E > kEMax) {
        w.E = 0;
        w.M = 0.0;
        w.inv_u = w.u = 0.0;
        return;
    }
    w.E = E;
    w.inv_u = bitsd(static_cast<uint64_t>(1075 + 1023 - E) << 52);
    w.u = bitsd(static_cast<uint64_t>(E - 52) << 52);
    w.M = s * w.inv_u;  // exact
}
SS_HD void walker_open(Walker& w) {
    w.len = 0;
    w.tied = 0;
    w.segE = 0;
    w.segneg = 0;
    for (int v = 0; v < 2; ++v) w.Q[v] = w.mn[v] = w.mx[v] = 0.0;
}
SS_HD void walker_init(Walker& w, double s) {
    walker_set(w, s);
    walker_open(w);
}
// the open segment as a finished Seg (int64 fields)
SS_HD Seg walker_seg(const Walker& w) {
    Seg g = seg_empty();
    if (w.len == 0) return g;
    g.E = w.segE;
    g.neg = w.segneg;
    g.len = w.len;
    g.bad = 0;
    g.tied = 1;
    const int v1 = w.tied ? 1 : 0;
    g.Q[0] = static_cast<int64_t>(w.Q[0]);
    g.mn[0] = static_cast<int64_t>(w.mn[0]);
    g.mx[0] = static_cast<int64_t>(w.mx[0]);
    g.Q[1] = static_cast<int64_t>(w.Q[v1]);
    g.mn[1] = static_cast<int64_t>(w.mn[v1]);
    g.mx[1] = static_cast<int64_t>(w.mx[v1]);
    return g;
}
SS_HD bool walker_try(Walker& w, double p) {
    if (w.E == 0) return false;
    const double x = p * w.inv_u;  // exact power-of-two scaling
    if (!(x < kTwo52 && x > -kTwo52)) return false;
#ifdef __CUDA_ARCH__
    const double q = rint(x);
    const double fa = fabs(x - q);
#else
    const double q = __builtin_rint(x);
    const double fa = __builtin_fabs(x - q);
#endif
    const bool tie = fa == 0.5;
    double qs = q;
    double lower = 0.0;
    if (tie) {  // round the total to even: depends on the parity of M
        lower = x - 0.5;
        qs = ((static_cast<int64_t>(w.M) + static_cast<int64_t>(lower)) & 1) ? lower + 1.0 : lower;
    }
    const double Mn = w.M + qs;
#ifdef __CUDA_ARCH__
    const double aM = fabs(Mn);
#else
    const double aM = __builtin_fabs(Mn);
#endif
    if (aM < static_cast<double>(kLo) || aM > static_cast<double>(kHi)) return false;
    if (w.len == 0) {
        w.segE = w.E;
        w.segneg = w.M < 0.0;
    }
    if (!w.tied && !tie) {
        const double P = w.Q[0] + qs;
        w.mn[0] = w.len == 0 ? P : (P < w.mn[0] ? P : w.mn[0]);
        w.mx[0] = w.len == 0 ? P : (P > w.mx[0] ? P : w.mx[0]);
        w.Q[0] = P;
    } else {
        if (!w.tied) {
            w.Q[1] = w.Q[0];
            w.mn[1] = w.mn[0];
            w.mx[1] = w.mx[0];
            w.tied = 1;
        }
        for (int v = 0; v < 2; ++v) {
            double qv = qs;
            if (tie) {
                const int64_t par = (v + static_cast<int64_t>(w.Q[v]) + static_cast<int64_t>(lower)) & 1;
                qv = par ? lower + 1.0 : lower;
            }
            const double P = w.Q[v] + qv;
            w.mn[v] = w.len == 0 ? P : (P < w.mn[v] ? P : w.mn[v]);
            w.mx[v] = w.len == 0 ? P : (P > w.mx[v] ? P : w.mx[v]);
            w.Q[v] = P;
        }
    }
    w.M = Mn;
    w.len += 1;
    return true;
}
// the reference's own step s = s + p from the walker's exact state
SS_HD void walker_real_add(Walker& w, double p) {
    const double s = (w.E != 0 ? w.M * w.u : w.s) + p;
    walker_set(w, s);
}

// The reference's own step s = s + p, from the exact (integer) state.
SS_HD void real_add(State& st, double p) {
    const double s = (st.E != 0 ? compose(st.M, st.E) : st.s) + p;
    st = make_state(s);
}

// Record as stored for the chain: the merged run of elements since the previous
// record, then optionally one break element at global index kb (applied with a
// real add). A record covers exactly the elements (prev.kb, kb]; with a break
// the last of them is the break element. A record that fails validation is
// re-walked exactly over its range. 64 bytes.
//   meta: E (11b) | neg<<11 | has_break<<12 | bad<<13 | literal<<14 | nonempty<<15
// `literal` marks a chunk with too many breaks to store: the chain re-walks
// (prev.kb, kb] (kb = the chunk's last element).
struct Rec {
    int64_t Q[2], mn[2], mx[2];
    double pb;
    uint32_t meta;
    uint32_t kb;
};

SS_HD Rec rec_make(Seg g, bool has_break, double pb, uint32_t kb) {
    seg_finish(g);
    Rec r;
    for (int p = 0; p < 2; ++p) {
        r.Q[p] = g.Q[p];
        r.mn[p] = g.mn[p];
        r.mx[p] = g.mx[p];
    }
    r.pb = pb;
    r.meta = static_cast<uint32_t>(g.E & 0x7ff) | (static_cast<uint32_t>(g.neg) << 11) |
             (static_cast<uint32_t>(has_break) << 12) | (static_cast<uint32_t>(g.bad) << 13) |
             (static_cast<uint32_t>(g.len > 0) << 15);
    r.kb = kb;
    return r;
}
SS_HD Rec rec_literal(uint32_t kb) {
    Rec r = rec_make(seg_empty(), false, 0.0, kb);
    r.meta |= 1u << 14;
    return r;
}
SS_HD Seg rec_seg(const Rec& r) {
    Seg g;
    g.E = static_cast<int>(r.meta & 0x7ff);
    g.neg = static_cast<int>((r.meta >> 11) & 1);
    g.bad = static_cast<int>((r.meta >> 13) & 1);
    g.tied = 1;
    g.len = static_cast<int>((r.meta >> 15) & 1);  // emptiness only
    for (int p = 0; p < 2; ++p) {
        g.Q[p] = r.Q[p];
        g.mn[p] = r.mn[p];
        g.mx[p] = r.mx[p];
    }
    return g;
}
SS_HD bool rec_has_break(const Rec& r) { return (r.meta >> 12) & 1; }
SS_HD bool rec_literal_flag(const Rec& r) { return (r.meta >> 14) & 1; }

}  // namespace gmg_ss
