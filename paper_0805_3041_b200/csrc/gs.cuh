// Lexicographic Gauss-Seidel / SOR smoothing on sm_100a as an anti-diagonal
// wavefront.
//
// The reference's "gauss_seidel" is a preconditioned Richardson step
// (smoother.cpp:389-399 with :297-309): with the defect d = A x - g of the
// current iterate,
//     z_k = (d_k - (om*w_k)*z_{k-1} [i>0] - (om*s_k)*z_{k-nx} [j>0]) / c_k
// in lexicographic order, then x'_k = x_k - damp*z_k. Only z is sequential: a
// 2-D recurrence on z(i-1,j) and z(i,j-1).
//
// Mapping: lane r of warp w owns row j = 32w + r and, at step tau, handles
// column i = tau - r, one column behind the row above. z(i,j-1) comes from
// lane r-1 by a warp shuffle (computed on the previous step). With one warp per
// scheduler the sweep is bound by the latency of everything a step issues, so
// the step is kept to the recurrence itself:
//   * Operands: the 32 rows of d and x of a warp pass through shared memory,
//     16 columns at a time in coalesced 16-byte cp.async chunks, two blocks
//     ahead; results go back into the same slots and leave as 16-byte stores a
//     block at a time. The sequential loop touches shared memory only, and all
//     of the staging and flushing is done by a helper warp per compute warp
//     (same scheduler: it issues in the compute warp's stall slots), the two
//     meeting at a named barrier once per block.
//   * The row above a warp (lane 31 of the warp before) arrives, inside a CTA,
//     through a shared-memory ring of {value, column} words read a window of 16
//     columns at a time (the consumer trails the producer by ~47 steps), and
//     between CTAs through global
//     memory as 16-byte {value, generation} words, one per column, stored with a
//     single relaxed vector store and fetched 16 columns at a time one window
//     ahead of use: no flags or fences. The
//     generation (one per launch) tells a fresh value from the previous sweep's.
//     A window that is not complete yet is polled when it is needed (start-up
//     only: the consumer then trails the producer far enough).
//     Measured alternatives, both slower: a shared-memory ring for the hand-offs inside
//     a CTA (GMG_GS_RING; the extra stores and polls lengthen the step from 92 to 148
//     cycles), and per-column fetches 16 steps ahead with per-step validity checks
//     (4x slower: the window-boundary register hand-over waits for the newest load).
//   * Coefficients and the finishing operand of the next column are fetched one
//     step ahead (table/field operators, ILU factors).
//   * All CTAs are co-resident (grid <= 148 CTAs of kGsWarps warps), so the
//     polls on predecessors always make progress.
// The critical path per anti-diagonal is one shuffle + two multiply-subtracts +
// the division by c (a multiplication when c is a power of two, div_rcp from the
// host-rounded reciprocal otherwise). The same kernel runs ILU(0)'s two
// triangular solves (policies below).
#pragma once

#include "common.cuh"

namespace gmg_dev {

constexpr int kGsWarps = 4;     // compute warps (x 32 rows) per CTA: one per scheduler; as many helper warps
constexpr int kGsWin = 16;      // edge values fetched per window
constexpr int kGsERing = 128;   // intra-CTA edge ring (columns)
#ifndef GMG_GS_RING
#define GMG_GS_RING 0  // 1: hand-offs inside a CTA through a shared-memory ring (A/B variant)
#endif
constexpr int kGsBlk = 16;      // staged column block (= kGsWin: one helper rendezvous per window)
constexpr int kGsSlots = 6;     // block groups: 3 the lanes span, 2 in flight, 1 being written back
constexpr int kGsCols = kGsBlk * kGsSlots;
constexpr int kGsStride = kGsCols + 2;  // even row stride: conflict-free diagonal reads, 16-B chunks

__device__ __forceinline__ void cp_async16z(double* smem, const double* gmem, int bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
// edge words {z bits, generation}: one relaxed 16-byte store / load (value and tag travel together)
__device__ __forceinline__ void edge_store(longlong2* p, double z, long long gen) {
    asm volatile("st.relaxed.gpu.global.v2.s64 [%0], {%1, %2};" ::"l"(p), "l"(__double_as_longlong(z)), "l"(gen)
                 : "memory");
}
__device__ __forceinline__ longlong2 edge_load(const longlong2* p) {
    longlong2 r;
    asm volatile("ld.relaxed.gpu.global.v2.s64 {%0, %1}, [%2];" : "=l"(r.x), "=l"(r.y) : "l"(p) : "memory");
    return r;
}

// ring words {value, column}: the value is stored before its tag and the tag is read before
// the value (volatile shared accesses of one thread stay in program order)
// (predicated inside the asm: no branch in the step for the one lane that stores)
__device__ __forceinline__ void ring_store(bool on, unsigned a, double z, int col) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %0, 0;\n\t"
        "@p st.volatile.shared.f64 [%1], %2;\n\t"
        "@p st.volatile.shared.s64 [%1+8], %3;\n\t}" ::"r"((int)on),
        "r"(a), "d"(z), "l"((long long)col)
        : "memory");
}
__device__ __forceinline__ void edge_store_if(bool on, longlong2* p, double z, long long gen) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tsetp.ne.s32 p, %0, 0;\n\t"
        "@p st.relaxed.gpu.global.v2.s64 [%1], {%2, %3};\n\t}" ::"r"((int)on),
        "l"(p), "l"(__double_as_longlong(z)), "l"(gen)
        : "memory");
}
__device__ __forceinline__ double lds64(unsigned a) {
    double v;
    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts64(unsigned a, double v) {
    asm volatile("st.shared.f64 [%0], %1;" ::"r"(a), "d"(v) : "memory");
}

// The recurrence a wave solves, z_k = finish(rhs_k - a1_k*z_left - a2_k*z_up):
//   Gauss-Seidel/SOR   a1 = om*w, a2 = om*s, finish = /c        (smoother.cpp:297-309)
//   ILU(0) forward     a1 = lw,   a2 = ls,   finish = identity  (smoother.cpp:318-325)
//   ILU(0) backward    reversed order, a1 = e, a2 = n, finish = /d (smoother.cpp:326-334)
// A policy loads a1/a2 and its finishing operand f at physical (i, j) — one
// step ahead of use — and finishes a point from them. REV runs the wave from
// the last node backwards (logical (i, j) = physical (nx-1-i, ny-1-j)); UPDATE
// writes x - damp*z, otherwise z itself.
struct GsOps {
    double a1, a2, f;
};

// FIN: how z = acc / c is formed for constant operators (chosen on the host, common.cuh):
// 0 = the class's own div_by_c, 1 = exact reciprocal multiply (c a power of two),
// 2 = div_rcp from the host-rounded reciprocal.
template <class Coef, int FIN = 0>
struct GsPolicy {
    static constexpr bool REV = false, UPDATE = true;
    Coef A;
    double om;
    __device__ __forceinline__ void load(int i, int j, GsOps& o) const {
        double C, Wc, E, S, N;
        A.load(i, j, C, Wc, E, S, N);
        o.a1 = om * Wc;
        o.a2 = om * S;
        o.f = C;
    }
    __device__ __forceinline__ double finish(double acc, const GsOps& o, int i, int j) const {
        if constexpr (FIN == 1) return acc * A.inv_c;
        else if constexpr (FIN == 2) return div_rcp(acc, A.c, A.rcp);
        else return div_loaded(A, acc, o.f, i, j);
    }
    // The same quotient without a call on the path; `slow` (FIN 2: a dividend outside the
    // range div_rcp's two FMAs are exact for, never seen in a solve) asks for finish().
    static constexpr bool kMaySlow = FIN == 2;
    __device__ __forceinline__ double finish_fast(double acc, const GsOps& o, int i, int j, bool& slow) const {
        slow = false;
        if constexpr (FIN == 2) return div_rcp_fast(acc, A.c, A.rcp, slow);
        else return finish(acc, o, i, j);
    }
};

struct IluFwdPolicy {
    static constexpr bool REV = false, UPDATE = false;
    const double *lw, *ls;
    long long pitch;
    __device__ __forceinline__ void load(int i, int j, GsOps& o) const {
        o.a1 = __ldg(lw + (long long)j * pitch + i);
        o.a2 = __ldg(ls + (long long)j * pitch + i);
        o.f = 0.0;
    }
    __device__ __forceinline__ double finish(double acc, const GsOps&, int, int) const { return acc; }
    static constexpr bool kMaySlow = false;
    __device__ __forceinline__ double finish_fast(double acc, const GsOps&, int, int, bool& slow) const {
        slow = false;
        return acc;
    }
};

template <class Coef>
struct IluBwdPolicy {
    static constexpr bool REV = true, UPDATE = true;
    Coef A;
    const double* dp;
    long long pitch;
    __device__ __forceinline__ void load(int i, int j, GsOps& o) const {
        double C, Wc, E, S, N;
        A.load(i, j, C, Wc, E, S, N);
        o.a1 = E;
        o.a2 = N;
        o.f = __ldg(dp + (long long)j * pitch + i);
    }
    __device__ __forceinline__ double finish(double acc, const GsOps& o, int, int) const { return acc / o.f; }
    static constexpr bool kMaySlow = false;
    __device__ __forceinline__ double finish_fast(double acc, const GsOps& o, int, int, bool& slow) const {
        slow = false;
        return acc / o.f;
    }
};

// named barrier of a compute warp and its helper (ids 1..kGsWarps; 0 is __syncthreads)
__device__ __forceinline__ void pair_bar(int w) { asm volatile("bar.sync %0, 64;" ::"r"(w + 1) : "memory"); }

// dynamic smem: kGsWarps * 2 * 32 * kGsStride doubles. gedge: [warps][epitch] edge words
// (epitch >= nx), gstate: {generation, finished-CTA count}; both zero at allocation.
template <class Pol>
__global__ void __launch_bounds__(2 * kGsWarps * 32) k_gs_wave(Grid g, Pol pol, const double* __restrict__ d,
                                                           const double* __restrict__ x, double* __restrict__ xo,
                                                           double damp, longlong2* __restrict__ gedge, int epitch,
                                                           long long* __restrict__ gstate) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ __align__(16) double stg[];
    __shared__ long long s_gen;
    // edge rings between the compute warps of this CTA: {value, column} words, 128 columns
    // deep; cpos[w] = columns of ring[w-1] warp w has consumed (back-pressure for the producer)
    __shared__ longlong2 ering[kGsWarps][kGsERing];
    __shared__ volatile int cpos[kGsWarps];
    const int lane = threadIdx.x & 31;
    const bool helper = (threadIdx.x >> 5) >= kGsWarps;  // warps kGsWarps.. stage and flush for warps 0..
    const int w = (threadIdx.x >> 5) & (kGsWarps - 1);
    const int W = blockIdx.x * kGsWarps + w;  // global (compute) warp index
    // This launch's generation = gstate[0] + 1, read once per CTA; the CTA that finishes its
    // warp 0 last (gstate[1] counts them) advances gstate[0] for the next launch. A device
    // counter, not a kernel argument: launches replayed from a CUDA graph get fresh tags too.
    if (threadIdx.x == 0) s_gen = *reinterpret_cast<volatile long long*>(gstate) + 1;
    for (int q = threadIdx.x; q < kGsWarps * kGsERing; q += blockDim.x) (&ering[0][0])[q] = make_longlong2(0, -1);
    if (threadIdx.x < kGsWarps) cpos[threadIdx.x] = 0;
    __syncthreads();
    const long long gen = s_gen;
    if (W * 32 >= g.ny) return;  // warp entirely below the grid (no block barriers from here on)
    const int nx = g.nx, ny = g.ny;
    const int j = W * 32 + lane;  // logical row
    const bool row_ok = j < ny;
    const int pj = Pol::REV ? ny - 1 - j : j;
    const unsigned full = 0xffffffffu;
    const bool has_up = W > 0;
    const bool has_down = (W + 1) * 32 < ny;
    // the warp above / below is in this CTA (shared-memory ring) or in the previous / next one
    // (global edge words)
    // (GMG_GS_RING=1; measured slower than the global words for every hand-off: the two extra
    // stores and the window polls lengthen the step from 92 to 148 cycles, and a consumer that
    // must see a whole 16-column window trails its producer no closer than through global memory)
    constexpr bool kRing = GMG_GS_RING != 0;
    const bool up_ring = kRing && has_up && w > 0, up_glob = has_up && !up_ring;
    const bool down_ring = kRing && has_down && w + 1 < kGsWarps, down_glob = has_down && !down_ring;
    double* sd = stg + (size_t)w * 2 * 32 * kGsStride;
    double* sr = Pol::UPDATE ? sd + 32 * kGsStride : sd;  // where results are kept until the flush
    const int rows = min(32, ny - W * 32);
    const int nblk = (nx + kGsBlk - 1) / kGsBlk;
    // REV walks the physical blocks from the last one down; the wave's clock is shifted so
    // that lane 0 still enters a new physical block every 32 steps (i' = i + shift)
    const int shift = Pol::REV ? nblk * kGsBlk - nx : 0;
    const longlong2* ein = gedge + (long long)(W - 1) * epitch;
    longlong2* eout = gedge + (long long)W * epitch;

    // The k-th block in sweep order covers physical columns [32 pb, 32 pb + 32), pb = k or
    // nblk-1-k (REV), kept in slot group pb % 3 at its physical position. This lane moves the
    // 16-byte chunks (row rr0 + 2m, column pair pp) of a block, m = 0..15.
    // 16-byte chunks of a 16-column block: this lane moves (row rr0 + 4m, column pair pp), m = 0..7
    const int pp = lane & 7, rr0 = lane >> 3;
    const long long rstep = (Pol::REV ? -4 : 4) * g.pitch;  // global rows advance with the logical rows
    const long long row0 = (long long)(Pol::REV ? ny - 1 - (W * 32 + rr0) : W * 32 + rr0) * g.pitch;
    double* const srow = sd + rr0 * kGsStride;
    auto stage = [&](int k) {
        if (k < nblk) {
            const int pb = Pol::REV ? nblk - 1 - k : k;
            const int col = pb * kGsBlk + 2 * pp;
            const int bytes = col + 1 < nx ? 16 : (col < nx ? 8 : 0);
            const int slot = (pb % kGsSlots) * kGsBlk + 2 * pp;
            if (bytes) {
                const double* pd = d + row0 + col;
                const double* px = Pol::UPDATE ? x + row0 + col : nullptr;
                double* ps = srow + slot;
#pragma unroll
                for (int m = 0; m < 8; ++m) {
                    if (rr0 + 4 * m < rows) {
                        cp_async16z(ps, pd, bytes);
                        if (Pol::UPDATE) cp_async16z(ps + 32 * kGsStride, px, bytes);
                    }
                    pd += rstep;
                    if (Pol::UPDATE) px += rstep;
                    ps += 4 * kGsStride;
                }
            }
        }
        cp_commit();
    };
    // results of the k-th block (complete in shared memory) -> xo
    auto flush = [&](int k) {
        const int pb = Pol::REV ? nblk - 1 - k : k;
        const int col = pb * kGsBlk + 2 * pp;
        const int slot = (pb % kGsSlots) * kGsBlk + 2 * pp;
        if (col < nx) {
            double* o = xo + row0 + col;
            const double* ps = (Pol::UPDATE ? srow + 32 * kGsStride : srow) + slot;
            double2 v[8];
#pragma unroll
            for (int m = 0; m < 8; ++m) v[m] = *reinterpret_cast<const double2*>(ps + 4 * m * kGsStride);
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                if (rr0 + 4 * m < rows) {
                    if (col + 1 < nx) *reinterpret_cast<double2*>(o) = v[m];
                    else *o = v[m].x;
                }
                o += rstep;
            }
        }
    };
    // the window of edge values [c0, c0 + kGsWin) from the warp above (lanes < kGsWin)
    auto edge_fetch = [&](int c0, double& v, bool& ok) {
        ok = true;
        v = 0.0;
        if (lane < kGsWin && c0 + lane >= 0 && c0 + lane < nx) {
            const longlong2 wd = edge_load(ein + c0 + lane);
            v = __longlong_as_double(wd.x);
            ok = wd.y == gen;
        }
    };

    // the same window from the ring of the warp above in this CTA (tag = column)
    auto ring_fetch = [&](int c0, double& v, bool& ok) {
        ok = true;
        v = 0.0;
        if (lane < kGsWin && c0 + lane >= 0 && c0 + lane < nx) {
            const int c = c0 + lane;
            const unsigned a = static_cast<unsigned>(__cvta_generic_to_shared(&ering[w - 1][c & (kGsERing - 1)]));
            long long vy;
            asm volatile("ld.volatile.shared.s64 %0, [%1+8];" : "=l"(vy) : "r"(a) : "memory");
            asm volatile("ld.volatile.shared.f64 %0, [%1];" : "=d"(v) : "r"(a) : "memory");
            ok = vy == (long long)c;
        }
    };

    const int steps = nx + shift + 31;
    const int kb_max = (steps - 1) / kGsBlk;  // block boundaries the step loop passes
    if (helper) {
        // rows below the grid (last warp only) hold zeros, so their lanes run the recurrence
        // on benign values
        if (rows < 32) {
            for (int q = rows * kGsStride + lane; q < 32 * kGsStride; q += 32) {
                sd[q] = 0.0;
                sd[32 * kGsStride + q] = 0.0;
            }
        }
        stage(0);
        stage(1);
        stage(2);
        cp_wait<1>();
        pair_bar(w);  // blocks 0 and 1 are resident, block 2 is on its way
        for (int kb = 1; kb <= kb_max; ++kb) {
            // the compute warp arrives when lane 0 enters block kb (resident: it was waited
            // for before this warp arrived at the previous rendezvous); the lanes span blocks
            // kb-2 .. kb, so block kb-3 is complete and its group is the one after next to fill
            pair_bar(w);
            if (kb >= 3) flush(kb - 3);
            stage(kb + 2);  // into the group block kb-4 left at the previous rendezvous
            cp_wait<1>();   // block kb+1 has landed; kb+2 may still be in flight
        }
        pair_bar(w);  // the sweep is complete: the last blocks still in shared memory
        for (int k = max(0, kb_max - 2); k < nblk; ++k) flush(k);
        return;
    }

    double up = 0.0, upn = 0.0;  // edge windows: current, next
    bool upn_ok = true;
    if (up_glob) {
        bool ok;
        edge_fetch(-shift, up, ok);
        while (!__all_sync(full, ok)) {
            __nanosleep(100);
            edge_fetch(-shift, up, ok);
        }
    }
    pair_bar(w);
    const unsigned a_ring = static_cast<unsigned>(__cvta_generic_to_shared(&ering[w][0]));

    // The step loop is written to compile to straight-line predicated code (one warp per
    // scheduler pays the latency of every instruction and branch it issues): every lane
    // executes every step on an always-valid shared-memory slot; only the result store, the
    // edge store and the slot advance are predicated on the lane being inside its row.
    GsOps cur{0.0, 0.0, 1.0}, nxt{0.0, 0.0, 1.0};
    const int pjc = row_ok ? pj : (Pol::REV ? 0 : ny - 1);  // rows below the grid load row ny-1's operands
    auto load_ops = [&](int ii, GsOps& o) {  // operands of logical column ii (clamped into the row)
        const int ic = min(max(ii, 0), nx - 1);
        pol.load(Pol::REV ? nx - 1 - ic : ic, pjc, o);
    };
    int i = -lane - shift;  // logical column of this lane at step 0
    load_ops(i, cur);
    double zl = 0.0, zprev = 0.0;
    // byte offset of the logical column in hand within the lane's shared-memory row (column 0
    // first): cyclic over kGsCols slots, forwards (backwards for REV)
    int off;
    {
        const int pi = Pol::REV ? nx - 1 : 0;
        off = 8 * (((pi / kGsBlk) % kGsSlots) * kGsBlk + (pi & (kGsBlk - 1)));
    }
    const unsigned a_d = static_cast<unsigned>(__cvta_generic_to_shared(sd + lane * kGsStride));
    const unsigned a_x = static_cast<unsigned>(__cvta_generic_to_shared(sd + (32 + lane) * kGsStride));
    const unsigned a_r = Pol::UPDATE ? a_x : a_d;
    const bool jpos = j > 0;
    const bool dg31 = down_glob && lane == 31, dr31 = down_ring && lane == 31;
    for (int t0 = 0; t0 < steps; t0 += kGsWin) {
        // lane 0 enters block t0/16: the helper has it resident, and takes block t0/16 - 3
        if (t0 > 0) pair_bar(w);
        const int c0 = t0 - shift;  // lane 0's logical column at step t0
        if (up_ring && c0 < nx) {
            // this window straight from the ring (a shared-memory round trip per 16 steps)
            bool ok;
            ring_fetch(c0, up, ok);
            while (!__all_sync(full, ok)) ring_fetch(c0, up, ok);
            if (lane == 0) cpos[w] = c0;  // everything before c0 sits in registers
        }
        if (down_ring) {
            // lane 31 writes columns c0-31 .. c0-16 in this window: their slots' previous
            // columns must have been read
            while (c0 - 16 - kGsERing >= cpos[w + 1]) {
            }
        }
        if (up_glob && c0 < nx) {
            if (t0 > 0) {
                // the window fetched one window ago; poll only if the producer was not there yet
                while (!__all_sync(full, upn_ok)) {
                    __nanosleep(100);
                    edge_fetch(c0, upn, upn_ok);
                }
                up = upn;
            }
            if (c0 + kGsWin < nx) edge_fetch(c0 + kGsWin, upn, upn_ok);
        }
        // The 16 steps of a window as straight-line code. Rows without a left / upper
        // neighbour skip that term as the reference does (i > 0, j > 0): j = 0 is lane 0 of
        // warp 0 only, which subtracts a2 * (0 with a2's sign) = +0, the exact identity; i = 0
        // happens in the first two windows (START), which select on it — every warp's first
        // 47 steps sit on the critical path of the whole sweep, so they run this body too.
        // Lanes ahead of their row (i < 0) or past it (i >= nx) compute on benign values and
        // store nothing. A dividend the fast quotient cannot take (kMaySlow) is voted on
        // before anything of the step is released; the rest of the window then runs the exact
        // rolled body below — the call it contains stays out of the hot loop.
        auto fast_window = [&](auto tag) -> int {
            constexpr bool START = decltype(tag)::value;
#pragma unroll
            for (int u = 0; u < kGsWin; ++u) {
                const double zs = __shfl_up_sync(full, zprev, 1);
                double e = __shfl_sync(full, up, u);
                if (!has_up) e = copysign(0.0, cur.a2);
                const double zup = lane == 0 ? e : zs;
                load_ops(i + 1, nxt);  // next column's operands, one step ahead
                const double dk = lds64(a_d + off);
                const double t1 = cur.a1 * zl;
                const double t2 = cur.a2 * zup;
                double acc = dk - t1;
                if (START) acc = i > 0 ? acc : dk;
                acc = acc - t2;
                bool slow;
                const double z = pol.finish_fast(acc, cur, Pol::REV ? nx - 1 - i : i, pjc, slow);
                if (Pol::kMaySlow) {
                    if (__any_sync(full, slow)) return u;  // nothing of step u has been released
                }
                const bool live = row_ok && (!START || i >= 0) && i < nx;
                double res = z;
                if (Pol::UPDATE) res = lds64(a_x + off) - damp * z;
                if (live) sts64(a_r + off, res);  // (rows below the grid stay zero)
                edge_store_if(live && dg31, eout + i, z, gen);
                ring_store(live && dr31, a_ring + ((i & (kGsERing - 1)) << 4), z, i);
                int offn;
                if (Pol::REV) offn = off == 0 ? 8 * (kGsCols - 1) : off - 8;
                else offn = off == 8 * (kGsCols - 1) ? 0 : off + 8;
                off = (!START || i >= 0) ? offn : off;
                zl = z;
                zprev = z;
                cur = nxt;
                ++i;
            }
            return kGsWin;
        };
        int u0 = c0 < 32 ? fast_window(std::true_type{}) : fast_window(std::false_type{});
#pragma unroll 1
        for (int u = u0; u < kGsWin; ++u) {  // exact steps (after a vote only)
            const double zs = __shfl_up_sync(full, zprev, 1);
            const double e = __shfl_sync(full, up, u);  // (0 without a warp above: unused, j == 0)
            const double zup = lane == 0 ? e : zs;
            const bool act = row_ok && static_cast<unsigned>(i) < static_cast<unsigned>(nx);
            load_ops(i + 1, nxt);
            const double dk = lds64(a_d + off);
            double acc = dk;
            if (i > 0) acc = acc - cur.a1 * zl;
            if (jpos) acc = acc - cur.a2 * zup;
            double z = pol.finish(acc, cur, Pol::REV ? nx - 1 - i : i, pjc);
            z = act ? z : 0.0;
            double res = z;
            if (Pol::UPDATE) res = lds64(a_x + off) - damp * z;
            if (act) sts64(a_r + off, res);
            edge_store_if(act && dg31, eout + i, z, gen);
            ring_store(act && dr31, a_ring + ((i & (kGsERing - 1)) << 4), z, i);
            if (Pol::REV) off = act ? (off == 0 ? 8 * (kGsCols - 1) : off - 8) : off;
            else off = act ? (off == 8 * (kGsCols - 1) ? 0 : off + 8) : off;
            zl = z;
            zprev = z;
            cur = nxt;
            ++i;
        }
    }
    pair_bar(w);  // the helper writes out the last blocks
    if (w == 0 && lane == 0) {
        __threadfence();
        if (atomicAdd(reinterpret_cast<unsigned long long*>(gstate) + 1, 1ull) == gridDim.x - 1) {
            gstate[1] = 0;
            __threadfence();
            atomicAdd(reinterpret_cast<unsigned long long*>(gstate), 1ull);
        }
    }
}

constexpr int kGsThreads = 2 * kGsWarps * 32;
constexpr size_t gs_smem() { return sizeof(double) * kGsWarps * 2 * 32 * kGsStride; }

}  // namespace gmg_dev
