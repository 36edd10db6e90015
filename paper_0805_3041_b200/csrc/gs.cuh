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
// lane r-1 by a warp shuffle (computed on the previous step).
//   * Operands: each warp stages its 32 rows of d and x through shared memory,
//     32 columns at a time with coalesced cp.async copies, three blocks deep,
//     so the sequential loop only ever touches shared memory.
//   * The row above a warp (lane 31 of the warp before) arrives through a
//     shared-memory ring with block-scope progress counters inside a CTA, and
//     through global memory with release/acquire flags between CTAs.
//   * All CTAs are co-resident (grid <= 148 CTAs of kGsWarps warps), so the
//     spin-waits on predecessors always make progress.
// The critical path per anti-diagonal is one division by c (a multiplication
// when c is a power of two) + two multiply-subtracts + one shuffle. The same
// kernel runs ILU(0)'s two triangular solves (policies below).
#pragma once

#include "common.cuh"

namespace gmg_dev {

constexpr int kGsWarps = 4;     // warps (x 32 rows) per CTA
constexpr int kGsRing = 128;    // intra-CTA edge ring (columns)
constexpr int kGsPub = 4;       // progress published every kGsPub columns
constexpr int kGsWin = 8;       // edge values fetched per refill
constexpr int kGsBlk = 32;      // staged column block
constexpr int kGsSlots = 3;     // staged blocks in flight
constexpr int kGsStride = kGsBlk * kGsSlots + 2;  // even row stride: conflict-free diagonal reads

__device__ __forceinline__ void cp_async8(double* smem, const double* gmem) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}
__device__ __forceinline__ int ld_acquire(const int* p) {
    int v;
    asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(int* p, int v) {
    asm volatile("st.release.gpu.global.b32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The recurrence a wave solves, z_k = finish(rhs_k - a1_k*z_left - a2_k*z_up):
//   Gauss-Seidel/SOR   a1 = om*w, a2 = om*s, finish = /c        (smoother.cpp:297-309)
//   ILU(0) forward     a1 = lw,   a2 = ls,   finish = identity  (smoother.cpp:318-325)
//   ILU(0) backward    reversed order, a1 = e, a2 = n, finish = /d (smoother.cpp:326-334)
// A policy gives a1/a2/finish at physical (i, j). REV runs the wave from the
// last node backwards (logical (i, j) = physical (nx-1-i, ny-1-j)); UPDATE
// writes x - damp*z, otherwise z itself.
template <class Coef>
struct GsPolicy {
    static constexpr bool REV = false, UPDATE = true;
    Coef A;
    double om;
    __device__ __forceinline__ void coefs(int i, int j, double& a1, double& a2) const {
        double C, Wc, E, S, N;
        A.load(i, j, C, Wc, E, S, N);
        a1 = om * Wc;
        a2 = om * S;
    }
    __device__ __forceinline__ double finish(double acc, int i, int j) const { return A.div_by_c(acc, i, j); }
};

struct IluFwdPolicy {
    static constexpr bool REV = false, UPDATE = false;
    const double *lw, *ls;
    long long pitch;
    __device__ __forceinline__ void coefs(int i, int j, double& a1, double& a2) const {
        a1 = __ldg(lw + (long long)j * pitch + i);
        a2 = __ldg(ls + (long long)j * pitch + i);
    }
    __device__ __forceinline__ double finish(double acc, int, int) const { return acc; }
};

template <class Coef>
struct IluBwdPolicy {
    static constexpr bool REV = true, UPDATE = true;
    Coef A;
    const double* dp;
    long long pitch;
    __device__ __forceinline__ void coefs(int i, int j, double& a1, double& a2) const {
        double C, Wc, E, S, N;
        A.load(i, j, C, Wc, E, S, N);
        a1 = E;
        a2 = N;
    }
    __device__ __forceinline__ double finish(double acc, int i, int j) const {
        return acc / __ldg(dp + (long long)j * pitch + i);
    }
};

// dynamic smem: kGsWarps * 2 * 32 * kGsStride doubles
template <class Pol>
__global__ void __launch_bounds__(kGsWarps * 32) k_gs_wave(Grid g, Pol pol, const double* __restrict__ d,
                                                           const double* __restrict__ x, double* __restrict__ xo,
                                                           double damp, double* __restrict__ gedge,
                                                           int* __restrict__ gprog) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ double stg[];
    __shared__ double ring[kGsWarps][kGsRing];
    __shared__ volatile int prog[kGsWarps];  // columns of row 32w+31 available in ring[w]
    __shared__ volatile int cons[kGsWarps];  // columns of ring[w-1] consumed by warp w
    const int lane = threadIdx.x & 31;
    const int w = threadIdx.x >> 5;
    const int W = blockIdx.x * kGsWarps + w;  // global warp index
    if (lane == 0) {
        prog[w] = 0;
        cons[w] = 0;
    }
    __syncthreads();
    if (W * 32 >= g.ny) return;  // warp entirely below the grid
    const int j = W * 32 + lane;
    const bool row_ok = j < g.ny;
    const int nx = g.nx;
    const unsigned full = 0xffffffffu;
    const bool from_global = (w == 0 && W > 0);
    const bool to_global = (w == kGsWarps - 1) && (W + 1) * 32 < g.ny;
    const bool to_ring = (w + 1 < kGsWarps) && (W + 1) * 32 < g.ny;
    double* sd = stg + (size_t)w * 2 * 32 * kGsStride;
    double* sx = sd + 32 * kGsStride;
    const int rows = min(32, g.ny - W * 32);

    // stage column block b of this warp's rows (lane = column within the block)
    auto stage = [&](int b) {
        const int col = b * kGsBlk + lane;
        if (col < nx) {
            const int slot = (b % kGsSlots) * kGsBlk + lane;
            for (int rr = 0; rr < rows; ++rr) {
                const int jr = W * 32 + rr;
                const long long k = Pol::REV ? g.at(nx - 1 - col, g.ny - 1 - jr) : g.at(col, jr);
                cp_async8(sd + rr * kGsStride + slot, d + k);
                if (Pol::UPDATE) cp_async8(sx + rr * kGsStride + slot, x + k);
            }
        }
        cp_commit();
    };
    stage(0);
    stage(1);
    cp_wait<1>();
    __syncwarp();

    double zl = 0.0, zprev = 0.0, up = 0.0;
    int ebase = -64;
    const int steps = nx + 31;
    for (int tau = 0; tau < steps; ++tau) {
        if ((tau & (kGsBlk - 1)) == 0 && tau > 0) {
            // block tau/32 must be resident; prefetch the one after it
            stage(tau / kGsBlk + 1);
            cp_wait<1>();
            __syncwarp();
        }
        const int i = tau - lane;
        double zup = __shfl_up_sync(full, zprev, 1);
        if (W > 0 && tau < nx) {
            if (tau >= ebase + kGsWin) {
                ebase = tau;
                const int need = min(tau + kGsWin, nx);
                if (from_global) {
                    if (lane < kGsWin) {
                        while (ld_acquire(gprog + (W - 1)) < need) __nanosleep(32);
                        up = (ebase + lane < nx) ? __ldcg(gedge + (long long)(W - 1) * nx + ebase + lane) : 0.0;
                    }
                } else {
                    if (lane == 0) {
                        while (prog[w - 1] < need) __nanosleep(16);
                    }
                    __syncwarp();
                    up = (lane < kGsWin && ebase + lane < nx)
                             ? reinterpret_cast<volatile double*>(ring[w - 1])[(ebase + lane) % kGsRing]
                             : 0.0;
                    __syncwarp();
                    if (lane == 0) cons[w] = ebase;  // everything before ebase has been read
                }
                __syncwarp();
            }
            const double e = __shfl_sync(full, up, tau - ebase);
            if (lane == 0) zup = e;
        }
        double z = 0.0;
        if (row_ok && i >= 0 && i < nx) {
            const int slot = ((i / kGsBlk) % kGsSlots) * kGsBlk + (i & (kGsBlk - 1));
            const double dk = sd[lane * kGsStride + slot];
            const int pi = Pol::REV ? nx - 1 - i : i, pj = Pol::REV ? g.ny - 1 - j : j;
            double a1, a2;
            pol.coefs(pi, pj, a1, a2);
            double acc = dk;
            if (i > 0) acc = acc - a1 * zl;
            if (j > 0) acc = acc - a2 * zup;
            z = pol.finish(acc, pi, pj);
            if (Pol::UPDATE) {
                const double xk = sx[lane * kGsStride + slot];
                xo[g.at(pi, pj)] = xk - damp * z;
            } else {
                xo[g.at(pi, pj)] = z;
            }
            zl = z;
            if (lane == 31) {
                if (to_ring) {
                    // back-pressure: never overwrite a slot warp w+1 has not read yet
                    while (i - kGsRing >= cons[w + 1]) __nanosleep(16);
                    ring[w][i % kGsRing] = z;
                    if ((i + 1) % kGsPub == 0 || i == nx - 1) {
                        __threadfence_block();
                        prog[w] = i + 1;
                    }
                }
                if (to_global) {
                    gedge[(long long)W * nx + i] = z;
                    if ((i + 1) % kGsWin == 0 || i == nx - 1) st_release(gprog + W, i + 1);
                }
            }
        }
        zprev = z;
    }
    cp_wait<0>();
}

constexpr size_t gs_smem() { return sizeof(double) * kGsWarps * 2 * 32 * kGsStride; }

}  // namespace gmg_dev
