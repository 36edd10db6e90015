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
// Mapping: lane r of global warp W owns row j = 32W + r and, at step tau,
// handles column i = tau - r, i.e. one column behind the row above it. z(i,j-1)
// comes from lane r-1 by a warp shuffle (it was computed on the previous step);
// the row above a warp (lane 31 of warp W-1) is published through a small
// L2-resident edge buffer with progress counters, refilled 32 columns at a
// time. All warps of the grid are resident (<= 148 CTAs of <= 1024 threads),
// so the spin-waits on predecessor progress always make progress. The critical
// path is one fp64 division + two multiply-subtracts per anti-diagonal; the
// defect comes from the streaming residual kernel (k_resid, neg mode).
#pragma once

#include "common.cuh"

namespace gmg_dev {

constexpr int kGsPub = 4;  // progress published every kGsPub columns
constexpr int kGsWin = 8;  // edge values fetched per refill (lag between warps ~ 31 + kGsWin)

template <class Coef>
__global__ void __launch_bounds__(1024) k_gs_wave(Grid g, Coef A, const double* __restrict__ d,
                                                  const double* __restrict__ x, double* __restrict__ xo,
                                                  double om, double damp, double* __restrict__ edge,
                                                  int* __restrict__ prog) {
    const int lane = threadIdx.x & 31;
    const int W = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (W * 32 >= g.ny) return;  // warp entirely below the grid
    const int j = W * 32 + lane;
    const bool row_ok = j < g.ny;
    const int nx = g.nx;
    const unsigned full = 0xffffffffu;

    double zl = 0.0;     // own z at column i-1
    double zprev = 0.0;  // own z of the previous step, shuffled to the lane below
    double up = 0.0;     // edge cache: z(row 32W-1, ebase + lane)
    int ebase = -64;
    for (int tau = 0; tau < nx + 31; ++tau) {
        const int i = tau - lane;
        double zup = __shfl_up_sync(full, zprev, 1);
        if (W > 0 && tau < nx) {
            if (tau >= ebase + kGsWin) {
                ebase = tau;
                const int need = min(tau + kGsWin, nx);
                if (lane == 0) {
                    const volatile int* pp = prog + (W - 1);
                    while (*pp < need) {
                    }
                }
                __syncwarp();
                __threadfence();
                up = (lane < kGsWin && ebase + lane < nx) ? __ldcg(edge + (long long)(W - 1) * nx + ebase + lane) : 0.0;
            }
            const double e = __shfl_sync(full, up, tau - ebase);
            if (lane == 0) zup = e;
        }
        double z = 0.0;
        if (row_ok && i >= 0 && i < nx) {
            const long long k = g.at(i, j);
            if (i + 16 < nx) {
                asm volatile("prefetch.global.L1 [%0];" ::"l"(d + k + 16));
                asm volatile("prefetch.global.L1 [%0];" ::"l"(x + k + 16));
            }
            double C, Wc, E, S, N;
            A.load(i, j, C, Wc, E, S, N);
            double acc = __ldg(d + k);
            if (i > 0) acc = acc - om * Wc * zl;
            if (j > 0) acc = acc - om * S * zup;
            z = A.div_by_c(acc, i, j);
            xo[k] = __ldg(x + k) - damp * z;
            zl = z;
            if (lane == 31) {
                edge[(long long)W * nx + i] = z;
                if ((i + 1) % kGsPub == 0 || i == nx - 1) {
                    __threadfence();
                    *reinterpret_cast<volatile int*>(prog + W) = i + 1;
                }
            }
        }
        zprev = z;
    }
}

}  // namespace gmg_dev
