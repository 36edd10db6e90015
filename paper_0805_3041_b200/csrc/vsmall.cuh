// k_vsmall: the whole V-cycle below a small level in one CTA.
//
// On the coarse levels (<= 63^2 unknowns) every kernel of a level visit is
// pure latency: a few microseconds for a handful of rows, and the F-cycle
// visits levels 1..6 about 60 times per cycle. This kernel runs
// gmg::mg_cycle (cycle.cpp:69-100, V recursion) for levels top..1 inside one
// CTA of 1024 threads with every level's u, g and d resident in shared memory:
//   descent  pre-smoothing (Jacobi), residual, restriction, zero coarse start
//   level 1  BandedCholesky::solve (stencil.cpp:190-210) or smoothing
//   ascent   prolongation, adaptive omega (cycle.cpp:40-51, both sums
//            left-to-right by one thread each, as k_ss_direct), u + w*corr,
//            post-smoothing
// with the reference's arithmetic per point (jacobi_point, stencil_apply,
// restrict_at, the prolongation's products and sums), so results are
// bit-identical to the level-by-level kernels it replaces.
#pragma once

#include "common.cuh"
#include "march.cuh"

namespace gmg_dev {

constexpr int kVTop = 6;        // highest level handled (<= 63^2 for a 1x1 coarse grid)
constexpr int kVThreads = 1024;
constexpr size_t kVSmemMax = 200 * 1024;

struct VLev {
    int nx, ny;
    int per;  // y periodic (polar): row neighbours and transfer rows wrap
    long long pitch;
    int kind;  // 0 CONST, 1 ROWX, 2 FIELD
    CoefConst cc;
    CoefRowX cr;
    CoefField cf;
    CoefAxes ca;
    const double *tx, *ty;  // prolongation weights (this level as fine)
    RestrictW rw;           // restriction weights (this level as coarse)
    int off;                // shared-memory offset (doubles) of U, G, D (each nx*ny)
};

struct VParams {
    VLev lv[kVTop + 1];  // [1..top]
    int top, pre, post, adaptive, direct, cn, cbw;
    double damp, corr_omega;
    const double* band;
    const double* g_top;  // rhs of the top level (pitched, global)
    const double* uc;     // start P*uc from level top-1 (pitched, global), or null: zero start
    double* out;          // result, top level (pitched, global)
    int* status;
    int toff;  // shared-memory offset of the two top-size scratch arrays
};

template <class F>
__device__ __forceinline__ void with_vcoef(const VLev& L, F&& f) {
    if (L.kind == 0) f(L.cc);
    else if (L.kind == 1) f(L.cr);
    else if (L.kind == 3) f(L.ca);
    else f(L.cf);
}

// fine value of the prolongation at interior (i, j) from coarse values cv(ci, cj)
// (0 outside the coarse interior): transfer.cpp:43-68 term for term (= Prolong::at).
template <class CV>
__device__ __forceinline__ double prolong_dense(const double* tx, const double* ty, int i, int j, CV&& cv) {
    const int pi = i + 1, pj = j + 1;
    if ((pi & 1) == 0 && (pj & 1) == 0) return cv(pi / 2 - 1, pj / 2 - 1);
    if ((pi & 1) == 1 && (pj & 1) == 0) {
        const int qx = (pi - 1) / 2;
        const double t = tx[i];
        return (1.0 - t) * cv(qx - 1, pj / 2 - 1) + t * cv(qx, pj / 2 - 1);
    }
    if ((pi & 1) == 0 && (pj & 1) == 1) {
        const int qy = (pj - 1) / 2;
        const double t = ty[j];
        return (1.0 - t) * cv(pi / 2 - 1, qy - 1) + t * cv(pi / 2 - 1, qy);
    }
    const int qx = (pi - 1) / 2, qy = (pj - 1) / 2;
    const double tX = tx[i], tY = ty[j];
    double v = (1.0 - tX) * (1.0 - tY) * cv(qx - 1, qy - 1);
    v = v + tX * (1.0 - tY) * cv(qx, qy - 1);
    v = v + (1.0 - tX) * tY * cv(qx - 1, qy);
    v = v + tX * tY * cv(qx, qy);
    return v;
}

__global__ void __launch_bounds__(kVThreads) k_vsmall(VParams P) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    extern __shared__ double vs[];
    const int t = threadIdx.x;
    double* T = vs + P.toff;                      // smoothing ping-pong / correction
    double* X = T + P.lv[P.top].nx * P.lv[P.top].ny;  // (A corr) * corr terms
    auto U = [&](int l) { return vs + P.lv[l].off; };
    auto G = [&](int l) { return vs + P.lv[l].off + P.lv[l].nx * P.lv[l].ny; };
    auto D = [&](int l) { return vs + P.lv[l].off + 2 * P.lv[l].nx * P.lv[l].ny; };

    // x' = x - damp * (A x - g) / c, `steps` times, result in u
    auto smooth = [&](int l, int steps, double* u, const double* g) {
        const VLev& L = P.lv[l];
        const int nx = L.nx, ny = L.ny, n = nx * ny;
        double* a = u;
        double* b = T;
        for (int s = 0; s < steps; ++s) {
            with_vcoef(L, [&](const auto& A) {
                for (int k = t; k < n; k += kVThreads) {
                    const int i = k % nx, j = k / nx;
                    const double xw = i > 0 ? a[k - 1] : 0.0, xe = i + 1 < nx ? a[k + 1] : 0.0;
                    const double xs = j > 0 ? a[k - nx] : (L.per ? a[k + (ny - 1) * nx] : 0.0);
                    const double xn = j + 1 < ny ? a[k + nx] : (L.per ? a[i] : 0.0);
                    b[k] = jacobi_point(A, i, j, a[k], xw, xe, xs, xn, g[k], P.damp);
                }
            });
            __syncthreads();
            double* tmp = a;
            a = b;
            b = tmp;
        }
        if (a != u) {
            for (int k = t; k < n; k += kVThreads) u[k] = a[k];
            __syncthreads();
        }
    };

    // ---- load the top level's rhs and start -------------------------------
    {
        const VLev& L = P.lv[P.top];
        const int nx = L.nx, n = nx * L.ny;
        double* g = G(P.top);
        double* u = U(P.top);
        for (int k = t; k < n; k += kVThreads) {
            const int i = k % nx, j = k / nx;
            g[k] = P.g_top[(long long)j * L.pitch + i];
            double v = 0.0;
            if (P.uc && P.top > 1) {
                const VLev& C = P.lv[P.top - 1];
                v = prolong_dense(L.tx, L.ty, i, j, [&](int ci, int cj) {
                    if (C.per && cj < 0) cj += C.ny;  // coarse node 0 == coarse node ny_c
                    return (ci >= 0 && ci < C.nx && cj >= 0 && cj < C.ny) ? P.uc[(long long)cj * C.pitch + ci] : 0.0;
                });
            }
            u[k] = v;
        }
        __syncthreads();
    }
    // ---- descent -------------------------------------------------------------
    for (int l = P.top; l >= 2; --l) {
        const VLev& L = P.lv[l];
        const int nx = L.nx, ny = L.ny, n = nx * ny;
        smooth(l, P.pre, U(l), G(l));
        const double* u = U(l);
        const double* g = G(l);
        double* d = D(l);
        with_vcoef(L, [&](const auto& A) {
            for (int k = t; k < n; k += kVThreads) {
                const int i = k % nx, j = k / nx;
                const double xw = i > 0 ? u[k - 1] : 0.0, xe = i + 1 < nx ? u[k + 1] : 0.0;
                const double xs = j > 0 ? u[k - nx] : (L.per ? u[k + (ny - 1) * nx] : 0.0);
                const double xn = j + 1 < ny ? u[k + nx] : (L.per ? u[i] : 0.0);
                d[k] = g[k] - stencil_apply(A, i, j, u[k], xw, xe, xs, xn);
            }
        });
        __syncthreads();
        const VLev& C = P.lv[l - 1];
        const int cn = C.nx * C.ny;
        double* gc = G(l - 1);
        double* ucz = U(l - 1);
        for (int k = t; k < cn; k += kVThreads) {
            const int Pc = k % C.nx, Qc = k / C.nx;
            gc[k] = restrict_at(C.rw, Pc, Qc, [&](int di, int dj) {
                const int r = 2 * Qc + 1 + dj;  // < ny, or == ny on a periodic level: row 0
                return d[(r < ny ? r : r - ny) * nx + 2 * Pc + 1 + di];
            });
            ucz[k] = 0.0;
        }
        __syncthreads();
    }
    // ---- level 1 ----------------------------------------------------------------
    {
        const VLev& L = P.lv[1];
        const int n = L.nx * L.ny;
        if (P.direct) {
            if (t == 0) {
                // BandedCholesky::solve: forward then backward in the reference's d-loop order
                double* xs = U(1);
                const double* b = G(1);
                for (int k = 0; k < P.cn; ++k) {
                    double acc = b[k];
                    const int dm = min(P.cbw, k);
                    for (int q = 1; q <= dm; ++q) acc = acc - P.band[(long long)q * P.cn + k] * xs[k - q];
                    xs[k] = acc / P.band[k];
                }
                for (int k = P.cn - 1; k >= 0; --k) {
                    double acc = xs[k];
                    const int dm = min(P.cbw, P.cn - 1 - k);
                    for (int q = 1; q <= dm; ++q) acc = acc - P.band[(long long)q * P.cn + k + q] * xs[k + q];
                    xs[k] = acc / P.band[k];
                }
            }
            __syncthreads();
        } else {
            if (P.top == 1 && P.uc == nullptr) {
                for (int k = t; k < n; k += kVThreads) U(1)[k] = 0.0;
                __syncthreads();
            }
            smooth(1, max(1, P.pre + P.post), U(1), G(1));
        }
    }
    // ---- ascent ------------------------------------------------------------------
    for (int l = 2; l <= P.top; ++l) {
        const VLev& L = P.lv[l];
        const VLev& C = P.lv[l - 1];
        const int nx = L.nx, ny = L.ny, n = nx * ny;
        const double* uc = U(l - 1);
        for (int k = t; k < n; k += kVThreads) {
            const int i = k % nx, j = k / nx;
            T[k] = prolong_dense(L.tx, L.ty, i, j, [&](int ci, int cj) {
                if (C.per && cj < 0) cj += C.ny;  // coarse node 0 == coarse node ny_c
                return (ci >= 0 && ci < C.nx && cj >= 0 && cj < C.ny) ? uc[cj * C.nx + ci] : 0.0;
            });
        }
        __syncthreads();
        __shared__ double sum2[2];
        double w = P.corr_omega;
        if (P.adaptive) {
            double* d = D(l);
            int any = 0;
            with_vcoef(L, [&](const auto& A) {
                for (int k = t; k < n; k += kVThreads) {
                    const int i = k % nx, j = k / nx;
                    const double b = T[k];
                    const double xw = i > 0 ? T[k - 1] : 0.0, xe = i + 1 < nx ? T[k + 1] : 0.0;
                    const double xs = j > 0 ? T[k - nx] : (L.per ? T[k + (ny - 1) * nx] : 0.0);
                    const double xn = j + 1 < ny ? T[k + nx] : (L.per ? T[i] : 0.0);
                    X[k] = stencil_apply(A, i, j, b, xw, xe, xs, xn) * b;
                    d[k] = d[k] * b;
                    any |= (b * b) != 0.0;
                }
            });
            any = __syncthreads_or(any);
            if (t == 0 || t == 32) {  // the two sums in parallel, each left to right from 0.0
                const double* v = t == 0 ? X : d;
                double a = 0.0;
                int k = 0;
                for (; k + 8 <= n; k += 8) {
                    double r[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) r[q] = v[k + q];
#pragma unroll
                    for (int q = 0; q < 8; ++q) a = a + r[q];
                }
                for (; k < n; ++k) a = a + v[k];
                sum2[t == 0 ? 0 : 1] = a;
            }
            __syncthreads();
            if (!any) {
                w = 1.0;
            } else if (!(sum2[0] > 0.0)) {
                if (t == 0) atomicCAS(P.status, 0, 3);
                w = 0.0;
            } else {
                w = sum2[1] / sum2[0];
            }
        }
        double* u = U(l);
        for (int k = t; k < n; k += kVThreads) u[k] = u[k] + w * T[k];
        __syncthreads();
        smooth(l, P.post, u, G(l));
    }
    // ---- result ---------------------------------------------------------------------
    {
        const VLev& L = P.lv[P.top];
        const int nx = L.nx, n = nx * L.ny;
        const double* u = U(P.top);
        for (int k = t; k < n; k += kVThreads) P.out[(long long)(k / nx) * L.pitch + k % nx] = u[k];
    }
}

}  // namespace gmg_dev
