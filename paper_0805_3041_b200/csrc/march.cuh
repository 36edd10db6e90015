// Row-streaming ("marching") stencil kernels for sm_100a.
//
// Each CTA owns a strip of TW columns (one thread per column) and a segment of
// rows, and walks the rows upward. For an M-step smoother the CTA carries M
// pipeline levels: at iteration J it loads input row J, produces level-1 row
// J-1, level-2 row J-2, ... and writes level-M row J-M. Vertical neighbours of
// a thread's own column live in registers (a 3-row window per level);
// horizontal neighbours come from a double-buffered shared-memory row per
// level, so one __syncthreads per row suffices. Each input row is read from HBM
// once and each output row written once: M Jacobi steps cost 24 B/DOF of
// compulsory traffic (x, g in; x' out) instead of 24*M. Strips overlap by M
// columns on each side (recomputed halo), segments by M rows.
//
// Inputs are fetched PF rows ahead into registers so each SM keeps enough
// bytes in flight to saturate HBM3e.
//
// Reference semantics reproduced per point (one Jacobi smooth_step,
// smoother.cpp:389-399 with :293-295, apply from stencil.cpp:129-146):
//     acc = c*x + w*xw + e*xe + s*xs + n*xn      (ghosts = +0)
//     d   = acc - g
//     z   = d / c
//     x'  = x - omega*z
#pragma once

#include <type_traits>

#include "common.cuh"

namespace gmg_dev {

// ---------------- level-0 sources ------------------------------------------
// fetch() issues the loads for fine point (i,j) (returns zeros outside the
// interior); make() finishes the value. Splitting them lets the loads run PF
// rows ahead of the arithmetic.

struct SrcZero {  // u0 = 0 (inner V-cycle visits, cycle.cpp:89)
    static constexpr double kReads = 0;  // fine-level arrays read per DOF (coarse = 1/4)
    struct Raw {};
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ Raw fetch(int, int) const { return Raw{}; }
    __device__ __forceinline__ double make(const Raw&, int, int) const { return 0.0; }
};

struct SrcU {  // u0 = u
    static constexpr double kReads = 1;  // fine-level arrays read per DOF (coarse = 1/4)
    const double* u;
    Grid g;
    struct Raw {
        double v;
    };
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ Raw fetch(int i, int j) const {
        return Raw{g.inside(i, j) ? __ldg(u + g.at(i, j)) : 0.0};
    }
    __device__ __forceinline__ double make(const Raw& r, int, int) const { return r.v; }
};

struct SrcSum {  // x + e: fcycle_pass's out = x; axpy(1.0, e, out) (cycle.cpp:139-140)
    static constexpr double kReads = 2;  // fine-level arrays read per DOF (coarse = 1/4)
    const double *x, *e;
    Grid g;
    struct Raw {
        double a, b;
    };
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ Raw fetch(int i, int j) const {
        if (!g.inside(i, j)) return Raw{0.0, 0.0};
        const long long k = g.at(i, j);
        return Raw{__ldg(x + k), __ldg(e + k)};
    }
    __device__ __forceinline__ double make(const Raw& r, int, int) const { return r.a + 1.0 * r.b; }
};

// Coarse-to-fine bilinear prolongation evaluated while streaming the fine rows.
struct ProlongRaw {
    double a, b, c, d, ty;
};
__device__ __forceinline__ ProlongRaw prolong_fetch(const Prolong& P, int i, int j, int fnx, int fny) {
    ProlongRaw r{0.0, 0.0, 0.0, 0.0, 0.0};
    if (P.cg.per) {  // periodic y (fine rows 2 ny_c): wrap first, the coarse rows wrap in cval
        j %= fny;
        if (j < 0) j += fny;
    }
    if (i < 0 || i >= fnx || j < 0 || j >= fny) return r;
    const int pi = i + 1, pj = j + 1;
    const int ci = (pi & 1) ? (pi - 1) / 2 - 1 : pi / 2 - 1;  // left/only coarse column
    const int cj = (pj & 1) ? (pj - 1) / 2 - 1 : pj / 2 - 1;  // lower/only coarse row
    r.a = P.cval(ci, cj);
    if (pi & 1) r.b = P.cval(ci + 1, cj);
    if (pj & 1) {
        r.c = P.cval(ci, cj + 1);
        if (pi & 1) r.d = P.cval(ci + 1, cj + 1);
        r.ty = __ldg(P.ty + j);
    }
    return r;
}
// transfer.cpp:53,57,63-64 term order
__device__ __forceinline__ double prolong_make(const ProlongRaw& r, int i, int j, double tX) {
    const int pi = i + 1, pj = j + 1;
    if (!(pi & 1) && !(pj & 1)) return r.a;
    if ((pi & 1) && !(pj & 1)) return (1.0 - tX) * r.a + tX * r.b;
    if (!(pi & 1) && (pj & 1)) return (1.0 - r.ty) * r.a + r.ty * r.c;
    const double tY = r.ty;
    double v = (1.0 - tX) * (1.0 - tY) * r.a;
    v = v + tX * (1.0 - tY) * r.b;
    v = v + (1.0 - tX) * tY * r.c;
    v = v + tX * tY * r.d;
    return v;
}

struct SrcProlong {  // u0 = P e (fcycle_pass, cycle.cpp:135)
    static constexpr double kReads = 0.25;  // fine-level arrays read per DOF (coarse = 1/4)
    Prolong P;
    int fnx, fny;
    double tX;
    using Raw = ProlongRaw;
    __device__ __forceinline__ void prepare(int i) {
        tX = (i >= 0 && i < fnx && ((i + 1) & 1)) ? __ldg(P.tx + i) : 0.0;
    }
    __device__ __forceinline__ Raw fetch(int i, int j) const { return prolong_fetch(P, i, j, fnx, fny); }
    __device__ __forceinline__ double make(const Raw& r, int i, int j) const {
        return prolong_make(r, i, j, tX);
    }
};

// Adaptive correction weight (cycle.cpp:40-51) finished from the device sums
// of the exact-order engine: sums[0] = (A corr, corr), sums[1] = (d, corr),
// *nz = 1 iff some corr_k*corr_k != 0 (i.e. the reference's nc != 0).
struct OmegaSrc {
    const double* sums;  // null => fixed omega
    const int* nz;
    double fixed;
    int* status;  // set to 3 (runtime_error) on nonpositive energy
    __device__ __forceinline__ double get(bool report) const {
        if (!sums) return fixed;
        if (!*nz) return 1.0;
        const double den = sums[0];
        if (!(den > 0.0)) {
            if (report) atomicCAS(status, 0, 3);
            return 0.0;
        }
        return sums[1] / den;
    }
};

struct SrcCorrect {  // u + omega * P uc  (axpy(wl, corr, u), cycle.cpp:93-96)
    static constexpr double kReads = 1.25;  // fine-level arrays read per DOF (coarse = 1/4)
    const double* u;
    Grid g;
    Prolong P;
    double omega;
    double tX;
    struct Raw {
        double u;
        ProlongRaw p;
    };
    __device__ __forceinline__ void prepare(int i) {
        tX = (i >= 0 && i < g.nx && ((i + 1) & 1)) ? __ldg(P.tx + i) : 0.0;
    }
    __device__ __forceinline__ Raw fetch(int i, int j) const {
        Raw r;
        r.u = g.inside(i, j) ? __ldg(u + g.at(i, j)) : 0.0;
        r.p = prolong_fetch(P, i, j, g.nx, g.ny);
        return r;
    }
    __device__ __forceinline__ double make(const Raw& r, int i, int j) const {
        return r.u + omega * prolong_make(r.p, i, j, tX);
    }
};

// ---------------- M-step Jacobi smoother ----------------------------------
template <class Coef>
__device__ __forceinline__ double jacobi_point(const Coef& A, int i, int j, double xc, double xw,
                                               double xe, double xs, double xn, double g,
                                               double omega) {
    double C;
    const double acc = stencil_apply_c(A, i, j, xc, xw, xe, xs, xn, C);
    const double d = acc - g;
    const double z = div_loaded(A, d, C, i, j);
    return xc - omega * z;
}

// jacobi_point with the division's fast path only; `slow` asks the caller to
// recompute the point with jacobi_point (Coef::kMaySlow, common.cuh).
template <class Coef>
__device__ __forceinline__ double jacobi_point_fast(const Coef& A, int i, int j, double xc, double xw, double xe,
                                                    double xs, double xn, double g, double omega, bool& slow) {
    const double acc = stencil_apply(A, i, j, xc, xw, xe, xs, xn);
    const double d = acc - g;
    const double z = A.div_by_c_fast(d, i, j, slow);
    return xc - omega * z;
}

// ---------------- residual (+ restriction) ---------------------------------
// d = g - A x0 (stencil.cpp:148-153), or with neg the smoother defect
// A x0 - g (smoother.cpp:393-394), optionally stored; x0 optionally stored;
// optionally g_c = R d (transfer.cpp:72-101) for the next coarser level.
// Strip stride TW-4, halo 2 columns; segments of `seg` rows (seg even).
template <int TW, int PF, class Coef, class Src>
__global__ void __launch_bounds__(TW) k_resid(Grid fg, Coef A, Src src, const double* __restrict__ g,
                                              double* __restrict__ dout, double* __restrict__ x0out,
                                              Grid cg, RestrictW rw, double* __restrict__ gc, int seg,
                                              int neg, OmegaSrc om) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const bool STORE_D = dout != nullptr, STORE_X0 = x0out != nullptr, RESTRICT = gc != nullptr;
    constexpr int OUTW = TW - 4;
    __shared__ double xs[2][TW];
    __shared__ double dr[4][TW];

    const int t = threadIdx.x;
    const int i = blockIdx.x * OUTW - 2 + t;
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    const bool col_in = i >= 0 && i < fg.nx;
    const bool owner = col_in && t >= 2 && t < TW - 2;
    src.prepare(i);
    if constexpr (std::is_same<Src, SrcCorrect>::value) {
        src.omega = om.get(blockIdx.x == 0 && blockIdx.y == 0 && t == 0);
    }

    double a = 0.0, b = 0.0, c = 0.0;  // x0 rows J-2, J-1, J in own column
    // d is exact from row Jbeg+1 on; a coarse row centred on an odd first row
    // (a row-slab window may start there) needs d one row above the window
    const int Jbeg = j0 - 2;
    const int Jend = j1 + 1;
    typename Src::Raw q[PF];
    double gq[PF];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
        const int Jf = Jbeg + p;
        q[p] = src.fetch(i, Jf);
        gq[p] = (col_in && fg.row_ok(Jf - 1)) ? __ldg(g + fg.at(i, Jf - 1)) : 0.0;
    }
    for (int Jb = Jbeg; Jb <= Jend; Jb += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int J = Jb + p;
            if (J > Jend) break;
            const typename Src::Raw raw = q[p];
            const double gR = gq[p];  // g at row J-1
            {
                const int Jf = J + PF;
                q[p] = src.fetch(i, Jf);
                gq[p] = (col_in && fg.row_ok(Jf - 1)) ? __ldg(g + fg.at(i, Jf - 1)) : 0.0;
            }
            const bool row_in = fg.row_ok(J);
            const double x0 = (col_in && row_in) ? src.make(raw, i, fg.wrap(J)) : 0.0;
            if (STORE_X0 && owner && J >= j0 && J < j1) x0out[fg.at(i, J)] = x0;
            a = b;
            b = c;
            c = x0;
            const int R = J - 1;
            const double xl = t > 0 ? xs[(J - 1) & 1][t - 1] : 0.0;
            const double xr = t < TW - 1 ? xs[(J - 1) & 1][t + 1] : 0.0;
            xs[J & 1][t] = x0;
            double d = 0.0;
            if (col_in && fg.row_ok(R)) {
                const double ax = stencil_apply(A, cix(i, fg.nx), fg.wrap(R), b, xl, xr, a, c);
                d = neg ? ax - gR : gR - ax;  // smoother defect (Ax - g) or residual (g - Ax)
            }
            if (STORE_D && owner && R >= j0 && R < j1) dout[fg.at(i, R)] = d;
            if (RESTRICT) dr[R & 3][t] = d;
            __syncthreads();
            if (RESTRICT) {
                // coarse row Q whose centre fine row 2Q+1 = R-1 is owned
                if (((R & 1) == 0) && R >= 2 && R - 1 >= j0 && R - 1 < j1 && owner && (i & 1)) {
                    const int Q = R / 2 - 1;
                    const int P = (i - 1) / 2;
                    if (P < cg.nx && Q < cg.ny) {
                        const double v = restrict_at(rw, P, Q, [&](int di, int dj) {
                            return dr[(R - 1 + dj) & 3][t + di];
                        });
                        gc[cg.at(P, Q)] = v;
                    }
                }
            }
        }
    }
}

// ---------------- adaptive-omega terms ---------------------------------------
// adaptive_omega (cycle.cpp:40-51) needs, for corr = P uc on the fine level,
// the products (A corr)_k * corr_k and d_k * corr_k in the reference's k order,
// and whether any corr_k * corr_k != 0 (nc != 0). This kernel streams the rows
// once — one prolongation per point, A corr from the register window plus the
// shared-memory row — and writes both product arrays densely (k = j*nx + i) for
// the exact-order summation engine. Strip stride TW-2 (1-column halo).
template <int TW, int PF, class Coef>
__global__ void __launch_bounds__(TW) k_omega_terms(Grid fg, Coef A, SrcProlong src,
                                                    const double* __restrict__ d, double* __restrict__ T0,
                                                    double* __restrict__ T1, int* __restrict__ nz, int seg) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    constexpr int OUTW = TW - 2;
    __shared__ double xs[2][TW];
    const int t = threadIdx.x;
    const int i = blockIdx.x * OUTW - 1 + t;
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    const bool col_in = i >= 0 && i < fg.nx;
    const bool owner = col_in && t >= 1 && t < TW - 1;
    src.prepare(i);

    double a = 0.0, b = 0.0, c = 0.0;  // corr rows J-2, J-1, J in own column
    int any = 0;
    const int Jbeg = j0 - 1;
    const int Jend = j1;
    ProlongRaw q[PF];
    double dq[PF];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
        const int Jf = Jbeg + p;
        q[p] = src.fetch(i, Jf);
        dq[p] = (col_in && fg.row_ok(Jf - 1)) ? __ldg(d + fg.at(i, Jf - 1)) : 0.0;
    }
    for (int Jb = Jbeg; Jb <= Jend; Jb += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int J = Jb + p;
            if (J > Jend) break;
            const ProlongRaw raw = q[p];
            const double dR = dq[p];
            {
                const int Jf = J + PF;
                q[p] = src.fetch(i, Jf);
                dq[p] = (col_in && fg.row_ok(Jf - 1)) ? __ldg(d + fg.at(i, Jf - 1)) : 0.0;
            }
            const double cj = (col_in && fg.row_ok(J)) ? src.make(raw, i, fg.wrap(J)) : 0.0;
            a = b;
            b = c;
            c = cj;
            const int R = J - 1;
            const double xl = t > 0 ? xs[(J - 1) & 1][t - 1] : 0.0;
            const double xr = t < TW - 1 ? xs[(J - 1) & 1][t + 1] : 0.0;
            xs[J & 1][t] = cj;
            if (owner && R >= j0 && R < j1) {
                const double ac = stencil_apply(A, cix(i, fg.nx), R, b, xl, xr, a, c);
                const long long k = (long long)R * fg.nx + i;
                T0[k] = ac * b;
                T1[k] = dR * b;
                any |= (b * b) != 0.0;
            }
            __syncthreads();
        }
    }
    if (__syncthreads_or(any) && t == 0) atomicOr(nz, 1);
}

}  // namespace gmg_dev
