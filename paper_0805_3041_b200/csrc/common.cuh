// Shared device definitions for the B200 multigrid path.
//
// Data layout in HBM: every level-l grid function lives in a
// pitched buffer, element (i,j) at base[j*pitch + i], pitch = nx rounded up to
// 32 doubles (256 B rows), base 256-B aligned, with a zero ghost ring
// (row -1, row ny, column -1 == previous row's padding, column nx..pitch-1).
// Kernels never write ghosts; all neighbour reads are guarded explicitly, so
// a ghost contributes coefficient * (+0), which is the identity on the
// accumulator exactly as the reference's skipped term (stencil.cpp:134-144).
//
// All arithmetic is fp64 in the reference's association order. The library is
// compiled with -fmad=false: no multiply-add contraction anywhere (SURVEY.md
// Appendix A); fused ops appear only inside correctly-rounded helpers that are
// bit-identical to the unfused IEEE result.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gmg_dev {

// Programmatic dependent launch (kernels are launched with the PDL attribute,
// solver.cu launch_k): every kernel first waits until the previous kernel in the
// stream has completed and its writes are visible. The early trigger that would
// let the next kernel's CTAs launch into this kernel's last wave is compiled out
// by default (-DGMG_PDL_TRIGGER enables it): measured on C4 it costs 3% — the
// waiting CTAs hold registers and shared memory the tail of this kernel could
// use. Without the launch attribute both are no-ops.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
#ifdef GMG_PDL_TRIGGER
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

constexpr int kWarp = 32;

// Rows [w0, w1) are the rows a kernel produces (the whole grid, or one rank's
// slab of it when a level is sharded); domain tests always use the
// full [0, ny).
// per: the level is periodic in y (polar theta, BASELINE config 3): every row
// index wraps modulo ny, and no row is outside the domain.
struct Grid {
    int nx, ny;
    long long pitch;
    int w0 = 0, w1 = 0;
    int per = 0;
    __host__ __device__ int wrap(int j) const {
        if (!per) return j;
        const int r = j % ny;
        return r < 0 ? r + ny : r;
    }
    __host__ __device__ bool row_ok(int j) const { return per || (j >= 0 && j < ny); }
    __host__ __device__ long long at(int i, int j) const { return (long long)wrap(j) * pitch + i; }
    __host__ __device__ bool inside(int i, int j) const { return i >= 0 && i < nx && row_ok(j); }
};

// ---------------------------------------------------------------------------
// Operator storage classes (classified on the host from the reference's five
// StencilOperator arrays, stencil.hpp:20-28).
//   CONST : c, w, e, s, n identical on every interior row/column and exactly 0
//           toward the boundary (cartesian uniform grids, all BASELINE configs
//           but C3): 0 B/DOF of coefficient traffic.
//   ROWX  : coefficients depend on i only (uniform cylindrical, C3'): 1-D tables.
//   FIELD : general graded / spherical: five pitched arrays.
// `div_by_c` is the Jacobi preconditioner z = r / c (smoother.cpp:293-295):
// the IEEE round-to-nearest quotient, computed as a multiplication by the exact
// reciprocal when c is a power of two, else by div_rcp from the host-rounded
// reciprocal (three fp64 ops instead of the division's iteration; identical
// result), else by a true division.
// ---------------------------------------------------------------------------

// RN(d / c) from y = RN(1 / c) (Markstein's theorem: q0 = RN(d y) is within one
// ulp of d / c, so r = d - q0 c is exact in one FMA and RN(q0 + r y) is the
// correctly rounded quotient; no underflow or overflow on the way for
// 2^-960 < |d| < 2^960 and c, y normal in [2^-500, 2^500], which the host checks).
// Zeros keep their sign (q0 = +-0); huge/tiny, inf and NaN dividends take the
// true division, out of line: an inlined IEEE division (~30 instructions and a
// slow path) per point and fused step would swamp the instruction cache of the
// unrolled streaming kernels.
static __device__ __noinline__ double div_ieee(double d, double c) { return d / c; }
__device__ __forceinline__ double div_rcp(double d, double c, double y) {
    const double q0 = d * y;
    const double a = fabs(d);
    if (!(a > 0x1p-960 && a < 0x1p960)) return d == 0.0 ? q0 : div_ieee(d, c);
    const double r = __fma_rn(-q0, c, d);
    return __fma_rn(r, y, q0);
}

// div_rcp without the out-of-line division: RN(d / c) unless `slow` is set
// (|d| outside the checked range and d != 0, or inf/NaN), in which case the
// caller recomputes the point through div_rcp / div_ieee. Range and zero tests
// are integer ops on d's bits (the fp64 pipe is the busy one); a zero keeps its
// sign through q0.
__device__ __forceinline__ double div_rcp_fast(double d, double c, double y, bool& slow) {
    const double q0 = d * y;
    const unsigned hi = static_cast<unsigned>(__double2hiint(d));
    const unsigned lo = static_cast<unsigned>(__double2loint(d));
    const unsigned e = (hi >> 20) & 0x7ffu;             // biased exponent
    const bool zero = ((hi << 1) | lo) == 0u;
    slow = !zero && (e - 64u) > 1918u;                  // in range: 2^-959 <= |d| < 2^960
    const double r = __fma_rn(-q0, c, d);
    const double q1 = __fma_rn(r, y, q0);
    return zero ? q0 : q1;
}

struct CoefConst {
    static constexpr bool kUnitWE = false, kUnitSN = false;  // legs known to be exactly -1
    static constexpr bool kMaySlow = false;                 // div_by_c_fast may ask for a recompute
    double c, w, e, s, n;
    double inv_c;  // exact reciprocal (valid only when c_pow2)
    int c_pow2;
    int rcp_ok;   // rcp = RN(1/c) usable by div_rcp (c in the checked range)
    double rcp;
    __device__ __forceinline__ void load(int, int, double& C, double& W, double& E, double& S,
                                         double& N) const {
        C = c;
        W = w;
        E = e;
        S = s;
        N = n;
    }
    __device__ __forceinline__ double diag(int, int) const { return c; }
    __device__ __forceinline__ double div_by_c(double r, int, int) const {
        return c_pow2 ? r * inv_c : (rcp_ok ? div_rcp(r, c, rcp) : div_ieee(r, c));
    }
    __device__ __forceinline__ double div_by_c_fast(double r, int i, int j, bool& slow) const {
        slow = false;
        return div_by_c(r, i, j);
    }
};

// Specialised constant rows for the streaming kernels of large levels (chosen on
// the host, so kernels carry no per-point branch). Multiplying by -1 is an exact
// negation and a + (-b) is a - b bit for bit, so a -1 leg is a subtraction.
//   CoefIso   : c a power of two and all four legs -1 (isotropic Poisson: C1, C4):
//               acc = c x - xw - xe - xs - xn, z = r * (1/c) exactly.
//   CoefUnitSN: s = n = -1 (beta = 1: the anisotropic C2, C5), w and e general:
//               acc = c x + w xw + e xe - xs - xn, z by the exact reciprocal
//               (c a power of two) or div_rcp.
struct CoefIso : CoefConst {
    static constexpr bool kUnitWE = true, kUnitSN = true;
    __device__ __forceinline__ double div_by_c(double r, int, int) const { return r * inv_c; }
    __device__ __forceinline__ double div_by_c_fast(double r, int, int, bool& slow) const {
        slow = false;
        return r * inv_c;
    }
};
struct CoefUnitSN : CoefConst {  // rcp_ok is required (host)
    static constexpr bool kUnitSN = true, kMaySlow = true;
    __device__ __forceinline__ double div_by_c(double r, int, int) const { return div_rcp(r, c, rcp); }
    __device__ __forceinline__ double div_by_c_fast(double r, int, int, bool& slow) const {
        return div_rcp_fast(r, c, rcp, slow);
    }
};

struct CoefRowX {
    static constexpr bool kUnitWE = false, kUnitSN = false, kMaySlow = false;
    const double *c, *w, *e, *s, *n;  // length nx each
    const double* rc;                 // RN(1/c[i]) for div_rcp, or null (some c outside the checked range)
    __device__ __forceinline__ void load(int i, int, double& C, double& W, double& E, double& S,
                                         double& N) const {
        C = __ldg(c + i);
        W = __ldg(w + i);
        E = __ldg(e + i);
        S = __ldg(s + i);
        N = __ldg(n + i);
    }
    __device__ __forceinline__ double diag(int i, int) const { return __ldg(c + i); }
    __device__ __forceinline__ double div_by_c(double r, int i, int) const {
        return rc ? div_rcp(r, __ldg(c + i), __ldg(rc + i)) : div_ieee(r, __ldg(c + i));
    }
    __device__ __forceinline__ double div_by_c_fast(double r, int i, int j, bool& slow) const {
        slow = false;
        return div_by_c(r, i, j);
    }
};

struct CoefField {
    static constexpr bool kUnitWE = false, kUnitSN = false, kMaySlow = false;
    const double *c, *w, *e, *s, *n;  // pitched like the level's grid functions
    long long pitch;
    __device__ __forceinline__ void load(int i, int j, double& C, double& W, double& E, double& S,
                                         double& N) const {
        const long long k = (long long)j * pitch + i;
        C = __ldg(c + k);
        W = __ldg(w + k);
        E = __ldg(e + k);
        S = __ldg(s + k);
        N = __ldg(n + k);
    }
    __device__ __forceinline__ double diag(int i, int j) const { return __ldg(c + (long long)j * pitch + i); }
    __device__ __forceinline__ double div_by_c(double r, int i, int j) const {
        return div_ieee(r, __ldg(c + (long long)j * pitch + i));
    }
    __device__ __forceinline__ double div_by_c_fast(double r, int i, int j, bool& slow) const {
        slow = false;
        return div_by_c(r, i, j);
    }
};

// AXES: the general graded / spherical operator computed on the fly from 1-D
// tables of the hierarchy, exactly as assemble builds it (stencil.cpp:77-127):
//   ce = ((alpha fw(x_e)) my) / h_e,   cw = ((alpha fw(x_w)) my) / h_w,
//   cn = ((beta fw(y_n)) mx) / h_n,    cs = ((beta fw(y_s)) mx) / h_s,
//   c = ((ce + cw) + cn) + cs; e, w, n, s = -ce, -cw, -cn, -cs (0 toward the boundary).
// Per column i: ae = alpha fw(x_e), aw, he, hw, mx (the transverse measure) and the
// reciprocals rhe, rhw; per row j: bn, bs, hn, hs, my, rhn, rhs. The host builds
// them with the reference's expressions and checks every coefficient against the
// given arrays bit for bit before choosing this class; the divisions are div_rcp
// (the IEEE quotient). 0 B/DOF instead of FIELD's 40.
struct CoefAxes {
    static constexpr bool kUnitWE = false, kUnitSN = false, kMaySlow = false;
    const double *ae, *aw, *he, *hw, *mx, *rhe, *rhw;  // length nx each
    const double *bn, *bs, *hn, *hs, *my, *rhn, *rhs;  // length ny each
    int nx, ny;
    __device__ __forceinline__ void fluxes(int i, int j, double& ce, double& cw, double& cn, double& cs) const {
        const double yj = __ldg(my + j), xi = __ldg(mx + i);
        ce = div_rcp(__ldg(ae + i) * yj, __ldg(he + i), __ldg(rhe + i));
        cw = div_rcp(__ldg(aw + i) * yj, __ldg(hw + i), __ldg(rhw + i));
        cn = div_rcp(__ldg(bn + j) * xi, __ldg(hn + j), __ldg(rhn + j));
        cs = div_rcp(__ldg(bs + j) * xi, __ldg(hs + j), __ldg(rhs + j));
    }
    __device__ __forceinline__ void load(int i, int j, double& C, double& W, double& E, double& S,
                                         double& N) const {
        double ce, cw, cn, cs;
        fluxes(i, j, ce, cw, cn, cs);
        C = ((ce + cw) + cn) + cs;
        E = i + 1 < nx ? -ce : 0.0;
        W = i > 0 ? -cw : 0.0;
        N = j + 1 < ny ? -cn : 0.0;
        S = j > 0 ? -cs : 0.0;
    }
    __device__ __forceinline__ double diag(int i, int j) const {
        double ce, cw, cn, cs;
        fluxes(i, j, ce, cw, cn, cs);
        return ((ce + cw) + cn) + cs;
    }
    __device__ __forceinline__ double div_by_c(double r, int i, int j) const { return div_ieee(r, diag(i, j)); }
    __device__ __forceinline__ double div_by_c_loaded(double r, double C, int, int) const { return div_ieee(r, C); }
    __device__ __forceinline__ double div_by_c_fast(double r, int i, int j, bool& slow) const {
        slow = false;
        return div_by_c(r, i, j);
    }
};

// Coefficient index clamp for points a streaming kernel evaluates outside the
// grid (halo columns/rows whose results are discarded): ROWX/FIELD tables are
// only read in bounds; for interior points the clamp is the identity.
__device__ __forceinline__ int cix(int v, int n) { return v < 0 ? 0 : (v >= n ? n - 1 : v); }

// y = (A x)(i,j) in the reference's order c, w, e, s, n (stencil.cpp:133-137).
// Cout: the diagonal the stencil used (for the preconditioner's division).
template <class Coef>
__device__ __forceinline__ double stencil_apply_c(const Coef& A, int i, int j, double xc, double xw, double xe,
                                                  double xs, double xn, double& Cout) {
    double C, W, E, S, N;
    A.load(i, j, C, W, E, S, N);
    Cout = C;
    double acc = C * xc;
    if constexpr (Coef::kUnitWE) {
        acc = acc - xw;
        acc = acc - xe;
    } else {
        acc = acc + W * xw;
        acc = acc + E * xe;
    }
    if constexpr (Coef::kUnitSN) {
        acc = acc - xs;
        acc = acc - xn;
    } else {
        acc = acc + S * xs;
        acc = acc + N * xn;
    }
    return acc;
}
template <class Coef>
__device__ __forceinline__ double stencil_apply(const Coef& A, int i, int j, double xc, double xw, double xe,
                                                double xs, double xn) {
    double C;
    return stencil_apply_c(A, i, j, xc, xw, xe, xs, xn, C);
}

// z = r / c given the diagonal c the stencil just loaded: classes that compute
// their coefficients (CoefAxes) divide by it instead of recomputing it.
template <class Coef>
__device__ __forceinline__ auto div_loaded(const Coef& A, double r, double C, int i, int j)
    -> decltype(A.div_by_c_loaded(r, C, i, j)) {
    return A.div_by_c_loaded(r, C, i, j);
}
template <class Coef, class... Ignored>
__device__ __forceinline__ double div_loaded(const Coef& A, double r, double, int i, int j, Ignored...) {
    return A.div_by_c(r, i, j);
}

// ---------------------------------------------------------------------------
// Grid transfers (transfer.cpp). Weights are host-precomputed 1-D tables with
// the reference's own expressions (odd_weight, transfer.cpp:26-28).
// ---------------------------------------------------------------------------
struct Prolong {
    const double* uc;  // coarse grid function (pitched)
    Grid cg;           // coarse grid
    const double* tx;  // per fine column i: odd_weight for odd node index pi=i+1
    const double* ty;  // per fine row j
    __device__ __forceinline__ double cval(int ci, int cj) const {
        return cg.inside(ci, cj) ? __ldg(uc + cg.at(ci, cj)) : 0.0;
    }
    // Fine interior point (i,j) — transfer.cpp:43-68 term for term.
    __device__ __forceinline__ double at(int i, int j) const {
        const int pi = i + 1, pj = j + 1;
        if ((pi & 1) == 0 && (pj & 1) == 0) return cval(pi / 2 - 1, pj / 2 - 1);
        if ((pi & 1) == 1 && (pj & 1) == 0) {
            const int qx = (pi - 1) / 2;
            const double t = __ldg(tx + i);
            return (1.0 - t) * cval(qx - 1, pj / 2 - 1) + t * cval(qx, pj / 2 - 1);
        }
        if ((pi & 1) == 0 && (pj & 1) == 1) {
            const int qy = (pj - 1) / 2;
            const double t = __ldg(ty + j);
            return (1.0 - t) * cval(pi / 2 - 1, qy - 1) + t * cval(pi / 2 - 1, qy);
        }
        const int qx = (pi - 1) / 2, qy = (pj - 1) / 2;
        const double tX = __ldg(tx + i), tY = __ldg(ty + j);
        double v = (1.0 - tX) * (1.0 - tY) * cval(qx - 1, qy - 1);
        v = v + tX * (1.0 - tY) * cval(qx, qy - 1);
        v = v + (1.0 - tX) * tY * cval(qx - 1, qy);
        v = v + tX * tY * cval(qx, qy);
        return v;
    }
};

struct RestrictW {
    // per coarse column P (0-based): west/east odd weights and the 1-D sum sx;
    // per coarse row Q likewise (transfer.cpp:80-85)
    const double *wxw, *wxe, *sx, *wys, *wyn, *sy;
};

// Full-weighting restriction of fine values f at coarse (P,Q), 9 terms in the
// reference's dj-outer / di-inner order from acc = 0 (transfer.cpp:86-97).
// `F(di, dj)` returns the fine value at fine interior (2P+1+di, 2Q+1+dj).
template <class F>
__device__ __forceinline__ double restrict_at(const RestrictW& rw, int P, int Q, F&& f) {
    const double wx[3] = {__ldg(rw.wxw + P), 1.0, __ldg(rw.wxe + P)};
    const double wy[3] = {__ldg(rw.wys + Q), 1.0, __ldg(rw.wyn + Q)};
    double acc = 0.0;
#pragma unroll
    for (int dj = -1; dj <= 1; ++dj)
#pragma unroll
        for (int di = -1; di <= 1; ++di) acc = acc + wx[di + 1] * wy[dj + 1] * f(di, dj);
    return acc / (__ldg(rw.sx + P) * __ldg(rw.sy + Q));
}

}  // namespace gmg_dev
