// Two-columns-per-thread variant of the row-streaming Jacobi smoother
// (march.cuh). Same pipeline — M fused Jacobi steps, one __syncthreads per row,
// register windows for vertical neighbours, a double-buffered shared row per
// level for horizontal ones — but every thread owns an even-aligned column
// pair, so loads and stores are 16-byte vectors and the per-row overhead
// (index math, guards, prefetch rotation, barrier) is paid once per two points.
// Bit-identical to k_smooth: each point is the same expression sequence.
#pragma once

#include "march.cuh"

namespace gmg_dev {

// (i even) pair at row j, zeros outside the interior
__device__ __forceinline__ double2 ld_pair(const double* a, const Grid& g, int i, int j) {
    double2 r = make_double2(0.0, 0.0);
    if (!g.row_ok(j)) return r;
    const double* p = a + g.at(i, j);
    if (i >= 0 && i + 1 < g.nx) return __ldg(reinterpret_cast<const double2*>(p));
    if (i >= 0 && i < g.nx) r.x = __ldg(p);
    if (i + 1 >= 0 && i + 1 < g.nx) r.y = __ldg(p + 1);
    return r;
}

struct Src2Zero {
    static constexpr const char* kProfName = "smooth(from 0)";
    static constexpr double kBytesPerDof = 16.0;
    struct Raw {};
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ Raw fetch(int, int) const { return Raw{}; }
    __device__ __forceinline__ double2 make(const Raw&, int, int) const { return make_double2(0.0, 0.0); }
};

struct Src2U {
    static constexpr const char* kProfName = "smooth(from u)";
    static constexpr double kBytesPerDof = 24.0;
    const double* u;
    Grid g;
    struct Raw {
        double2 v;
    };
    __device__ __forceinline__ void prepare(int) {}
    __device__ __forceinline__ Raw fetch(int i, int j) const { return Raw{ld_pair(u, g, i, j)}; }
    __device__ __forceinline__ double2 make(const Raw& r, int, int) const { return r.v; }
};

// Bilinear prolongation for the pair (i even: node i+1 odd -> interpolated
// between coarse columns i/2-1 and i/2; node i+2 even -> coarse column i/2),
// transfer.cpp:43-68 term for term.
struct Pair2Raw {
    double a, b, c, d, ty;  // (m-1,r0) (m,r0) (m-1,r1) (m,r1)
};
__device__ __forceinline__ Pair2Raw prolong2_fetch(const Prolong& P, int i, int j, int fny) {
    Pair2Raw r{0.0, 0.0, 0.0, 0.0, 0.0};
    if (P.cg.per) {  // periodic y (fine rows 2 ny_c): wrap first, the coarse rows wrap in cval
        j %= fny;
        if (j < 0) j += fny;
    }
    if (j < 0 || j >= fny) return r;
    const int m = i / 2;  // i even (may be negative only on the halo, handled by cval)
    const int pj = j + 1;
    const int r0 = (pj & 1) ? (pj - 1) / 2 - 1 : pj / 2 - 1;
    r.a = P.cval(m - 1, r0);
    r.b = P.cval(m, r0);
    if (pj & 1) {
        r.c = P.cval(m - 1, r0 + 1);
        r.d = P.cval(m, r0 + 1);
        r.ty = __ldg(P.ty + j);
    }
    return r;
}
__device__ __forceinline__ double2 prolong2_make(const Pair2Raw& r, int i, int j, int fnx, double tX) {
    double v0, v1;
    if (((j + 1) & 1) == 0) {  // even node row: one coarse row
        v0 = (1.0 - tX) * r.a + tX * r.b;
        v1 = r.b;
    } else {
        const double tY = r.ty;
        v0 = (1.0 - tX) * (1.0 - tY) * r.a;
        v0 = v0 + tX * (1.0 - tY) * r.b;
        v0 = v0 + (1.0 - tX) * tY * r.c;
        v0 = v0 + tX * tY * r.d;
        v1 = (1.0 - tY) * r.b + tY * r.d;
    }
    return make_double2((i >= 0 && i < fnx) ? v0 : 0.0, (i + 1 >= 0 && i + 1 < fnx) ? v1 : 0.0);
}

struct Src2Prolong {
    static constexpr const char* kProfName = "smooth(from P e)";
    static constexpr double kBytesPerDof = 18.0;
    Prolong P;
    int fnx, fny;
    double tX;
    using Raw = Pair2Raw;
    __device__ __forceinline__ void prepare(int i) { tX = (i >= 0 && i < fnx) ? __ldg(P.tx + i) : 0.0; }
    __device__ __forceinline__ Raw fetch(int i, int j) const { return prolong2_fetch(P, i, j, fny); }
    __device__ __forceinline__ double2 make(const Raw& r, int i, int j) const {
        return prolong2_make(r, i, j, fnx, tX);
    }
};

struct Src2Correct {  // u + omega * P uc (axpy(wl, corr, u), cycle.cpp:93-96)
    static constexpr const char* kProfName = "smooth(u + w P uc)";
    static constexpr double kBytesPerDof = 26.0;
    const double* u;
    Grid g;
    Prolong P;
    double omega;
    double tX;
    struct Raw {
        double2 u;
        Pair2Raw p;
    };
    __device__ __forceinline__ void prepare(int i) { tX = (i >= 0 && i < g.nx) ? __ldg(P.tx + i) : 0.0; }
    __device__ __forceinline__ Raw fetch(int i, int j) const {
        Raw r;
        r.u = ld_pair(u, g, i, j);
        r.p = prolong2_fetch(P, i, j, g.ny);
        return r;
    }
    __device__ __forceinline__ double2 make(const Raw& r, int i, int j) const {
        const double2 c = prolong2_make(r.p, i, j, g.nx, tX);
        return make_double2(r.u.x + omega * c.x, r.u.y + omega * c.y);
    }
};

// Launch: grid (ceil(nx / (2TW - 2H)), ceil(ny / seg)), block TW; H = M rounded up to even.
template <int M, int TW, int PF, class Coef, class Src>
__global__ void __launch_bounds__(TW) k_smooth2(Grid fg, Coef A, Src src, OmegaSrc om, const double* __restrict__ g,
                                                double* __restrict__ out, double omega_damp, int seg) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    constexpr int H = (M + 1) & ~1;
    constexpr int OUTW = 2 * TW - 2 * H;
    constexpr int ML = M > 0 ? M : 1;
    __shared__ double2 sh[2][ML][TW];

    const int t = threadIdx.x;
    const int i = blockIdx.x * OUTW - H + 2 * t;  // even
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    const bool in0 = i >= 0 && i < fg.nx, in1 = i + 1 >= 0 && i + 1 < fg.nx;
    const bool owner = 2 * t >= H && 2 * t < 2 * TW - H;

    src.prepare(i);
    if constexpr (std::is_same<Src, Src2Correct>::value) {
        src.omega = om.get(blockIdx.x == 0 && blockIdx.y == 0 && t == 0);
    }

    double2 win[ML][3];
    double2 gring[ML];
#pragma unroll
    for (int l = 0; l < ML; ++l) {
        win[l][0] = win[l][1] = win[l][2] = make_double2(0.0, 0.0);
        gring[l] = make_double2(0.0, 0.0);
    }

    const int Jbeg = j0 - M;
    const int Jend = j1 - 1 + M;
    typename Src::Raw q[PF];
    double2 gq[PF];
#pragma unroll
    for (int p = 0; p < PF; ++p) {
        q[p] = src.fetch(i, Jbeg + p);
        gq[p] = M > 0 ? ld_pair(g, fg, i, Jbeg + p) : make_double2(0.0, 0.0);
    }
    for (int Jb = Jbeg; Jb <= Jend; Jb += PF) {
#pragma unroll
        for (int p = 0; p < PF; ++p) {
            const int J = Jb + p;
            if (J > Jend) break;  // uniform
            const typename Src::Raw raw = q[p];
            const double2 gnew = gq[p];
            q[p] = src.fetch(i, J + PF);
            gq[p] = M > 0 ? ld_pair(g, fg, i, J + PF) : make_double2(0.0, 0.0);
            const bool row_in = fg.row_ok(J);
            double2 nv = row_in ? src.make(raw, i, fg.wrap(J)) : make_double2(0.0, 0.0);
            if (!in0) nv.x = 0.0;
            if (!in1) nv.y = 0.0;
            if constexpr (M == 0) {
                if (owner && J >= j0 && J < j1) {
                    if (in0 && in1) {
                        *reinterpret_cast<double2*>(out + fg.at(i, J)) = nv;
                    } else {
                        if (in0) out[fg.at(i, J)] = nv.x;
                        if (in1) out[fg.at(i + 1, J)] = nv.y;
                    }
                }
            } else {
                const int pb = (J - 1) & 1, cb = J & 1;
#pragma unroll
                for (int l = 0; l < M; ++l) {
                    win[l][0] = win[l][1];
                    win[l][1] = win[l][2];
                    win[l][2] = nv;
                    sh[cb][l][t] = nv;
                    const int R = J - l - 1;
                    const double xl = t > 0 ? sh[pb][l][t - 1].y : 0.0;
                    const double xr = t < TW - 1 ? sh[pb][l][t + 1].x : 0.0;
                    const double2 c = win[l][1], dn = win[l][0], up = win[l][2];
                    const int Rc = fg.per ? fg.wrap(R) : cix(R, fg.ny);
                    const double y0 = jacobi_point(A, cix(i, fg.nx), Rc, c.x, xl, c.y, dn.x, up.x, gring[l].x, omega_damp);
                    const double y1 =
                        jacobi_point(A, cix(i + 1, fg.nx), Rc, c.y, c.x, xr, dn.y, up.y, gring[l].y, omega_damp);
                    const bool rin = fg.row_ok(R);
                    nv = make_double2((rin && in0) ? y0 : 0.0, (rin && in1) ? y1 : 0.0);
                }
                const int RM = J - M;
                if (owner && RM >= j0 && RM < j1) {
                    if (in0 && in1) {
                        *reinterpret_cast<double2*>(out + fg.at(i, RM)) = nv;
                    } else {
                        if (in0) out[fg.at(i, RM)] = nv.x;
                        if (in1) out[fg.at(i + 1, RM)] = nv.y;
                    }
                }
#pragma unroll
                for (int l = ML - 1; l > 0; --l) gring[l] = gring[l - 1];
                gring[0] = gnew;
                __syncthreads();
            }
        }
    }
}

}  // namespace gmg_dev

namespace gmg_dev {

// ---------------------------------------------------------------------------
// cp.async helpers of the warp-strip kernels (march4.cuh): 16- and 8-byte copies
// into shared memory, zero-filled beyond src_bytes (rows/columns outside the
// interior read nothing and land as +0).
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cpa16(void* smem, const void* gmem, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cpa8(void* smem, const void* gmem, int src_bytes) {
    const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(sa), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;"); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N));
}

// stage one coarse value (zeros outside the coarse interior). The warp-strip
// kernels march non-periodic levels only (Lev::strips), so no row wrap here.
__device__ __forceinline__ void stage_coarse(double* dst, const double* uc, const Grid& cg, int ci, int cj) {
    const bool in = ci >= 0 && ci < cg.nx && cj >= 0 && cj < cg.ny;
    cpa8(dst, in ? uc + (long long)cj * cg.pitch + ci : uc, in ? 8 : 0);
}

enum SrcKind3 { K3_ZERO = 0, K3_U = 1, K3_PROLONG = 2, K3_CORRECT = 3 };

}  // namespace gmg_dev
