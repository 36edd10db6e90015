// k_smooth4: the fused M-step Jacobi smoother for large levels, built to cut
// instructions per point (the row-streaming kernels before it were issue-bound
// at ~60 instructions per point update).
//
//   * Every warp is an independent column strip of 128 columns (4 per lane),
//     H = M rounded up to even halo columns on each side; horizontal neighbours
//     come from the adjacent lanes by shuffles, so there is no block barrier
//     and no shared-memory exchange in the row loop.
//   * Inputs (u, g, and the two coarse rows a prolongation needs) stream
//     through per-warp shared-memory rings filled by cp.async (zero-fill
//     outside the interior), 3 rows ahead.
//   * The row loop is unrolled by 3 so the per-level 3-row register windows
//     rotate by renaming instead of moves.
//   * Domain masks only where a warp strip or a row touches the boundary
//     (warp-uniform branches).
// Arithmetic per point is jacobi_point (march.cuh) on the same operands as the
// reference, so results are bit-identical to the other smoother kernels.
#pragma once

#include "march.cuh"
#include "march2.cuh"

namespace gmg_dev {

constexpr int kS4W = 4;  // warps per CTA (independent strips)
// CTAs per SM the register budgets are sized for. These kernels are latency-bound: occupancy
// buys more than the instructions a tighter register budget costs (profiles/r02_summary.md).
#ifndef GMG_S4_SPLIT_MINM
#define GMG_S4_SPLIT_MINM 3  // fused step counts from which the march is split into interior / boundary paths
#endif
#ifndef GMG_S4_GSMEM_MINM
#define GMG_S4_GSMEM_MINM 3   // fused step counts from which the right-hand side is re-read from a deeper ring
#endif
#ifndef GMG_S4_GRING_ALL
#define GMG_S4_GRING_ALL 0  // 1: the 3-slot register ring for the right-hand side on the general path too
#endif
#ifndef GMG_S4_TYPRE
#define GMG_S4_TYPRE 1  // 1: the row's prolongation weight fetched one row ahead
#endif
#ifndef GMG_S4_M3_MINB
#define GMG_S4_M3_MINB 4  // CTAs per SM of the 3-/4-step kernels without a streamed iterate (their smem allows 4)
#endif
#ifndef GMG_S4_MINB
#define GMG_S4_MINB 4
#endif
#ifndef GMG_R4_MINB
#define GMG_R4_MINB 4
#endif
#ifndef GMG_O4_MINB
#define GMG_O4_MINB 4
#endif

template <int SK, int M>
struct Smooth4Smem {
    static constexpr bool HAS_U = SK == K3_U || SK == K3_CORRECT;
    static constexpr bool HAS_C = SK == K3_PROLONG || SK == K3_CORRECT;
    // GSMEM (M >= 3): the right-hand side of the M rows the fused steps work on is re-read
    // from a deeper ring instead of riding in registers (a 4 x M doubles window): at their
    // 168-register budget the 3- and 4-step kernels had spilled loop invariants and reloaded
    // them every row (25% of the stall samples of C5's finest post-smoother; -1.6% per C5 cycle)
    static constexpr bool GSMEM = M >= GMG_S4_GSMEM_MINM;
    // ring depth: rows in flight per warp = D-1 (a deeper ring, 8, for the sources with one
    // streamed array measured 25% slower in the cycle)
#ifndef GMG_S4_DEEP
#define GMG_S4_DEEP 4
#endif
    static constexpr int D = HAS_U ? 4 : GMG_S4_DEEP;
    // [slot][half][lane]: lane's columns 4l..4l+1 in half 0, 4l+2..4l+3 in half 1
    // (16-B lane stride: conflict-free 128-bit accesses)
    static constexpr int GD = GSMEM ? 8 : D;  // rows J-M .. J+D-1 live at once
    double2 g[GD][2][32];
    double2 u[HAS_U ? D : 1][2][32];
    double c[HAS_C ? D : 1][68];  // coarse rows, slot = coarse row & (D-1)
};

// The march of one warp strip. BND = false: the strip and every row it touches
// (staged rows included) lie inside the domain with both coarse parents present,
// so no bounds predicate, zero-fill byte count or masking select is issued — the
// common case (all but the first/last strips and row segments). BND = true: the
// general path with domain masks. Same arithmetic per point in both.
template <int M, int SK, class Coef, bool BND>
__device__ __forceinline__ void smooth4_march(Smooth4Smem<SK, M>& S, const Grid& fg, const Coef& A,
                                              const double* __restrict__ u, const Prolong& P, double omega,
                                              const double* __restrict__ g, double* __restrict__ out,
                                              double omega_damp, int i0, int j0, int j1) {
    using SM = Smooth4Smem<SK, M>;
    constexpr bool HAS_U = SM::HAS_U, HAS_C = SM::HAS_C, GSMEM = SM::GSMEM;
    constexpr int D = SM::D, GD = SM::GD;
    constexpr int H = (M + 1) & ~1;  // halo columns, even: 16-B aligned strips
    constexpr int ML = M > 0 ? M : 1;
    // coarse columns are staged from the even column mS = m0 - COFF (16-B pairs)
    constexpr int COFF = (H == 2) ? 0 : 1;
    const int lane = threadIdx.x & 31;
    const int i = i0 + 4 * lane;
    const int nx = fg.nx, ny = fg.ny;
    const bool edge = BND && (i0 < 0 || i0 + 128 > nx);
    bool cin[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) cin[k] = !BND || (i + k >= 0 && i + k < nx);
    const int m0 = i0 / 2 - 1;  // first coarse column needed (i0 even)
    const double tX0 = (HAS_C && cin[0]) ? __ldg(P.tx + i) : 0.0;
    const double tX2 = (HAS_C && cin[2]) ? __ldg(P.tx + i + 2) : 0.0;

    const int Jbeg = j0 - M;
    const int Jend = j1 - 1 + M;
    auto slot_of = [](int J) { return (J + 8) & (D - 1); };
    auto chunk_bytes = [&](int c) { return (c >= 0 && c < nx) ? (c + 1 < nx ? 16 : 8) : 0; };
    const int cb0 = BND ? chunk_bytes(i) : 16, cb1 = BND ? chunk_bytes(i + 2) : 16;
    // running pointers of the next row to stage / the next row to store
    const long long pitch = fg.pitch;
    long long soff = (long long)Jbeg * pitch + i;
    long long roff = soff;
    const long long cpitch = P.cg.pitch;
    auto stage_crow = [&](int q) {
        double* dst = S.c[(q + 8) & (D - 1)];
        if constexpr (BND) {
            stage_coarse(dst + COFF + 2 * lane, P.uc, P.cg, m0 + 2 * lane, q);
            stage_coarse(dst + COFF + 2 * lane + 1, P.uc, P.cg, m0 + 2 * lane + 1, q);
            if (lane == 0) stage_coarse(dst + COFF + 64, P.uc, P.cg, m0 + 64, q);
        } else {
            // all of [m0, m0 + 64] x {q} is inside the coarse grid: aligned pairs
            const double* src = P.uc + (long long)q * cpitch + (m0 - COFF);
            cpa16(dst + 2 * lane, src + 2 * lane, 16);
            if (lane == 0) cpa8(dst + COFF + 64, src + COFF + 64, 8);
            if (COFF && lane == 1) cpa8(dst + 64, src + 64, 8);
        }
    };
    auto gslot_of = [](int J) { return (J + 8) & (GD - 1); };
    auto stage = [&](int J) {
        const int sl = slot_of(J), gsl = gslot_of(J);
        const bool row_in = !BND || (J >= 0 && J < ny);
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            if constexpr (BND) {
                const int bytes = row_in ? (h ? cb1 : cb0) : 0;
                const long long o = bytes ? soff + 2 * h : 0;
                cpa16(&S.g[gsl][h][lane], g + o, bytes);
                if constexpr (HAS_U) cpa16(&S.u[sl][h][lane], u + o, bytes);
            } else {
                cpa16(&S.g[gsl][h][lane], g + soff + 2 * h, 16);
                if constexpr (HAS_U) cpa16(&S.u[sl][h][lane], u + soff + 2 * h, 16);
            }
        }
        soff += pitch;
        if constexpr (HAS_C) {
            // fine row J needs coarse rows floor(J/2)-1 (J even only) and floor(J/2):
            // a new coarse row every other fine row, staged once
            if (((J + 8) & 1) == 0) stage_crow((J + 8) / 2 - 4);
        }
        cpa_commit();
    };
#if GMG_S4_TYPRE
    double ty_cur = (HAS_C && ((Jbeg + 1) & 1) && Jbeg >= 0 && Jbeg < ny) ? __ldg(P.ty + Jbeg) : 0.0;
#endif
    // the source value of row J for this lane's 4 columns (zero outside the interior)
    auto source = [&](int J, int sl, double (&nv)[4]) {
#if GMG_S4_TYPRE
        double tyJ = 0.0;
        if constexpr (HAS_C) {  // this row's weight was fetched an iteration ago; fetch the next row's
            tyJ = ty_cur;
            const int Jn = J + 1;
            ty_cur = (((Jn + 1) & 1) && Jn >= 0 && Jn < ny) ? __ldg(P.ty + Jn) : 0.0;
        }
#endif
#pragma unroll
        for (int k = 0; k < 4; ++k) nv[k] = 0.0;
        if (BND && (J < 0 || J >= ny)) return;
        if constexpr (SK == K3_U) {
            const double2 a = S.u[sl][0][lane];
            const double2 b = S.u[sl][1][lane];
            nv[0] = a.x;
            nv[1] = a.y;
            nv[2] = b.x;
            nv[3] = b.y;
        }
        if constexpr (HAS_C) {
            const int qf = (J + 8) / 2 - 4;  // floor(J/2)
            const bool even = ((J + 8) & 1) == 0;
            const double* ca = &S.c[((even ? qf - 1 : qf) + 8) & (D - 1)][COFF + 2 * lane];
            const double* cb = &S.c[(qf + 8) & (D - 1)][COFF + 2 * lane];
            Pair2Raw r;
#if GMG_S4_TYPRE
            r.ty = tyJ;
#else
            r.ty = ((J + 1) & 1) ? __ldg(P.ty + J) : 0.0;
#endif
            r.a = ca[0];
            r.b = ca[1];
            r.c = cb[0];
            r.d = cb[1];
            const double2 p0 = prolong2_make(r, BND ? i : 0, J, BND ? nx : 4, tX0);
            r.a = ca[1];
            r.b = ca[2];
            r.c = cb[1];
            r.d = cb[2];
            const double2 p1 = prolong2_make(r, BND ? i + 2 : 0, J, BND ? nx : 4, tX2);
            if constexpr (SK == K3_PROLONG) {
                nv[0] = p0.x;
                nv[1] = p0.y;
                nv[2] = p1.x;
                nv[3] = p1.y;
            } else {
                const double2 a = S.u[sl][0][lane];
                const double2 b = S.u[sl][1][lane];
                nv[0] = a.x + omega * p0.x;
                nv[1] = a.y + omega * p0.y;
                nv[2] = b.x + omega * p1.x;
                nv[3] = b.y + omega * p1.y;
            }
        }
        if (edge) {
#pragma unroll
            for (int k = 0; k < 4; ++k)
                if (!cin[k]) nv[k] = 0.0;
        }
    };
    // lanes 0 and 31 hold the halo columns: with H = 2 each still produces one pair
    const bool st_lo = lane > 0 && (H == 2 || lane < 31);   // columns 4l, 4l+1
    const bool st_hi = lane < 31 && (H == 2 || lane > 0);   // columns 4l+2, 4l+3
    auto store = [&](long long off, const double (&v)[4]) {
        double* o = out + off;
        if constexpr (!BND && H > 0) {
            if (st_lo) *reinterpret_cast<double2*>(o) = make_double2(v[0], v[1]);
            if (st_hi) *reinterpret_cast<double2*>(o + 2) = make_double2(v[2], v[3]);
            return;
        }
        if (!edge && lane > 0 && lane < 31) {  // all four columns are produced here
            *reinterpret_cast<double2*>(o) = make_double2(v[0], v[1]);
            *reinterpret_cast<double2*>(o + 2) = make_double2(v[2], v[3]);
            return;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int c = 4 * lane + k;
            if (c >= H && c < 128 - H && cin[k]) o[k] = v[k];
        }
    };

    if constexpr (GSMEM) {
        // rows before Jbeg are never staged: their slots read as zero right-hand sides
#pragma unroll
        for (int q = 0; q < GD; ++q) {
            S.g[q][0][lane] = make_double2(0.0, 0.0);
            S.g[q][1][lane] = make_double2(0.0, 0.0);
        }
        __syncwarp();
    }
    if constexpr (HAS_C) {
        // coarse rows of fine rows Jbeg .. Jbeg+D-2 that stage() itself will not fetch
        // Jbeg even: floor(Jbeg/2)-1 (its pair partner comes with stage(Jbeg));
        // Jbeg odd: floor(Jbeg/2)
        const int qf = (Jbeg + 8) / 2 - 4;
        stage_crow(((Jbeg + 8) & 1) ? qf : qf - 1);
    }
#pragma unroll
    for (int p = 0; p < D - 1; ++p) stage(Jbeg + p);
    cpa_wait<D - 2>();
    __syncwarp();

    // register windows: w[l] = rows J-l, J-l-1, J-l-2 of step l's input; gw = the
    // right-hand side of rows J, J-1, .. J-M. Slots are named by PH = (J - Jbeg) mod 3
    // (w) so the unrolled-by-3 row loop rotates them by renaming; gw is a 3-slot ring
    // as well when M <= 2, else a shifted window.
    double w[ML][3][4];
    constexpr bool GRING = M <= 2 && (!BND || GMG_S4_GRING_ALL);
    constexpr int GS = GSMEM ? 1 : (GRING ? 3 : ML + 1);
    double gw[GS][4];
#pragma unroll
    for (int l = 0; l < ML; ++l)
#pragma unroll
        for (int k = 0; k < 4; ++k) w[l][0][k] = w[l][1][k] = w[l][2][k] = 0.0;
#pragma unroll
    for (int q = 0; q < GS; ++q)
#pragma unroll
        for (int k = 0; k < 4; ++k) gw[q][k] = 0.0;

    // one row J; PH = (J - Jbeg) mod 3 names the window slots statically
    auto row = [&](int J, auto ph) {
        constexpr int PH = decltype(ph)::value;
        stage(J + D - 1);  // into the slot of row J-1, read last iteration
        const int sl = slot_of(J);
        const long long rJ = roff;  // offset of row J in this lane's columns
        roff += pitch;
        double nv[4];
        source(J, sl, nv);
        if constexpr (M == 0) {
            if (J >= j0 && J < j1) store(rJ, nv);
        } else {
            // g of row J into its slot (ring: slot PH; shifted window: slot 0 after the shift)
            constexpr int gJ = GRING ? PH : 0;
            if constexpr (!GSMEM) {  // (GSMEM: every step reads its row from the ring below)
                if constexpr (!GRING) {
#pragma unroll
                    for (int q = GS - 1; q > 0; --q)
#pragma unroll
                        for (int k = 0; k < 4; ++k) gw[q][k] = gw[q - 1][k];
                }
                const double2 a = S.g[gslot_of(J)][0][lane];
                const double2 b = S.g[gslot_of(J)][1][lane];
                gw[gJ][0] = a.x;
                gw[gJ][1] = a.y;
                gw[gJ][2] = b.x;
                gw[gJ][3] = b.y;
            }
#pragma unroll
            for (int l = 0; l < M; ++l) {
                const int sn = (PH - l + 30) % 3;      // newest row J-l
                const int sc = (PH - l - 1 + 30) % 3;  // centre row J-l-1
                const int sd = (PH - l - 2 + 30) % 3;  // row J-l-2
                const int gs = GRING ? (PH - l - 1 + 30) % 3 : l + 1;  // g of row J-l-1
#pragma unroll
                for (int k = 0; k < 4; ++k) w[l][sn][k] = nv[k];
                const int R = J - l - 1;
                double gk[4];
                if constexpr (GSMEM) {
                    const double2 a = S.g[gslot_of(R)][0][lane];
                    const double2 b = S.g[gslot_of(R)][1][lane];
                    gk[0] = a.x;
                    gk[1] = a.y;
                    gk[2] = b.x;
                    gk[3] = b.y;
                } else {
#pragma unroll
                    for (int k = 0; k < 4; ++k) gk[k] = gw[gs][k];
                }
                const double xl = __shfl_up_sync(0xffffffffu, w[l][sc][3], 1);
                const double xr = __shfl_down_sync(0xffffffffu, w[l][sc][0], 1);
                double y[4];
                bool slow[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double xw = k == 0 ? xl : w[l][sc][k - 1];
                    const double xe = k == 3 ? xr : w[l][sc][k + 1];
                    y[k] = jacobi_point_fast(A, cix(i + k, fg.nx), cix(R, fg.ny), w[l][sc][k], xw, xe, w[l][sd][k],
                                             w[l][sn][k], gk[k], omega_damp, slow[k]);
                }
                if constexpr (Coef::kMaySlow) {
                    // one warp vote per fused step and row; the exact division only where asked
                    if (__any_sync(0xffffffffu, slow[0] | slow[1] | slow[2] | slow[3])) {
                        for (int k = 0; k < 4; ++k) {
                            if (!slow[k]) continue;
                            const double xw = k == 0 ? xl : w[l][sc][k - 1];
                            const double xe = k == 3 ? xr : w[l][sc][k + 1];
                            y[k] = jacobi_point(A, cix(i + k, fg.nx), cix(R, fg.ny), w[l][sc][k], xw, xe,
                                                w[l][sd][k], w[l][sn][k], gk[k], omega_damp);
                        }
                    }
                }
                if constexpr (BND) {
                    if (R < 0 || R >= ny) {
#pragma unroll
                        for (int k = 0; k < 4; ++k) y[k] = 0.0;
                    } else if (edge) {
#pragma unroll
                        for (int k = 0; k < 4; ++k)
                            if (!cin[k]) y[k] = 0.0;
                    }
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) nv[k] = y[k];
            }
            const int RM = J - M;
            if (RM >= j0 && (!BND || RM < j1)) store(rJ - M * pitch, nv);
        }
        cpa_wait<D - 2>();  // row J+1 has landed (for this lane)
        __syncwarp();       // ... for every lane; slot of row J is free again
    };
    if constexpr (BND && M >= GMG_S4_SPLIT_MINM) {
        // the rare path (first/last strips and row segments) stays small in the instruction
        // cache: one row body, the windows shifted by moves (slot names of PH = 0)
#pragma unroll 1
        for (int J = Jbeg; J <= Jend; ++J) {
            row(J, std::integral_constant<int, 0>{});
#pragma unroll
            for (int l = 0; l < M; ++l) {
                const int sn = (30 - l) % 3, sc = (29 - l) % 3, sd = (28 - l) % 3;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    w[l][sd][k] = w[l][sc][k];
                    w[l][sc][k] = w[l][sn][k];
                }
            }
        }
    } else {
        for (int J = Jbeg; J <= Jend; J += 3) {
            row(J, std::integral_constant<int, 0>{});
            if (J + 1 > Jend) break;
            row(J + 1, std::integral_constant<int, 1>{});
            if (J + 2 > Jend) break;
            row(J + 2, std::integral_constant<int, 2>{});
        }
    }
    cpa_wait<0>();
}

template <int M, int SK, class Coef>
__global__ void __launch_bounds__(kS4W * 32, (M <= 2 ? GMG_S4_MINB
                                                         : ((SK == K3_ZERO || SK == K3_PROLONG) ? GMG_S4_M3_MINB : 3)))
    k_smooth4(Grid fg, Coef A, const double* __restrict__ u, Prolong P, OmegaSrc om, const double* __restrict__ g,
              double* __restrict__ out, double omega_damp, int seg) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    using SM = Smooth4Smem<SK, M>;
    constexpr int H = (M + 1) & ~1;  // halo columns, even: 16-B aligned strips
    constexpr int OW = 128 - 2 * H;  // columns each strip produces
    extern __shared__ __align__(16) unsigned char sm4raw[];
    SM& S = reinterpret_cast<SM*>(sm4raw)[threadIdx.x >> 5];

    const int strip = blockIdx.x * kS4W + (threadIdx.x >> 5);
    const int i0 = strip * OW - H;
    if (i0 + H >= fg.nx) return;  // warp-uniform; the kernel has no block barriers
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    double omega = 0.0;
    if constexpr (SK == K3_CORRECT) omega = om.get(blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x == 0);
    // interior: the strip's 128 columns, every row it stages (j0-M .. j1-1+M+D-1) and their
    // coarse parents (rows >= 2 and <= ny-3 have both) are inside the domain
    bool interior = i0 >= 4 && i0 + 128 <= fg.nx && j0 - M >= 2 && j1 + M + SM::D <= fg.ny - 2;
    if constexpr (SM::HAS_C)  // ... which the nested grids guarantee (fine n = 2 coarse n + 1); checked anyway
        interior = interior && i0 / 2 + 63 < P.cg.nx && (j1 + M + SM::D) / 2 < P.cg.ny;
    // The split pays for M >= 3 (C5's 3+3: -18% on the finest level; the one-path loop is
    // instruction-cache bound there). For M <= 2 the single general loop measured faster
    // (C4 finest post-smoother 0.336 vs 0.354 ms), so every strip takes it.
    if (M >= GMG_S4_SPLIT_MINM && interior)
        smooth4_march<M, SK, Coef, false>(S, fg, A, u, P, omega, g, out, omega_damp, i0, j0, j1);
    else
        smooth4_march<M, SK, Coef, true>(S, fg, A, u, P, omega, g, out, omega_damp, i0, j0, j1);
}

// ---------------------------------------------------------------------------
// k_resid4: residual d = g - A x0 (stencil.cpp:148-153) of x0 = x or x + e
// (fcycle_pass's x + 1.0*e, cycle.cpp:139-140), optionally storing d and x0,
// and optionally the full-weighting restriction of d into the coarse right-hand
// side (transfer.cpp:72-101) — one pass, the warp-strip layout of k_smooth4.
// ---------------------------------------------------------------------------
template <bool SUM>
struct Resid4Smem {
    static constexpr int D = 4;
    double2 x[D][2][32];
    double2 e[SUM ? D : 1][2][32];
    double2 g[D][2][32];
};

template <bool SUM, class Coef>
__global__ void __launch_bounds__(kS4W * 32, GMG_R4_MINB)
    k_resid4(Grid fg, Coef A, const double* __restrict__ x, const double* __restrict__ e,
             const double* __restrict__ g, double* __restrict__ dout, double* __restrict__ x0out, Grid cg,
             RestrictW rw, double* __restrict__ gc, int seg) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    using SM = Resid4Smem<SUM>;
    constexpr int D = SM::D;
    constexpr int H = 2;
    constexpr int OW = 128 - 2 * H;
    extern __shared__ __align__(16) unsigned char r4raw[];
    SM& S = reinterpret_cast<SM*>(r4raw)[threadIdx.x >> 5];
    const bool STORE_D = dout != nullptr, STORE_X0 = x0out != nullptr, RESTRICT = gc != nullptr;

    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kS4W + (threadIdx.x >> 5);
    const int i0 = strip * OW - H;
    if (i0 + H >= fg.nx) return;  // warp-uniform; no block barriers below
    const int i = i0 + 4 * lane;
    const int nx = fg.nx, ny = fg.ny;
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    const bool edge = i0 < 0 || i0 + 128 > nx;
    bool cin[4], cout_[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cin[k] = i + k >= 0 && i + k < nx;
        const int c = 4 * lane + k;
        cout_[k] = cin[k] && c >= H && c < 128 - H;
    }
    auto chunk_bytes = [&](int c) { return (c >= 0 && c < nx) ? (c + 1 < nx ? 16 : 8) : 0; };
    const int cb0 = chunk_bytes(i), cb1 = chunk_bytes(i + 2);
    const long long pitch = fg.pitch;
    // d is exact from row Jbeg+1 on; the restriction needs it from row j0-1
    const int Jbeg = j0 - 2;
    const int Jend = j1 + 1;
    long long soff = (long long)Jbeg * pitch + i;
    long long roff = soff;
    auto slot_of = [](int J) { return (J + 8) & (D - 1); };
    auto stage = [&](int J) {
        const int sl = slot_of(J);
        const bool row_in = J >= 0 && J < ny;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int bytes = row_in ? (h ? cb1 : cb0) : 0;
            const long long o = bytes ? soff + 2 * h : 0;
            cpa16(&S.x[sl][h][lane], x + o, bytes);
            if constexpr (SUM) cpa16(&S.e[sl][h][lane], e + o, bytes);
            cpa16(&S.g[sl][h][lane], g + o, bytes);
        }
        soff += pitch;
        cpa_commit();
    };
    auto store4 = [&](double* base, long long off, const double (&v)[4]) {
        double* o = base + off;
        if (!edge && lane > 0 && lane < 31) {
            *reinterpret_cast<double2*>(o) = make_double2(v[0], v[1]);
            *reinterpret_cast<double2*>(o + 2) = make_double2(v[2], v[3]);
            return;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k)
            if (cout_[k]) o[k] = v[k];
    };
    // coarse columns of this lane's two odd (centre) fine columns i+1, i+3
    const int P0 = i / 2, P1 = i / 2 + 1;  // (i even)
    const bool p0ok = RESTRICT && lane > 0 && i + 1 < nx && P0 >= 0 && P0 < cg.nx;
    const bool p1ok = RESTRICT && lane < 31 && i + 3 < nx && P1 >= 0 && P1 < cg.nx;

    stage(Jbeg);
    stage(Jbeg + 1);
    cpa_wait<1>();
    __syncwarp();

    double xw[3][4], dw[3][4];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) xw[r][k] = dw[r][k] = 0.0;

    auto row = [&](int J, auto ph) {
        constexpr int PH = decltype(ph)::value;
        constexpr int sJ = PH % 3, sJ1 = (PH + 2) % 3, sJ2 = (PH + 1) % 3;  // rows J, J-1, J-2
        stage(J + 2);  // slot of row J-2: no longer read
        const int sl = slot_of(J), sl1 = slot_of(J - 1);
        const long long rJ = roff;
        roff += pitch;
        // x0 of row J
        {
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            if (J >= 0 && J < ny) {
                const double2 a = S.x[sl][0][lane], b = S.x[sl][1][lane];
                v[0] = a.x;
                v[1] = a.y;
                v[2] = b.x;
                v[3] = b.y;
                if constexpr (SUM) {
                    const double2 c = S.e[sl][0][lane], f = S.e[sl][1][lane];
                    v[0] = v[0] + 1.0 * c.x;
                    v[1] = v[1] + 1.0 * c.y;
                    v[2] = v[2] + 1.0 * f.x;
                    v[3] = v[3] + 1.0 * f.y;
                }
                if (edge) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (!cin[k]) v[k] = 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) xw[sJ][k] = v[k];
            if (STORE_X0 && J >= j0 && J < j1) store4(x0out, rJ, v);
        }
        // d of row R = J-1
        const int R = J - 1;
        {
            double d[4] = {0.0, 0.0, 0.0, 0.0};
            if (R >= 0 && R < ny) {
                const double2 ga = S.g[sl1][0][lane], gb = S.g[sl1][1][lane];
                const double gv[4] = {ga.x, ga.y, gb.x, gb.y};
                const double xl = __shfl_up_sync(0xffffffffu, xw[sJ1][3], 1);
                const double xr = __shfl_down_sync(0xffffffffu, xw[sJ1][0], 1);
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const double xe_ = k == 3 ? xr : xw[sJ1][k + 1];
                    const double xwv = k == 0 ? xl : xw[sJ1][k - 1];
                    const double ax =
                        stencil_apply(A, cix(i + k, fg.nx), R, xw[sJ1][k], xwv, xe_, xw[sJ2][k], xw[sJ][k]);
                    d[k] = gv[k] - ax;
                }
                if (edge) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (!cin[k]) d[k] = 0.0;
                }
            } else {
                // keep the shuffles warp-uniform: nothing to exchange on rows outside
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) dw[sJ1][k] = d[k];
            if (STORE_D && R >= j0 && R < j1) store4(dout, rJ - pitch, d);
        }
        // coarse row Q whose centre fine row 2Q+1 = R-1 lies in the segment
        if (RESTRICT && ((R & 1) == 0) && R >= 2 && R - 1 >= j0 && R - 1 < j1) {
            const int Q = R / 2 - 1;
            // rows dj = -1, 0, +1 are R-2, R-1, R = slots sJ, sJ2, sJ1 of dw
            const double n0 = __shfl_down_sync(0xffffffffu, dw[sJ][0], 1);
            const double n1 = __shfl_down_sync(0xffffffffu, dw[sJ2][0], 1);
            const double n2 = __shfl_down_sync(0xffffffffu, dw[sJ1][0], 1);
            if (Q < cg.ny) {
                double* crow = gc + (long long)Q * cg.pitch;
                if (p0ok) {
                    crow[P0] = restrict_at(rw, P0, Q, [&](int di, int dj) {
                        const double* rowv = dj < 0 ? dw[sJ] : (dj == 0 ? dw[sJ2] : dw[sJ1]);
                        return rowv[1 + di];
                    });
                }
                if (p1ok) {
                    crow[P1] = restrict_at(rw, P1, Q, [&](int di, int dj) {
                        const double* rowv = dj < 0 ? dw[sJ] : (dj == 0 ? dw[sJ2] : dw[sJ1]);
                        if (di < 1) return rowv[3 + di];
                        return dj < 0 ? n0 : (dj == 0 ? n1 : n2);
                    });
                }
            }
        }
        cpa_wait<1>();  // row J+1 has landed
        __syncwarp();
    };
    for (int J = Jbeg; J <= Jend; J += 3) {
        row(J, std::integral_constant<int, 0>{});
        if (J + 1 > Jend) break;
        row(J + 1, std::integral_constant<int, 1>{});
        if (J + 2 > Jend) break;
        row(J + 2, std::integral_constant<int, 2>{});
    }
    cpa_wait<0>();
}

// ---------------------------------------------------------------------------
// k_omega4: the adaptive-omega terms (cycle.cpp:40-51) for corr = P uc:
// T0_k = (A corr)_k * corr_k and T1_k = d_k * corr_k written densely in the
// reference's k order, and whether some corr_k^2 != 0 — warp-strip layout,
// coarse rows staged once per two fine rows as in k_smooth4.
// ---------------------------------------------------------------------------
struct Omega4Smem {
    static constexpr int D = 4;
    double2 d[D][2][32];
    double c[D][68];
    double t[2][128];  // one row of T0, T1 for coalesced stores
};

template <class Coef>
__global__ void __launch_bounds__(kS4W * 32, GMG_O4_MINB)
    k_omega4(Grid fg, Coef A, Prolong P, const double* __restrict__ dd, double* __restrict__ T0,
             double* __restrict__ T1, int* __restrict__ nz, int seg) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    using SM = Omega4Smem;
    constexpr int D = SM::D;
    constexpr int H = 2;
    constexpr int OW = 128 - 2 * H;
    extern __shared__ __align__(16) unsigned char o4raw[];
    SM& S = reinterpret_cast<SM*>(o4raw)[threadIdx.x >> 5];

    const int lane = threadIdx.x & 31;
    const int strip = blockIdx.x * kS4W + (threadIdx.x >> 5);
    const int i0 = strip * OW - H;
    if (i0 + H >= fg.nx) return;
    const int i = i0 + 4 * lane;
    const int nx = fg.nx, ny = fg.ny;
    const int j0 = fg.w0 + blockIdx.y * seg;
    const int j1 = min(j0 + seg, fg.w1);
    const bool edge = i0 < 0 || i0 + 128 > nx;
    bool cin[4], cout_[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
        cin[k] = i + k >= 0 && i + k < nx;
        const int c = 4 * lane + k;
        cout_[k] = cin[k] && c >= H && c < 128 - H;
    }
    const int m0 = i0 / 2 - 1;
    const double tX0 = cin[0] ? __ldg(P.tx + i) : 0.0;
    const double tX2 = cin[2] ? __ldg(P.tx + i + 2) : 0.0;
    auto chunk_bytes = [&](int c) { return (c >= 0 && c < nx) ? (c + 1 < nx ? 16 : 8) : 0; };
    const int cb0 = chunk_bytes(i), cb1 = chunk_bytes(i + 2);
    const long long pitch = fg.pitch;
    const int Jbeg = j0 - 1;  // corr rows j0-1 .. j1 give A corr on rows j0 .. j1-1
    const int Jend = j1;
    long long soff = (long long)Jbeg * pitch + i;
    auto slot_of = [](int J) { return (J + 8) & (D - 1); };
    auto stage_crow = [&](int q) {
        double* dst = S.c[(q + 8) & (D - 1)];
        stage_coarse(dst + 2 * lane, P.uc, P.cg, m0 + 2 * lane, q);
        stage_coarse(dst + 2 * lane + 1, P.uc, P.cg, m0 + 2 * lane + 1, q);
        if (lane == 0) stage_coarse(dst + 64, P.uc, P.cg, m0 + 64, q);
    };
    // fine row J: d of row J (used as d_R one iteration later) + the coarse row it adds
    auto stage = [&](int J) {
        const int sl = slot_of(J);
        const bool row_in = J >= 0 && J < ny;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int bytes = row_in ? (h ? cb1 : cb0) : 0;
            cpa16(&S.d[sl][h][lane], dd + (bytes ? soff + 2 * h : 0), bytes);
        }
        soff += pitch;
        if (((J + 8) & 1) == 0) stage_crow((J + 8) / 2 - 4);
        cpa_commit();
    };
    {
        const int qf = (Jbeg + 8) / 2 - 4;
        stage_crow(((Jbeg + 8) & 1) ? qf : qf - 1);
    }
    stage(Jbeg);
    stage(Jbeg + 1);
    cpa_wait<1>();
    __syncwarp();

    double ty_cur = (((Jbeg + 1) & 1) && Jbeg >= 0 && Jbeg < ny) ? __ldg(P.ty + Jbeg) : 0.0;
    double cw[3][4];
#pragma unroll
    for (int r = 0; r < 3; ++r)
#pragma unroll
        for (int k = 0; k < 4; ++k) cw[r][k] = 0.0;
    int any = 0;

    auto row = [&](int J, auto ph) {
        constexpr int PH = decltype(ph)::value;
        constexpr int sJ = PH % 3, sJ1 = (PH + 2) % 3, sJ2 = (PH + 1) % 3;  // rows J, J-1, J-2
        stage(J + 2);
        const int sl1 = slot_of(J - 1);
        // corr of row J (its prolongation weight was fetched an iteration ago; fetch the next row's)
        {
            const double tyJ = ty_cur;
            {
                const int Jn = J + 1;
                ty_cur = (((Jn + 1) & 1) && Jn >= 0 && Jn < ny) ? __ldg(P.ty + Jn) : 0.0;
            }
            double v[4] = {0.0, 0.0, 0.0, 0.0};
            if (J >= 0 && J < ny) {
                const int qf = (J + 8) / 2 - 4;
                const bool even = ((J + 8) & 1) == 0;
                const double* ca = &S.c[((even ? qf - 1 : qf) + 8) & (D - 1)][2 * lane];
                const double* cb = &S.c[(qf + 8) & (D - 1)][2 * lane];
                Pair2Raw r;
                r.ty = tyJ;
                r.a = ca[0];
                r.b = ca[1];
                r.c = cb[0];
                r.d = cb[1];
                const double2 p0 = prolong2_make(r, i, J, nx, tX0);
                r.a = ca[1];
                r.b = ca[2];
                r.c = cb[1];
                r.d = cb[2];
                const double2 p1 = prolong2_make(r, i + 2, J, nx, tX2);
                v[0] = p0.x;
                v[1] = p0.y;
                v[2] = p1.x;
                v[3] = p1.y;
                if (edge) {
#pragma unroll
                    for (int k = 0; k < 4; ++k)
                        if (!cin[k]) v[k] = 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < 4; ++k) cw[sJ][k] = v[k];
        }
        const int R = J - 1;
        if (R >= j0 && R < j1) {
            const double xl = __shfl_up_sync(0xffffffffu, cw[sJ1][3], 1);
            const double xr = __shfl_down_sync(0xffffffffu, cw[sJ1][0], 1);
            const double2 da = S.d[sl1][0][lane], db = S.d[sl1][1][lane];
            const double dv[4] = {da.x, da.y, db.x, db.y};
            double t0[4], t1[4];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const double b = cw[sJ1][k];
                const double xwv = k == 0 ? xl : cw[sJ1][k - 1];
                const double xev = k == 3 ? xr : cw[sJ1][k + 1];
                const double ac = stencil_apply(A, cix(i + k, fg.nx), R, b, xwv, xev, cw[sJ2][k], cw[sJ][k]);
                t0[k] = ac * b;
                t1[k] = dv[k] * b;
                if (cout_[k]) any |= (b * b) != 0.0;
            }
            // through shared memory so that consecutive lanes store consecutive k
            *reinterpret_cast<double2*>(&S.t[0][4 * lane]) = make_double2(t0[0], t0[1]);
            *reinterpret_cast<double2*>(&S.t[0][4 * lane + 2]) = make_double2(t0[2], t0[3]);
            *reinterpret_cast<double2*>(&S.t[1][4 * lane]) = make_double2(t1[0], t1[1]);
            *reinterpret_cast<double2*>(&S.t[1][4 * lane + 2]) = make_double2(t1[2], t1[3]);
            __syncwarp();
            const long long kr = (long long)R * nx + i0;  // k of the strip's first column
#pragma unroll
            for (int m = 0; m < 4; ++m) {
                const int c = lane + 32 * m;
                if (c >= H && c < 128 - H && i0 + c < nx) {
                    T0[kr + c] = S.t[0][c];
                    T1[kr + c] = S.t[1][c];
                }
            }
            __syncwarp();
        }
        cpa_wait<1>();
        __syncwarp();
    };
    for (int J = Jbeg; J <= Jend; J += 3) {
        row(J, std::integral_constant<int, 0>{});
        if (J + 1 > Jend) break;
        row(J + 1, std::integral_constant<int, 1>{});
        if (J + 2 > Jend) break;
        row(J + 2, std::integral_constant<int, 2>{});
    }
    cpa_wait<0>();
    if (__any_sync(0xffffffffu, any) && lane == 0) atomicOr(nz, 1);
}

constexpr size_t omega4_smem() { return sizeof(Omega4Smem) * kS4W; }

template <bool SUM>
constexpr size_t resid4_smem() {
    return sizeof(Resid4Smem<SUM>) * kS4W;
}

template <int SK, int M>
constexpr size_t smooth4_smem() {
    return sizeof(Smooth4Smem<SK, M>) * kS4W;
}

}  // namespace gmg_dev
