// Line smoothers (tri_x, tri_y, adi, gstri_x, gstri_y, gsadi) and the
// Richardson step on sm_100a: SURVEY.md §8 row a16, reference
// /root/reference/proj/src/smoother.cpp:74-182 (factor / solve) and :339-384
// (apply_preconditioner cases).
//
// Every line solve is the reference's Thomas recurrence, element for element:
//   forward   y_t = y_t - sub_t * y_{t-1}           (t >= 1)      :120-121
//   backward  z_{n-1} = y_{n-1} / diag_{n-1}
//             z_t = (y_t - sup_t * z_{t+1}) / diag_t               :122-124
// so the order inside a line is fixed; the parallelism is across lines.
//   * tri_x / tri_y / adi: lines are independent -> one thread per line
//     (k_line). For y-lines (columns) a warp's loads are coalesced; for x-lines
//     each thread walks its own row, served by L1 sectors. Loads are issued a
//     block of kLineU steps ahead of the recurrence.
//   * gstri_x / gstri_y / gsadi: line t's right-hand side needs line t-1's
//     finished solution (smoother.cpp:160-162), and a line finishes at its first
//     element, where the next line starts: the whole sweep is one sequential
//     chain. One warp runs it (k_gstri): lanes load 32 steps at a time,
//     coalesced, and every lane evaluates the chain from shuffled operands, so
//     the only serial latency is the arithmetic itself.
// The factors (sub, diag, sup) are the reference's factor_lines_x/y arrays,
// computed on the device once per (smoother, omega) by k_tri_factor and kept
// pitched like the level's grid functions.
#pragma once

#include "common.cuh"

namespace gmg_dev {

struct LineFactors {
    const double *sub, *diag, *sup;  // pitched like the level
};

// output of a line solve: out = x - damp*z | z | x - damp*(z1 + z)
enum LineOut { LO_UPDATE = 0, LO_Z = 1, LO_SUM_UPDATE = 2 };

template <int DIR>
__device__ __forceinline__ long long line_at(const Grid& g, int line, int t) {
    return DIR == 0 ? g.at(t, line) : g.at(line, t);
}

template <int MODE>
__device__ __forceinline__ double line_out(double z, const double* x, const double* z1, long long k, double damp) {
    if (MODE == LO_Z) return z;
    if (MODE == LO_UPDATE) return x[k] - damp * z;
    const double zs = z1[k] + z;
    return x[k] - damp * zs;
}

// factor_lines_x (DIR 0, smoother.cpp:74-95) / factor_lines_y (DIR 1, :99-115),
// one thread per line. A zero pivot sets *status = 4.
template <int DIR, class Coef>
__global__ void k_tri_factor(Grid g, Coef A, double om, double* __restrict__ sub, double* __restrict__ diag,
                             double* __restrict__ sup, int* __restrict__ status) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = DIR == 0 ? g.ny : g.nx, n = DIR == 0 ? g.nx : g.ny;
    if (line >= nl) return;
    double dprev = 0.0, sprev = 0.0;
    for (int t = 0; t < n; ++t) {
        const int i = DIR == 0 ? t : line, j = DIR == 0 ? line : t;
        double C, W, E, S, N;
        A.load(i, j, C, W, E, S, N);
        double dg = om * C;
        double sb = om * (DIR == 0 ? W : S);
        const double sp = om * (DIR == 0 ? E : N);
        if (t > 0) {
            if (dprev == 0.0) *status = 4;
            const double m = sb / dprev;
            dg = dg - m * sprev;
            sb = m;
        }
        const long long k = line_at<DIR>(g, line, t);
        sub[k] = sb;
        diag[k] = dg;
        sup[k] = sp;
        dprev = dg;
        sprev = sp;
    }
}

constexpr int kLineU = 8;    // steps per prefetched block
constexpr int kLineT = 128;  // threads per CTA

// Thomas solves of independent lines; rhs may alias ybuf (in place).
template <int DIR, int MODE>
__global__ void __launch_bounds__(kLineT) k_line(Grid g, LineFactors f, const double* rhs, double* ybuf,
                                                 const double* __restrict__ x, const double* __restrict__ z1,
                                                 double* __restrict__ out, double damp) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int nl = DIR == 0 ? g.ny : g.nx, n = DIR == 0 ? g.nx : g.ny;
    if (line >= nl) return;
    constexpr int U = kLineU;
    const int nb = (n + U - 1) / U;
    // forward elimination
    {
        double cr[U], cs[U], nr[U], ns[U];
        auto load = [&](int b, double* r, double* s) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = b * U + u;
                if (t < n) {
                    const long long k = line_at<DIR>(g, line, t);
                    r[u] = rhs[k];
                    s[u] = __ldg(f.sub + k);
                }
            }
        };
        load(0, cr, cs);
        double y = 0.0;
        for (int b = 0; b < nb; ++b) {
            if (b + 1 < nb) load(b + 1, nr, ns);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = b * U + u;
                if (t < n) {
                    y = (t == 0) ? cr[u] : cr[u] - cs[u] * y;
                    ybuf[line_at<DIR>(g, line, t)] = y;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                cr[u] = nr[u];
                cs[u] = ns[u];
            }
        }
    }
    // back substitution (same thread wrote ybuf: program order makes it visible)
    {
        double cy[U], cp[U], cd[U], ny_[U], np[U], nd[U];
        auto load = [&](int b, double* yv, double* pv, double* dv) {
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = n - 1 - (b * U + u);
                if (t >= 0) {
                    const long long k = line_at<DIR>(g, line, t);
                    yv[u] = ybuf[k];
                    pv[u] = __ldg(f.sup + k);
                    dv[u] = __ldg(f.diag + k);
                }
            }
        };
        load(0, cy, cp, cd);
        double z = 0.0;
        for (int b = 0; b < nb; ++b) {
            if (b + 1 < nb) load(b + 1, ny_, np, nd);
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int t = n - 1 - (b * U + u);
                if (t >= 0) {
                    z = (t == n - 1) ? cy[u] / cd[u] : (cy[u] - cp[u] * z) / cd[u];
                    const long long k = line_at<DIR>(g, line, t);
                    out[k] = line_out<MODE>(z, x, z1, k, damp);
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                cy[u] = ny_[u];
                cp[u] = np[u];
                cd[u] = nd[u];
            }
        }
    }
}

// Line Gauss-Seidel sweep (solve_gstri_x DIR 0, smoother.cpp:156-167;
// solve_gstri_y DIR 1, :169-182): lines in order; line L's rhs is
// r - (om*s)*z(line L-1) (x-lines) or r - (om*w)*z(line L-1) (y-lines).
// One warp. zline / ybuf: scratch of max(nx, ny) doubles.
template <int DIR, int MODE, class Coef>
__global__ void __launch_bounds__(32) k_gstri(Grid g, Coef A, double om, LineFactors f,
                                              const double* __restrict__ rhs, const double* __restrict__ x,
                                              const double* __restrict__ z1, double* __restrict__ out,
                                              double* __restrict__ zline, double* __restrict__ ybuf,
                                              double damp) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int lane = threadIdx.x;
    const unsigned full = 0xffffffffu;
    const int nl = DIR == 0 ? g.ny : g.nx, n = DIR == 0 ? g.nx : g.ny;
    const int nc = (n + 31) / 32;
    for (int L = 0; L < nl; ++L) {
        // ---- forward: rhs with the previous line folded in, then elimination
        auto fload = [&](int c, double& r, double& s) {
            const int t = c * 32 + lane;
            r = 0.0;
            s = 0.0;
            if (t < n) {
                const int i = DIR == 0 ? t : L, j = DIR == 0 ? L : t;
                const long long k = g.at(i, j);
                double rv = rhs[k];
                if (L > 0) {
                    double C, W, E, S, N;
                    A.load(i, j, C, W, E, S, N);
                    rv = rv - om * (DIR == 0 ? S : W) * zline[t];
                }
                r = rv;
                s = __ldg(f.sub + k);
            }
        };
        double r, s, rn = 0.0, sn = 0.0;
        fload(0, r, s);
        double y = 0.0;
        for (int c = 0; c < nc; ++c) {
            if (c + 1 < nc) fload(c + 1, rn, sn);
            const int cnt = min(32, n - c * 32);
            double mine = 0.0;
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const double rq = __shfl_sync(full, r, q);
                const double sq = __shfl_sync(full, s, q);
                if (q < cnt) {
                    y = (c == 0 && q == 0) ? rq : rq - sq * y;
                    if (lane == q) mine = y;
                }
            }
            if (lane < cnt) ybuf[c * 32 + lane] = mine;
            r = rn;
            s = sn;
        }
        __syncwarp();
        // ---- back substitution, chunks from the end
        auto bload = [&](int c, double& yv, double& pv, double& dv) {
            const int t = c * 32 + lane;
            yv = 0.0;
            pv = 0.0;
            dv = 1.0;
            if (t < n) {
                const int i = DIR == 0 ? t : L, j = DIR == 0 ? L : t;
                const long long k = g.at(i, j);
                yv = ybuf[t];
                pv = __ldg(f.sup + k);
                dv = __ldg(f.diag + k);
            }
        };
        double yv, pv, dv, yn = 0.0, pn = 0.0, dn = 1.0;
        bload(nc - 1, yv, pv, dv);
        double z = 0.0;
        for (int c = nc - 1; c >= 0; --c) {
            if (c > 0) bload(c - 1, yn, pn, dn);
            const int cnt = min(32, n - c * 32);
            double mine = 0.0;
#pragma unroll
            for (int q = 31; q >= 0; --q) {
                const double yq = __shfl_sync(full, yv, q);
                const double pq = __shfl_sync(full, pv, q);
                const double dq = __shfl_sync(full, dv, q);
                if (q < cnt) {
                    z = (c * 32 + q == n - 1) ? yq / dq : (yq - pq * z) / dq;
                    if (lane == q) mine = z;
                }
            }
            const int t = c * 32 + lane;
            if (lane < cnt) {
                const int i = DIR == 0 ? t : L, j = DIR == 0 ? L : t;
                const long long k = g.at(i, j);
                out[k] = line_out<MODE>(mine, x, z1, k, damp);
                zline[t] = mine;
            }
            yv = yn;
            pv = pn;
            dv = dn;
        }
        __syncwarp();
    }
}

// Richardson step (smoother.cpp:284-285 with :389-399): x - damp*(rw*d).
__global__ void k_rich_update(Grid g, const double* __restrict__ d, const double* __restrict__ x,
                              double* __restrict__ out, double rw, double damp) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= g.nx) return;
    const long long k = g.at(i, j);
    const double z = rw * d[k];
    out[k] = x[k] - damp * z;
}

// power_apply_A's normalisation y_k / lambda (smoother.cpp:223).
__global__ void k_div_scalar(Grid g, double* __restrict__ y, double lambda) {
    pdl_wait();  // programmatic dependent launch: inputs of the previous kernel are complete
    pdl_trigger();
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    const int j = blockIdx.y;
    if (i >= g.nx) return;
    const long long k = g.at(i, j);
    y[k] = y[k] / lambda;
}

}  // namespace gmg_dev
