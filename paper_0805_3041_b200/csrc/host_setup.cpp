// Host setup for the B200 multigrid path. Compiled with -ffp-contract=off so
// every expression rounds exactly as the reference's.
#include "host_setup.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <stdexcept>

#include "seqsum_core.h"

namespace gmg_host {

namespace {

constexpr double kPi = 3.14159265358979323846;  // std::numbers::pi

// grade_axis (mesh.cpp:48-75): n interior nodes, geometric cell widths.
std::vector<double> graded_unit_axis(int n, double ratio) {
    if (n < 1) throw std::invalid_argument("grade_axis: n must be >= 1");
    if (!(ratio > 0.0)) throw std::invalid_argument("grade_axis: factor must be > 0");
    const int cells = n + 1;
    const double first = ratio == 1.0 ? 1.0 / cells : (ratio - 1.0) / (std::pow(ratio, cells) - 1.0);
    std::vector<double> u(static_cast<std::size_t>(n) + 2);
    u[0] = 0.0;
    double h = first;
    for (int q = 1; q <= n; ++q) {
        u[q] = u[q - 1] + h;
        h *= ratio;
    }
    u[n + 1] = 1.0;
    for (int q = 0; q <= n; ++q)
        if (!(u[q] < u[q + 1])) throw std::invalid_argument("grade_axis: factor too extreme for n points");
    return u;
}

// axis_range (mesh.cpp:25-36) then physical_axis (mesh.cpp:79-93).
std::vector<double> mapped_axis(int n, double ratio, int coords, int axis) {
    double lo = 0.0, hi = 1.0;
    if ((coords == 1 || coords == 3) && axis == 0) lo = 0.1;
    if (coords == 2) {
        lo = 0.1;
        if (axis == 1) hi = kPi - 0.1;
    }
    std::vector<double> p = graded_unit_axis(n, ratio);
    for (double& v : p) v = lo + (hi - lo) * v;
    p.front() = lo;
    p.back() = hi;
    for (std::size_t q = 0; q + 1 < p.size(); ++q)
        if (!(p[q] < p[q + 1]))
            throw std::invalid_argument("grading: factor too extreme for this resolution and axis range");
    return p;
}

// Flux-form coefficients (stencil.cpp:49-73); polar (cs 3) as in host_setup.h.
const double kPolarThetaWeight = 1.0 / (4.0 * kPi * kPi);
double face_x(int cs, double x) { return cs == 0 ? 1.0 : ((cs == 1 || cs == 3) ? x : x * x); }
double face_y(int cs, double y) { return cs == 2 ? std::sin(y) : (cs == 3 ? kPolarThetaWeight : 1.0); }
double measure_x(int cs, double a, double b) {
    return cs == 1 ? 0.5 * (b * b - a * a) : (cs == 3 ? std::log(b / a) : b - a);
}
double measure_y(int cs, double a, double b) { return cs == 2 ? std::cos(a) - std::cos(b) : b - a; }

// y = theta / (2 pi) on a periodic axis of ny nodes: y[q] = q / ny for q = 0 .. ny+1
// (q = 0 and ny+1 are the wrapped neighbours of the first and last node).
std::vector<double> periodic_axis(int ny) {
    std::vector<double> y(static_cast<std::size_t>(ny) + 2);
    for (int q = 0; q <= ny + 1; ++q) y[q] = static_cast<double>(q) / static_cast<double>(ny);
    return y;
}

void assemble_level(Level& L, int cs, double alpha, double beta) {
    const int nx = L.nx, ny = L.ny;
    const std::size_t N = static_cast<std::size_t>(nx) * ny;
    L.c.assign(N, 0.0);
    L.n.assign(N, 0.0);
    L.s.assign(N, 0.0);
    L.e.assign(N, 0.0);
    L.w.assign(N, 0.0);
    for (int j = 0; j < ny; ++j) {
        const double ys = 0.5 * (L.y[j] + L.y[j + 1]);
        const double yn = 0.5 * (L.y[j + 1] + L.y[j + 2]);
        const double dys = L.y[j + 1] - L.y[j];
        const double dyn = L.y[j + 2] - L.y[j + 1];
        const double my = measure_y(cs, ys, yn);
        for (int i = 0; i < nx; ++i) {
            const double xw = 0.5 * (L.x[i] + L.x[i + 1]);
            const double xe = 0.5 * (L.x[i + 1] + L.x[i + 2]);
            const double dxw = L.x[i + 1] - L.x[i];
            const double dxe = L.x[i + 2] - L.x[i + 1];
            const double mx = measure_x(cs, xw, xe);
            const double fe = alpha * face_x(cs, xe) * my / dxe;
            const double fw = alpha * face_x(cs, xw) * my / dxw;
            const double fn = beta * face_y(cs, yn) * mx / dyn;
            const double fs = beta * face_y(cs, ys) * mx / dys;
            const std::size_t k = static_cast<std::size_t>(j) * nx + i;
            L.c[k] = fe + fw + fn + fs;
            if (i + 1 < nx) L.e[k] = -fe;
            if (i > 0) L.w[k] = -fw;
            if (j + 1 < ny || L.periodic) L.n[k] = -fn;
            if (j > 0 || L.periodic) L.s[k] = -fs;
        }
    }
}

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof(double)) == 0; }

}  // namespace

std::vector<Level> build_problem(int num_levels, int cnx, int cny, double gx, double gy, int coords,
                                 double alpha, double beta) {
    if (num_levels < 1) throw std::invalid_argument("levels: must be >= 1");
    if (cnx < 1 || cny < 1) throw std::invalid_argument("coarse_n: interior counts must be >= 1");
    if (!(gx > 0.0) || !(gy > 0.0)) throw std::invalid_argument("grading: factors must be > 0");
    if (coords < 0 || coords > 3) throw std::invalid_argument("coords: unknown coordinate system");
    if (!(alpha > 0.0) || !(beta > 0.0)) throw std::invalid_argument("alpha/beta must be > 0");
    if (coords == 3) {
        if (gy != 1.0) throw std::invalid_argument("grading_y: the periodic polar theta axis must be uniform");
        if (cny < 2) throw std::invalid_argument("coarse_n: the periodic polar theta axis needs >= 2 nodes");
        std::vector<Level> lv(static_cast<std::size_t>(num_levels));
        Level& f = lv.back();
        f.level = num_levels;
        f.nx = ((cnx + 1) << (num_levels - 1)) - 1;
        f.x = mapped_axis(f.nx, gx, coords, 0);
        for (int l = num_levels; l >= 1; --l) {
            Level& L = lv[l - 1];
            L.level = l;
            L.periodic = true;
            L.ny = cny << (l - 1);
            L.y = periodic_axis(L.ny);
            if (l < num_levels) {
                const Level& fine = lv[l];
                L.nx = (fine.nx - 1) / 2;
                L.x.resize(static_cast<std::size_t>(L.nx) + 2);
                for (std::size_t q = 0; q < L.x.size(); ++q) L.x[q] = fine.x[2 * q];
            }
        }
        for (Level& L : lv) assemble_level(L, coords, alpha, beta);
        return lv;
    }
    std::vector<Level> lv(static_cast<std::size_t>(num_levels));
    Level& f = lv.back();
    f.level = num_levels;
    f.nx = ((cnx + 1) << (num_levels - 1)) - 1;
    f.ny = ((cny + 1) << (num_levels - 1)) - 1;
    f.x = mapped_axis(f.nx, gx, coords, 0);
    f.y = mapped_axis(f.ny, gy, coords, 1);
    for (int l = num_levels - 1; l >= 1; --l) {
        const Level& fine = lv[l];
        Level& coarse = lv[l - 1];
        coarse.level = l;
        coarse.nx = (fine.nx - 1) / 2;
        coarse.ny = (fine.ny - 1) / 2;
        coarse.x.resize(static_cast<std::size_t>(coarse.nx) + 2);
        coarse.y.resize(static_cast<std::size_t>(coarse.ny) + 2);
        for (std::size_t q = 0; q < coarse.x.size(); ++q) coarse.x[q] = fine.x[2 * q];
        for (std::size_t q = 0; q < coarse.y.size(); ++q) coarse.y[q] = fine.y[2 * q];
    }
    for (Level& L : lv) assemble_level(L, coords, alpha, beta);
    return lv;
}

std::vector<double> cholesky_band(const double* c, const double* w, const double* s, int nx, int ny) {
    const int n = nx * ny, bw = nx;
    std::vector<double> band(static_cast<std::size_t>(bw + 1) * n, 0.0);
    auto B = [&](int d, int k) -> double& { return band[static_cast<std::size_t>(d) * n + k]; };
    for (int k = 0; k < n; ++k) {
        B(0, k) = c[k];
        if (k % nx != 0) B(1, k) = w[k];
        if (k >= nx) B(bw, k) = s[k];
    }
    for (int col = 0; col < n; ++col) {
        double d = B(0, col);
        for (int m = std::max(0, col - bw); m < col; ++m) {
            const double l = B(col - m, col);
            d -= l * l;
        }
        if (!(d > 0.0)) throw std::runtime_error("BandedCholesky: matrix not positive definite");
        const double piv = std::sqrt(d);
        B(0, col) = piv;
        for (int row = col + 1; row <= std::min(n - 1, col + bw); ++row) {
            double a = B(row - col, row);
            for (int m = std::max(0, row - bw); m < col; ++m) a -= B(row - m, row) * B(col - m, col);
            B(row - col, row) = a / piv;
        }
    }
    return band;
}

CoefClass classify(int nx, int ny, const double* c, const double* n, const double* s, const double* e,
                   const double* w, bool periodic) {
    CoefClass cc;
    const std::size_t N = static_cast<std::size_t>(nx) * ny;
    // reference interior values (the row/column that has the neighbour)
    const double C = c[0];
    const double W = nx > 1 ? w[1] : 0.0;
    const double E = nx > 1 ? e[0] : 0.0;
    const double S = ny > 1 ? s[nx] : 0.0;
    const double Nn = ny > 1 ? n[0] : 0.0;
    bool isconst = true;
    for (std::size_t k = 0; k < N && isconst; ++k) {
        const int i = static_cast<int>(k % nx), j = static_cast<int>(k / nx);
        isconst = same_bits(c[k], C) && same_bits(w[k], i > 0 ? W : 0.0) &&
                  same_bits(e[k], i + 1 < nx ? E : 0.0) && same_bits(s[k], (j > 0 || periodic) ? S : 0.0) &&
                  same_bits(n[k], (j + 1 < ny || periodic) ? Nn : 0.0);
    }
    if (isconst) {
        cc.kind = COEF_CONST;
        cc.c = C;
        cc.w = W;
        cc.e = E;
        cc.s = S;
        cc.n = Nn;
        return cc;
    }
    // x-varying rows: every row equals row 0 except s (0 on row 0) and n (0 on the last row)
    bool rowx = true;
    for (int j = 0; j < ny && rowx; ++j)
        for (int i = 0; i < nx && rowx; ++i) {
            const std::size_t k = static_cast<std::size_t>(j) * nx + i;
            const double Si = ny > 1 ? s[static_cast<std::size_t>(nx) + i] : 0.0;
            rowx = same_bits(c[k], c[i]) && same_bits(w[k], w[i]) && same_bits(e[k], e[i]) &&
                   same_bits(s[k], (j > 0 || periodic) ? Si : 0.0) &&
                   same_bits(n[k], (j + 1 < ny || periodic) ? n[i] : 0.0);
        }
    if (rowx) {
        cc.kind = COEF_ROWX;
        cc.rc.assign(c, c + nx);
        cc.rw.assign(w, w + nx);
        cc.re.assign(e, e + nx);
        cc.rs.resize(nx);
        for (int i = 0; i < nx; ++i) cc.rs[i] = ny > 1 ? s[static_cast<std::size_t>(nx) + i] : 0.0;
        cc.rn.assign(n, n + nx);
        return cc;
    }
    cc.kind = COEF_FIELD;
    return cc;
}

static double odd_w(const std::vector<double>& xf, const std::vector<double>& xc, int q) {
    return (xf[2 * q + 1] - xc[q]) / (xc[q + 1] - xc[q]);
}

std::vector<double> prolong_weights(const std::vector<double>& xf, const std::vector<double>& xc, int nf) {
    std::vector<double> t(static_cast<std::size_t>(nf), 0.0);
    for (int i = 0; i < nf; ++i)
        if ((i + 1) % 2 == 1) t[i] = odd_w(xf, xc, i / 2);
    return t;
}

void restrict_weights(const std::vector<double>& xf, const std::vector<double>& xc, int nc,
                      std::vector<double>& ww, std::vector<double>& we, std::vector<double>& sw) {
    ww.resize(nc);
    we.resize(nc);
    sw.resize(nc);
    for (int P = 0; P < nc; ++P) {
        ww[P] = odd_w(xf, xc, P);
        we[P] = 1.0 - odd_w(xf, xc, P + 1);
        sw[P] = ww[P] + 1.0 + we[P];
    }
}

double polar_theta_weight() { return kPolarThetaWeight; }

bool axis_tables(const Level& L, int cs, double alpha, double beta, const double* c, const double* n,
                 const double* s, const double* e, const double* w, AxisTables& T) {
    if (cs < 0 || cs > 2 || !(alpha > 0.0) || !(beta > 0.0) || L.periodic) return false;
    const int nx = L.nx, ny = L.ny;
    T = AxisTables{};
    for (int i = 0; i < nx; ++i) {
        const double xw = 0.5 * (L.x[i] + L.x[i + 1]);
        const double xe = 0.5 * (L.x[i + 1] + L.x[i + 2]);
        const double dxw = L.x[i + 1] - L.x[i];
        const double dxe = L.x[i + 2] - L.x[i + 1];
        T.ae.push_back(alpha * face_x(cs, xe));
        T.aw.push_back(alpha * face_x(cs, xw));
        T.he.push_back(dxe);
        T.hw.push_back(dxw);
        T.mx.push_back(measure_x(cs, xw, xe));
        T.rhe.push_back(1.0 / dxe);
        T.rhw.push_back(1.0 / dxw);
    }
    for (int j = 0; j < ny; ++j) {
        const double ys = 0.5 * (L.y[j] + L.y[j + 1]);
        const double yn = 0.5 * (L.y[j + 1] + L.y[j + 2]);
        const double dys = L.y[j + 1] - L.y[j];
        const double dyn = L.y[j + 2] - L.y[j + 1];
        T.bn.push_back(beta * face_y(cs, yn));
        T.bs.push_back(beta * face_y(cs, ys));
        T.hn.push_back(dyn);
        T.hs.push_back(dys);
        T.my.push_back(measure_y(cs, ys, yn));
        T.rhn.push_back(1.0 / dyn);
        T.rhs.push_back(1.0 / dys);
    }
    // the reciprocal path (div_rcp) needs normal spacings in [2^-500, 2^500]
    for (const std::vector<double>* v : {&T.he, &T.hw, &T.hn, &T.hs})
        for (double h : *v)
            if (!std::isnormal(h) || std::fabs(h) < 0x1p-500 || std::fabs(h) > 0x1p500) return false;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const double ce = (T.ae[i] * T.my[j]) / T.he[i];
            const double cw = (T.aw[i] * T.my[j]) / T.hw[i];
            const double cn = (T.bn[j] * T.mx[i]) / T.hn[j];
            const double cs_ = (T.bs[j] * T.mx[i]) / T.hs[j];
            const std::size_t k = static_cast<std::size_t>(j) * nx + i;
            if (!same_bits(c[k], ((ce + cw) + cn) + cs_) || !same_bits(e[k], i + 1 < nx ? -ce : 0.0) ||
                !same_bits(w[k], i > 0 ? -cw : 0.0) || !same_bits(n[k], j + 1 < ny ? -cn : 0.0) ||
                !same_bits(s[k], j > 0 ? -cs_ : 0.0))
                return false;
        }
    return true;
}

std::vector<double> cholesky_periodic(const double* c, const double* w, const double* e, const double* s,
                                      const double* n, int nx, int ny) {
    const int N = nx * ny, bw = N - 1;
    // dense lower triangle of A (row k, column m < k), couplings accumulated in
    // the order c, w, e, s, n of apply (stencil.cpp:133-137) with y wrapped
    std::vector<double> A(static_cast<std::size_t>(N) * N, 0.0);
    auto at = [&](int r, int q) -> double& { return A[static_cast<std::size_t>(r) * N + q]; };
    for (int k = 0; k < N; ++k) {
        const int i = k % nx, j = k / nx;
        at(k, k) = at(k, k) + c[k];
        if (i > 0) at(k, k - 1) = at(k, k - 1) + w[k];
        if (i + 1 < nx) at(k, k + 1) = at(k, k + 1) + e[k];
        const int js = (j + ny - 1) % ny, jn = (j + 1) % ny;
        at(k, js * nx + i) = at(k, js * nx + i) + s[k];
        at(k, jn * nx + i) = at(k, jn * nx + i) + n[k];
    }
    std::vector<double> band(static_cast<std::size_t>(bw + 1) * N, 0.0);
    auto B = [&](int d, int k) -> double& { return band[static_cast<std::size_t>(d) * N + k]; };
    for (int k = 0; k < N; ++k)
        for (int d = 0; d <= k; ++d) B(d, k) = at(k, k - d);
    for (int col = 0; col < N; ++col) {
        double d = B(0, col);
        for (int m = std::max(0, col - bw); m < col; ++m) {
            const double l = B(col - m, col);
            d -= l * l;
        }
        if (!(d > 0.0)) throw std::runtime_error("BandedCholesky: matrix not positive definite");
        const double piv = std::sqrt(d);
        B(0, col) = piv;
        for (int row = col + 1; row <= std::min(N - 1, col + bw); ++row) {
            double a = B(row - col, row);
            for (int m = std::max(0, row - bw); m < col; ++m) a -= B(row - m, row) * B(col - m, col);
            B(row - col, row) = a / piv;
        }
    }
    return band;
}

std::string check_nested(const Level& coarse, const Level& fine) {
    if (fine.periodic != coarse.periodic) return "levels are not parent and child";
    if (fine.periodic) {
        if (fine.level != coarse.level + 1 || fine.nx != 2 * coarse.nx + 1 || fine.ny != 2 * coarse.ny)
            return "levels are not parent and child";
        for (int q = 0; q < coarse.nx + 2; ++q)
            if (std::abs(coarse.x[q] - fine.x[2 * q]) > 1e-14) return "grids are not nested";
        for (int q = 0; q <= coarse.ny; ++q)
            if (std::abs(coarse.y[q] - fine.y[2 * q]) > 1e-14) return "grids are not nested";
        return "";
    }
    if (fine.level != coarse.level + 1 || fine.nx != 2 * coarse.nx + 1 || fine.ny != 2 * coarse.ny + 1)
        return "levels are not parent and child";
    for (int q = 0; q < coarse.nx + 2; ++q)
        if (std::abs(coarse.x[q] - fine.x[2 * q]) > 1e-14) return "grids are not nested";
    for (int q = 0; q < coarse.ny + 2; ++q)
        if (std::abs(coarse.y[q] - fine.y[2 * q]) > 1e-14) return "grids are not nested";
    return "";
}

// ---------------------------------------------------------------------------
// Host emulation of the device pipeline (seqsum.cuh) with identical chunking:
// approximate prefixes as speculation, per-thread walks, runs merged across
// threads and chunks, one record per break (+ the final record), replayed from
// the exact state with literal re-sums of any record that fails validation.
// stats: [0] chunks, [1] records, [2] literal re-sums, [3] breaks.
void factor_ilu0(int nx, int ny, const double* c, const double* w, const double* e, const double* s,
                 const double* n, double* lw, double* ls, double* d) {
    // row-major sweep: the pivot of node k needs the pivots of its west and
    // south neighbours, which the sweep has already produced
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const std::size_t k = static_cast<std::size_t>(j) * nx + i;
            double piv = c[k];
            double a = 0.0, b = 0.0;
            if (i > 0) {
                a = w[k] / d[k - 1];
                piv -= a * e[k - 1];
            }
            if (j > 0) {
                b = s[k] / d[k - nx];
                piv -= b * n[k - nx];
            }
            if (piv <= 0.0) throw std::runtime_error("ilu0 factorization: nonpositive pivot");
            lw[k] = a;
            ls[k] = b;
            d[k] = piv;
        }
}

SlabPlan slab_plan(const std::vector<int>& ny, int world, int min_rows, int halo) {
    const int L = static_cast<int>(ny.size());
    SlabPlan sp;
    sp.Ls = L + 1;
    if (world > 1)
        for (int l = 1; l <= L; ++l)
            if (ny[l - 1] >= min_rows && ny[l - 1] >= world * halo) {
                sp.Ls = l;
                break;
            }
    sp.w0.assign(L, std::vector<int>(world, 0));
    sp.w1.assign(L, std::vector<int>(world, 0));
    for (int l = 1; l <= L; ++l)
        for (int r = 0; r < world; ++r) {
            if (l < sp.Ls) {
                sp.w1[l - 1][r] = ny[l - 1];
            } else if (l == sp.Ls) {
                sp.w0[l - 1][r] = static_cast<int>(static_cast<long long>(r) * ny[l - 1] / world);
                sp.w1[l - 1][r] = static_cast<int>(static_cast<long long>(r + 1) * ny[l - 1] / world);
            } else {
                sp.w0[l - 1][r] = r == 0 ? 0 : 2 * sp.w0[l - 2][r];
                sp.w1[l - 1][r] = r == world - 1 ? ny[l - 1] : 2 * sp.w1[l - 2][r];
            }
        }
    return sp;
}

double seqsum_emulate(const double* p, long long n, int T, int EPT, long long* stats) {
    using namespace gmg_ss;
    const long long C = static_cast<long long>(T) * EPT;
    const long long nch = (n + C - 1) / C;
    std::vector<Rec> recs;
    Seg carry = seg_empty();  // run since the last break, across chunks
    double approx = 0.0;
    long long nbreaks = 0;
    for (long long c = 0; c < nch; ++c) {
        const long long base = c * C;
        const int clen = static_cast<int>(std::min(C, n - base));
        double acc = approx;
        for (int t = 0; t < T; ++t) {
            const double pred = acc;
            double ts = 0.0;
            for (int m = 0; m < EPT; ++m) {
                const int e = t * EPT + m;
                if (e < clen) ts += p[base + e];
            }
            acc += ts;
            Walker wk;
            walker_init(wk, pred);
            for (int m = 0; m < EPT; ++m) {
                const int e = t * EPT + m;
                if (e >= clen) break;
                const double v = p[base + e];
                if (!walker_try(wk, v)) {
                    ++nbreaks;
                    recs.push_back(rec_make(seg_merge(carry, walker_seg(wk)), true, v, static_cast<uint32_t>(base + e)));
                    carry = seg_empty();
                    walker_open(wk);
                    walker_real_add(wk, v);
                }
            }
            carry = seg_merge(carry, walker_seg(wk));
        }
        approx = acc;
    }
    recs.push_back(rec_make(carry, false, 0.0, static_cast<uint32_t>(n - 1)));
    long long nlit = 0, prev = -1;
    State st = make_state(0.0);
    for (const Rec& r : recs) {
        const Seg g = rec_seg(r);
        const bool brk = rec_has_break(r);
        const long long kb = r.kb;
        if (!seg_valid(g, st)) {
            ++nlit;
            double s = st.s;
            for (long long k = prev + 1; k < (brk ? kb : kb + 1); ++k) s = s + p[k];
            st = make_state(s);
            if (brk) st = make_state(st.s + r.pb);
        } else if (brk) {
            const double sb = g.len ? compose(st.M + ((st.M & 1) ? g.Q[1] : g.Q[0]), st.E) : st.s;
            st = make_state(sb + r.pb);
        } else {
            seg_apply(g, st);
        }
        prev = kb;
    }
    if (stats) {
        stats[0] = nch;
        stats[1] = static_cast<long long>(recs.size());
        stats[2] = nlit;
        stats[3] = nbreaks;
    }
    return st.s;
}

}  // namespace gmg_host
