/* TEST INFRASTRUCTURE ONLY — CPU oracle for the gmg2d F-cycle path.
 * See gmg_oracle.h for scope and the pinning story. Reference paths below are
 * relative to /root/reference/proj. Arrays are interior-only, row-major with x
 * fastest (k = j*nx + i), as GridFunction (include/gmg/grid_function.hpp:10-26).
 */
#include "gmg_oracle.h"

#include <math.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

static char g_err[256];
static int fail(int code, const char* msg) {
    snprintf(g_err, sizeof g_err, "%s", msg);
    return code;
}
const char* orc_last_error(void) { return g_err; }

enum { K_RICH, K_JACOBI, K_GS, K_SOR, K_ILU0, K_TRIX, K_TRIY, K_ADI, K_GSTRIX, K_GSTRIY, K_GSADI };
enum { CS_CART, CS_CYL, CS_SPH, CS_POLAR };

/* CS_POLAR has no reference counterpart (the reference has cartesian, cylindrical
 * and spherical only, mesh.hpp:8): BASELINE config 3's polar Poisson problem,
 * restated with the reference's own discretisation rules and marked "parity
 * unpinned". x = r in [0.1, 1] (Dirichlet, graded like the
 * cylindrical radius), y = theta / (2 pi) in [0, 1) PERIODIC: level l has
 * coarse_ny * 2^(l-1) nodes y_j = (j+1)/ny (node ny-1 at 1 == 0); y[0] = 0 and
 * y[ny+1] = (ny+1)/ny are the wrapped neighbours. Flux form as stencil.cpp:49-127
 * with x-flux face weight r, y-flux face weight 1/(2 pi)^2 and transverse measures
 * dy and int dr/r = log(r_e/r_w): -(r u_r)_r - (1/r) u_theta theta times the cell.
 * Every y index wraps (apply, transfers, the level-1 factorization); only the
 * pointwise smoothers (jacobi, richardson) are defined on it. */

typedef struct {
    int level, nx, ny, coords;
    int per; /* y periodic (CS_POLAR) */
    double *x, *y; /* nx+2 / ny+2 node coordinates including the boundary */
} grid_t;

typedef struct {
    double *c, *n, *s, *e, *w;
} op_t;

struct orc_problem {
    int L;
    grid_t* g; /* g[l-1] = level l */
    op_t* op;
    int chol_n, chol_bw;
    double* band; /* band[d*n + k] = L(k, k-d) */
};

static double* dalloc(size_t n) { return (double*)calloc(n ? n : 1, sizeof(double)); }
static size_t nlev(const grid_t* g) { return (size_t)g->nx * (size_t)g->ny; }

/* ---- geometry: mesh.cpp ------------------------------------------------ */

/* grade_axis, mesh.cpp:48-75 */
static int grade_axis(int n, double factor, double* out) {
    if (n < 1) return fail(ORC_ERR_INVALID, "grade_axis: n must be >= 1");
    if (!(factor > 0.0)) return fail(ORC_ERR_INVALID, "grade_axis: factor must be > 0");
    const int cells = n + 1;
    double w0 = factor == 1.0 ? 1.0 / cells : (factor - 1.0) / (pow(factor, cells) - 1.0);
    out[0] = 0.0;
    double width = w0;
    for (int i = 1; i <= n; ++i) {
        out[i] = out[i - 1] + width;
        width *= factor;
    }
    out[n + 1] = 1.0;
    for (int i = 0; i <= n; ++i)
        if (!(out[i] < out[i + 1]))
            return fail(ORC_ERR_INVALID, "grade_axis: factor too extreme for n points");
    return ORC_OK;
}

/* axis_range, mesh.cpp:25-36 (kRadialMin 0.1, kPolarMargin 0.1, mesh.hpp:20-21) */
static void axis_range(int cs, int axis, double* lo, double* hi) {
    const double pi = 3.14159265358979323846;
    *lo = 0.0;
    *hi = 1.0;
    if ((cs == CS_CYL || cs == CS_POLAR) && axis == 0) *lo = 0.1;
    if (cs == CS_SPH) {
        if (axis == 0) {
            *lo = 0.1;
        } else {
            *lo = 0.1;
            *hi = pi - 0.1;
        }
    }
}

/* physical_axis, mesh.cpp:79-93 */
static int physical_axis(int n, double factor, int cs, int axis, double* p) {
    int st = grade_axis(n, factor, p);
    if (st) return st;
    double lo, hi;
    axis_range(cs, axis, &lo, &hi);
    for (int i = 0; i < n + 2; ++i) p[i] = lo + (hi - lo) * p[i];
    p[0] = lo;
    p[n + 1] = hi;
    for (int i = 0; i + 1 < n + 2; ++i)
        if (!(p[i] < p[i + 1]))
            return fail(ORC_ERR_INVALID,
                        "grading: factor too extreme for this resolution and axis range");
    return ORC_OK;
}

/* ---- assembly: stencil.cpp:49-127 --------------------------------------- */

static const double kPolarPi = 3.14159265358979323846;
static double face_weight_x(int cs, double x) {
    return cs == CS_CART ? 1.0 : ((cs == CS_CYL || cs == CS_POLAR) ? x : x * x);
}
static double face_weight_y(int cs, double y) {
    return cs == CS_SPH ? sin(y) : (cs == CS_POLAR ? 1.0 / (4.0 * kPolarPi * kPolarPi) : 1.0);
}
static double cell_measure_x(int cs, double lo, double hi) {
    return cs == CS_CYL ? 0.5 * (hi * hi - lo * lo) : (cs == CS_POLAR ? log(hi / lo) : hi - lo);
}
static double cell_measure_y(int cs, double lo, double hi) {
    return cs == CS_SPH ? cos(lo) - cos(hi) : hi - lo;
}

static void assemble(const grid_t* g, double alpha, double beta, op_t* op) {
    const int nx = g->nx, ny = g->ny, cs = g->coords;
    const size_t n = nlev(g);
    op->c = dalloc(n);
    op->n = dalloc(n);
    op->s = dalloc(n);
    op->e = dalloc(n);
    op->w = dalloc(n);
    for (int j = 0; j < ny; ++j) {
        const double fys = 0.5 * (g->y[j] + g->y[j + 1]);
        const double fyn = 0.5 * (g->y[j + 1] + g->y[j + 2]);
        const double hs = g->y[j + 1] - g->y[j];
        const double hn = g->y[j + 2] - g->y[j + 1];
        const double my = cell_measure_y(cs, fys, fyn);
        for (int i = 0; i < nx; ++i) {
            const double fxw = 0.5 * (g->x[i] + g->x[i + 1]);
            const double fxe = 0.5 * (g->x[i + 1] + g->x[i + 2]);
            const double hw = g->x[i + 1] - g->x[i];
            const double he = g->x[i + 2] - g->x[i + 1];
            const double mx = cell_measure_x(cs, fxw, fxe);
            const double ce = alpha * face_weight_x(cs, fxe) * my / he;
            const double cw = alpha * face_weight_x(cs, fxw) * my / hw;
            const double cn = beta * face_weight_y(cs, fyn) * mx / hn;
            const double csth = beta * face_weight_y(cs, fys) * mx / hs;
            const size_t k = (size_t)j * nx + i;
            op->c[k] = ce + cw + cn + csth;
            if (i + 1 < nx) op->e[k] = -ce;
            if (i > 0) op->w[k] = -cw;
            if (j + 1 < ny || g->per) op->n[k] = -cn;
            if (j > 0 || g->per) op->s[k] = -csth;
        }
    }
}

/* ---- BLAS-1 and the operator: stencil.cpp:9-31,129-153 ------------------- */

double orc_norm_l2(long long n, const double* v) {
    double s = 0.0;
    for (long long k = 0; k < n; ++k) s += v[k] * v[k];
    return sqrt(s);
}

double orc_dot(long long n, const double* a, const double* b) {
    double s = 0.0;
    for (long long k = 0; k < n; ++k) s += a[k] * b[k];
    return s;
}

void orc_axpy(long long n, double alpha, const double* x, double* y) {
    for (long long k = 0; k < n; ++k) y[k] += alpha * x[k];
}

/* apply, stencil.cpp:129-146: c, w, e, s, n accumulation order */
static void op_apply(const grid_t* g, const op_t* A, const double* x, double* y) {
    const int nx = g->nx, ny = g->ny;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)j * nx + i;
            double acc = A->c[k] * x[k];
            if (i > 0) acc += A->w[k] * x[k - 1];
            if (i + 1 < nx) acc += A->e[k] * x[k + 1];
            if (g->per) {
                acc += A->s[k] * x[(size_t)((j + ny - 1) % ny) * nx + i];
                acc += A->n[k] * x[(size_t)((j + 1) % ny) * nx + i];
            } else {
                if (j > 0) acc += A->s[k] * x[k - nx];
                if (j + 1 < ny) acc += A->n[k] * x[k + nx];
            }
            y[k] = acc;
        }
}

/* residual, stencil.cpp:148-153: r = b - Ax */
static void op_residual(const grid_t* g, const op_t* A, const double* x, const double* b, double* r) {
    op_apply(g, A, x, r);
    const size_t n = nlev(g);
    for (size_t k = 0; k < n; ++k) r[k] = b[k] - r[k];
}

/* ---- banded Cholesky: stencil.cpp:155-210 -------------------------------- */

static int chol_factor(orc_problem* p) {
    const grid_t* g = &p->g[0];
    const op_t* A = &p->op[0];
    const int n = (int)nlev(g), nx = g->nx;
    const int bw = g->per ? n - 1 : g->nx; /* periodic: the dense lower triangle */
    p->chol_n = n;
    p->chol_bw = bw;
    p->band = dalloc((size_t)(bw + 1) * n);
    double* B = p->band;
#define ENT(d, k) B[(size_t)(d) * n + (k)]
    if (g->per) {
        /* couplings accumulated in apply's order c, w, e, s, n with y wrapped */
        const int ny = g->ny;
        double* D = dalloc((size_t)n * n);
        for (int k = 0; k < n; ++k) {
            const int i = k % nx, j = k / nx;
            D[(size_t)k * n + k] = D[(size_t)k * n + k] + A->c[k];
            if (i > 0) D[(size_t)k * n + k - 1] = D[(size_t)k * n + k - 1] + A->w[k];
            if (i + 1 < nx) D[(size_t)k * n + k + 1] = D[(size_t)k * n + k + 1] + A->e[k];
            const int ks = ((j + ny - 1) % ny) * nx + i, kn = ((j + 1) % ny) * nx + i;
            D[(size_t)k * n + ks] = D[(size_t)k * n + ks] + A->s[k];
            D[(size_t)k * n + kn] = D[(size_t)k * n + kn] + A->n[k];
        }
        for (int k = 0; k < n; ++k)
            for (int d = 0; d <= k; ++d) ENT(d, k) = D[(size_t)k * n + k - d];
        free(D);
    } else {
        for (int k = 0; k < n; ++k) {
            ENT(0, k) = A->c[k];
            if (k % nx != 0) ENT(1, k) = A->w[k];
            if (k >= nx) ENT(bw, k) = A->s[k];
        }
    }
    for (int jc = 0; jc < n; ++jc) {
        double d = ENT(0, jc);
        for (int m = jc - bw > 0 ? jc - bw : 0; m < jc; ++m) {
            const double l = ENT(jc - m, jc);
            d -= l * l;
        }
        if (!(d > 0.0)) return fail(ORC_ERR_RUNTIME, "BandedCholesky: matrix not positive definite");
        const double ljj = sqrt(d);
        ENT(0, jc) = ljj;
        const int last = n - 1 < jc + bw ? n - 1 : jc + bw;
        for (int ir = jc + 1; ir <= last; ++ir) {
            double a = ENT(ir - jc, ir);
            for (int m = ir - bw > 0 ? ir - bw : 0; m < jc; ++m) a -= ENT(ir - m, ir) * ENT(jc - m, jc);
            ENT(ir - jc, ir) = a / ljj;
        }
    }
    return ORC_OK;
}

static void chol_solve(const orc_problem* p, const double* b, double* x) {
    const int n = p->chol_n, bw = p->chol_bw;
    const double* B = p->band;
    for (int k = 0; k < n; ++k) {
        double acc = b[k];
        const int dm = bw < k ? bw : k;
        for (int d = 1; d <= dm; ++d) acc -= ENT(d, k) * x[k - d];
        x[k] = acc / ENT(0, k);
    }
    for (int k = n - 1; k >= 0; --k) {
        double acc = x[k];
        const int dm = bw < n - 1 - k ? bw : n - 1 - k;
        for (int d = 1; d <= dm; ++d) acc -= ENT(d, k + d) * x[k + d];
        x[k] = acc / ENT(0, k);
    }
#undef ENT
}

/* ---- transfers: transfer.cpp:26-101 -------------------------------------- */

static double odd_weight(const double* xf, const double* xc, int q) {
    return (xf[2 * q + 1] - xc[q]) / (xc[q + 1] - xc[q]);
}

static int require_nested(const grid_t* c, const grid_t* f) {
    const int fny = f->per ? 2 * c->ny : 2 * c->ny + 1;
    if (f->level != c->level + 1 || f->nx != 2 * c->nx + 1 || f->ny != fny)
        return fail(ORC_ERR_LOGIC, "levels are not parent and child");
    return ORC_OK;
}

/* periodic y: coarse node 0 is coarse node cny (y = 0 == 1) */
static double prolong_cv(const grid_t* cg, const double* cv, int qx, int qy) {
    if (cg->per && qy == 0) qy = cg->ny;
    if (qx < 1 || qx > cg->nx || qy < 1 || qy > cg->ny) return 0.0;
    return cv[(size_t)(qy - 1) * cg->nx + (qx - 1)];
}

static void prolong(const grid_t* cg, const grid_t* fg, const double* cv, double* fv) {
#define CV(qx, qy) prolong_cv(cg, cv, (qx), (qy))
    for (int j = 0; j < fg->ny; ++j) {
        const int pj = j + 1;
        for (int i = 0; i < fg->nx; ++i) {
            const int pi = i + 1;
            double val;
            if (pi % 2 == 0 && pj % 2 == 0) {
                val = CV(pi / 2, pj / 2);
            } else if (pi % 2 == 1 && pj % 2 == 0) {
                const int qx = (pi - 1) / 2;
                const double t = odd_weight(fg->x, cg->x, qx);
                val = (1.0 - t) * CV(qx, pj / 2) + t * CV(qx + 1, pj / 2);
            } else if (pi % 2 == 0 && pj % 2 == 1) {
                const int qy = (pj - 1) / 2;
                const double t = odd_weight(fg->y, cg->y, qy);
                val = (1.0 - t) * CV(pi / 2, qy) + t * CV(pi / 2, qy + 1);
            } else {
                const int qx = (pi - 1) / 2, qy = (pj - 1) / 2;
                const double tx = odd_weight(fg->x, cg->x, qx);
                const double ty = odd_weight(fg->y, cg->y, qy);
                val = (1.0 - tx) * (1.0 - ty) * CV(qx, qy) + tx * (1.0 - ty) * CV(qx + 1, qy) +
                      (1.0 - tx) * ty * CV(qx, qy + 1) + tx * ty * CV(qx + 1, qy + 1);
            }
            fv[(size_t)j * fg->nx + i] = val;
        }
    }
#undef CV
}

static void restrict_(const grid_t* fg, const grid_t* cg, const double* fv, double* cv) {
    const int fnx = fg->nx;
    for (int qj = 1; qj <= cg->ny; ++qj) {
        const double wys = odd_weight(fg->y, cg->y, qj - 1);
        const double wyn = 1.0 - odd_weight(fg->y, cg->y, qj);
        const double sy = wys + 1.0 + wyn;
        for (int qi = 1; qi <= cg->nx; ++qi) {
            const double wxw = odd_weight(fg->x, cg->x, qi - 1);
            const double wxe = 1.0 - odd_weight(fg->x, cg->x, qi);
            const double sx = wxw + 1.0 + wxe;
            const double wx[3] = {wxw, 1.0, wxe};
            const double wy[3] = {wys, 1.0, wyn};
            double acc = 0.0;
            for (int dj = -1; dj <= 1; ++dj)
                for (int di = -1; di <= 1; ++di)
                    acc += wx[di + 1] * wy[dj + 1] *
                           fv[(size_t)(fg->per ? (2 * qj + dj - 1) % fg->ny : 2 * qj + dj - 1) * fnx +
                              (2 * qi + di - 1)];
            cv[(size_t)(qj - 1) * cg->nx + (qi - 1)] = acc / (sx * sy);
        }
    }
}

/* ---- smoothers: smoother.cpp ---------------------------------------------- */

/* mt19937 + uniform_real_distribution<double>(-1,1) as libstdc++ computes it
 * (generate_canonical with two 32-bit draws). */
typedef struct {
    uint32_t mt[624];
    int idx;
} mt_t;
static void mt_seed(mt_t* m, uint32_t s) {
    m->mt[0] = s;
    for (int i = 1; i < 624; ++i) m->mt[i] = 1812433253u * (m->mt[i - 1] ^ (m->mt[i - 1] >> 30)) + (uint32_t)i;
    m->idx = 624;
}
static uint32_t mt_next(mt_t* m) {
    if (m->idx >= 624) {
        for (int i = 0; i < 624; ++i) {
            uint32_t y = (m->mt[i] & 0x80000000u) | (m->mt[(i + 1) % 624] & 0x7fffffffu);
            m->mt[i] = m->mt[(i + 397) % 624] ^ (y >> 1) ^ ((y & 1u) ? 0x9908b0dfu : 0u);
        }
        m->idx = 0;
    }
    uint32_t y = m->mt[m->idx++];
    y ^= y >> 11;
    y ^= (y << 7) & 0x9d2c5680u;
    y ^= (y << 15) & 0xefc60000u;
    y ^= y >> 18;
    return y;
}
static double mt_uniform(mt_t* m) {
    double sum = 0.0, tmp = 1.0;
    for (int k = 0; k < 2; ++k) {
        sum += (double)mt_next(m) * tmp;
        tmp *= 4294967296.0;
    }
    double r = sum / tmp;
    if (r >= 1.0) r = nextafter(1.0, 0.0);
    return (1.0 - -1.0) * r + -1.0;
}
void orc_random_vector(long long n, unsigned seed, double* out) {
    mt_t m;
    mt_seed(&m, seed);
    for (long long k = 0; k < n; ++k) out[k] = mt_uniform(&m);
}

typedef struct {
    int kind;
    double omega;
    const grid_t* g;
    const op_t* A;
    double* ws; /* line factors (3*neq per direction) or ILU(0) diagonals (5*neq) */
    double rich_omega;
} smoother_t;

static int uses_x_lines(int k) { return k == K_TRIX || k == K_ADI || k == K_GSTRIX || k == K_GSADI; }
static int uses_y_lines(int k) { return k == K_TRIY || k == K_ADI || k == K_GSTRIY || k == K_GSADI; }

/* check_omega, smoother.cpp:51-69 */
static int check_omega(int kind, double w) {
    switch (kind) {
        case K_RICH:
        case K_JACOBI:
        case K_ILU0:
            if (!(w > 0.0)) return fail(ORC_ERR_INVALID, "smoother_omega: must be > 0");
            return ORC_OK;
        case K_GS:
        case K_SOR:
            if (!(w > 0.0 && w < 2.0))
                return fail(ORC_ERR_INVALID, "smoother_omega: must be in (0, 2) for gauss_seidel/sor");
            return ORC_OK;
        default:
            if (!(w > 0.0 && w <= 1.0))
                return fail(ORC_ERR_INVALID, "smoother_omega: must be in (0, 1] for line smoothers");
            return ORC_OK;
    }
}

/* factor_lines_x / factor_lines_y, smoother.cpp:74-115 */
static int factor_x(const grid_t* g, const op_t* A, double om, double* sub, double* dg, double* sup) {
    const int nx = g->nx, ny = g->ny;
    for (int j = 0; j < ny; ++j) {
        const size_t b = (size_t)j * nx;
        for (int i = 0; i < nx; ++i) {
            dg[b + i] = om * A->c[b + i];
            sub[b + i] = om * A->w[b + i];
            sup[b + i] = om * A->e[b + i];
        }
        for (int i = 1; i < nx; ++i) {
            const size_t k = b + i;
            if (dg[k - 1] == 0.0) return fail(ORC_ERR_RUNTIME, "tri factorization: zero pivot");
            const double m = sub[k] / dg[k - 1];
            dg[k] -= m * sup[k - 1];
            sub[k] = m;
        }
    }
    return ORC_OK;
}
static int factor_y(const grid_t* g, const op_t* A, double om, double* sub, double* dg, double* sup) {
    const int nx = g->nx, ny = g->ny;
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < ny; ++j) {
            const size_t k = (size_t)j * nx + i;
            dg[k] = om * A->c[k];
            sub[k] = om * A->s[k];
            sup[k] = om * A->n[k];
        }
        for (int j = 1; j < ny; ++j) {
            const size_t k = (size_t)j * nx + i, km = k - nx;
            if (dg[km] == 0.0) return fail(ORC_ERR_RUNTIME, "tri factorization: zero pivot");
            const double m = sub[k] / dg[km];
            dg[k] -= m * sup[km];
            sub[k] = m;
        }
    }
    return ORC_OK;
}

/* solve_one_line_x / _y, smoother.cpp:117-138 */
static void line_x(int j, int nx, const double* sub, const double* dg, const double* sup, double* z) {
    const size_t b = (size_t)j * nx;
    for (int i = 1; i < nx; ++i) z[b + i] -= sub[b + i] * z[b + i - 1];
    z[b + nx - 1] /= dg[b + nx - 1];
    for (int i = nx - 2; i >= 0; --i) z[b + i] = (z[b + i] - sup[b + i] * z[b + i + 1]) / dg[b + i];
}
static void line_y(int i, int nx, int ny, const double* sub, const double* dg, const double* sup, double* z) {
    for (int j = 1; j < ny; ++j) {
        const size_t k = (size_t)j * nx + i;
        z[k] -= sub[k] * z[k - nx];
    }
    const size_t last = (size_t)(ny - 1) * nx + i;
    z[last] /= dg[last];
    for (int j = ny - 2; j >= 0; --j) {
        const size_t k = (size_t)j * nx + i;
        z[k] = (z[k] - sup[k] * z[k + nx]) / dg[k];
    }
}

/* factor_ilu0, smoother.cpp:187-210 */
static int factor_ilu0(const grid_t* g, const op_t* A, double* lw, double* ls, double* d, double* ue, double* un) {
    const int nx = g->nx, ny = g->ny;
    for (int j = 0; j < ny; ++j)
        for (int i = 0; i < nx; ++i) {
            const size_t k = (size_t)j * nx + i;
            double piv = A->c[k];
            lw[k] = 0.0;
            ls[k] = 0.0;
            if (i > 0) {
                lw[k] = A->w[k] / d[k - 1];
                piv -= lw[k] * ue[k - 1];
            }
            if (j > 0) {
                ls[k] = A->s[k] / d[k - nx];
                piv -= ls[k] * un[k - nx];
            }
            if (piv <= 0.0) return fail(ORC_ERR_RUNTIME, "ilu0 factorization: nonpositive pivot");
            d[k] = piv;
            ue[k] = A->e[k];
            un[k] = A->n[k];
        }
    return ORC_OK;
}

/* setup, smoother.cpp:231-276 (richardson power iteration :212-227) */
static int sm_setup(smoother_t* s, int kind, double omega, const grid_t* g, const op_t* A) {
    memset(s, 0, sizeof *s);
    int st = check_omega(kind, omega);
    if (st) return st;
    if (g->per && kind != K_JACOBI && kind != K_RICH)
        return fail(ORC_ERR_INVALID, "smoother: periodic (polar) grids support jacobi and richardson only");
    s->kind = kind;
    s->omega = omega;
    s->g = g;
    s->A = A;
    const size_t n = nlev(g);
    if (kind == K_RICH) {
        double* x = dalloc(n);
        double* y = dalloc(n);
        mt_t m;
        mt_seed(&m, 0x2d5a11u);
        for (size_t k = 0; k < n; ++k) x[k] = mt_uniform(&m);
        double lambda = 0.0;
        for (int t = 0; t < 20; ++t) {
            op_apply(g, A, x, y);
            lambda = orc_norm_l2((long long)n, y);
            if (lambda == 0.0) break;
            for (size_t k = 0; k < n; ++k) y[k] /= lambda;
            double* tmp = x;
            x = y;
            y = tmp;
        }
        free(x);
        free(y);
        s->rich_omega = (lambda > 0.0 && omega > 1.0 / lambda) ? 0.9 / lambda : omega;
    } else if (kind == K_ILU0) {
        s->ws = dalloc(5 * n);
        st = factor_ilu0(g, A, s->ws, s->ws + n, s->ws + 2 * n, s->ws + 3 * n, s->ws + 4 * n);
    } else if (kind != K_JACOBI && kind != K_GS && kind != K_SOR) {
        const int fx = uses_x_lines(kind), fy = uses_y_lines(kind);
        s->ws = dalloc(3 * n * (size_t)(fx + fy));
        double* q = s->ws;
        if (fx) {
            st = factor_x(g, A, omega, q, q + n, q + 2 * n);
            q += 3 * n;
        }
        if (!st && fy) st = factor_y(g, A, omega, q, q + n, q + 2 * n);
    }
    return st;
}
static void sm_free(smoother_t* s) { free(s->ws); }

static void gstri_x(const smoother_t* sm, const double* q, const double* r, double* z) {
    const int nx = sm->g->nx, ny = sm->g->ny;
    const size_t n = nlev(sm->g);
    for (int j = 0; j < ny; ++j) {
        const size_t b = (size_t)j * nx;
        for (int i = 0; i < nx; ++i) {
            double rhs = r[b + i];
            if (j > 0) rhs -= sm->omega * sm->A->s[b + i] * z[b + i - nx];
            z[b + i] = rhs;
        }
        line_x(j, nx, q, q + n, q + 2 * n, z);
    }
}
static void gstri_y(const smoother_t* sm, const double* q, const double* r, double* z) {
    const int nx = sm->g->nx, ny = sm->g->ny;
    const size_t n = nlev(sm->g);
    for (int i = 0; i < nx; ++i) {
        for (int j = 0; j < ny; ++j) {
            const size_t k = (size_t)j * nx + i;
            double rhs = r[k];
            if (i > 0) rhs -= sm->omega * sm->A->w[k] * z[k - 1];
            z[k] = rhs;
        }
        line_y(i, nx, ny, q, q + n, q + 2 * n, z);
    }
}

/* apply_preconditioner, smoother.cpp:278-387: z = C^{-1} r */
static void precond(const smoother_t* sm, const double* r, double* z) {
    const grid_t* g = sm->g;
    const op_t* A = sm->A;
    const int nx = g->nx, ny = g->ny;
    const size_t n = nlev(g);
    const double om = sm->omega;
    memset(z, 0, n * sizeof(double));
    switch (sm->kind) {
        case K_RICH:
            for (size_t k = 0; k < n; ++k) z[k] = sm->rich_omega * r[k];
            break;
        case K_JACOBI:
            for (size_t k = 0; k < n; ++k) z[k] = r[k] / A->c[k];
            break;
        case K_GS:
        case K_SOR:
            for (int j = 0; j < ny; ++j)
                for (int i = 0; i < nx; ++i) {
                    const size_t k = (size_t)j * nx + i;
                    double acc = r[k];
                    if (i > 0) acc -= om * A->w[k] * z[k - 1];
                    if (j > 0) acc -= om * A->s[k] * z[k - nx];
                    z[k] = acc / A->c[k];
                }
            break;
        case K_ILU0: {
            const double *lw = sm->ws, *ls = lw + n, *d = lw + 2 * n, *ue = lw + 3 * n, *un = lw + 4 * n;
            for (int j = 0; j < ny; ++j)
                for (int i = 0; i < nx; ++i) {
                    const size_t k = (size_t)j * nx + i;
                    double acc = r[k];
                    if (i > 0) acc -= lw[k] * z[k - 1];
                    if (j > 0) acc -= ls[k] * z[k - nx];
                    z[k] = acc;
                }
            for (int j = ny - 1; j >= 0; --j)
                for (int i = nx - 1; i >= 0; --i) {
                    const size_t k = (size_t)j * nx + i;
                    double acc = z[k];
                    if (i + 1 < nx) acc -= ue[k] * z[k + 1];
                    if (j + 1 < ny) acc -= un[k] * z[k + nx];
                    z[k] = acc / d[k];
                }
            break;
        }
        case K_TRIX:
            memcpy(z, r, n * sizeof(double));
            for (int j = 0; j < ny; ++j) line_x(j, nx, sm->ws, sm->ws + n, sm->ws + 2 * n, z);
            break;
        case K_TRIY:
            memcpy(z, r, n * sizeof(double));
            for (int i = 0; i < nx; ++i) line_y(i, nx, ny, sm->ws, sm->ws + n, sm->ws + 2 * n, z);
            break;
        case K_ADI:
        case K_GSADI: {
            const double* px = sm->ws;
            const double* py = px + 3 * n;
            if (sm->kind == K_ADI) {
                memcpy(z, r, n * sizeof(double));
                for (int j = 0; j < ny; ++j) line_x(j, nx, px, px + n, px + 2 * n, z);
            } else {
                gstri_x(sm, px, r, z);
            }
            double* t = dalloc(n);
            double* z2 = dalloc(n);
            op_residual(g, A, z, r, t);
            if (sm->kind == K_ADI) {
                memcpy(z2, t, n * sizeof(double));
                for (int i = 0; i < nx; ++i) line_y(i, nx, ny, py, py + n, py + 2 * n, z2);
            } else {
                gstri_y(sm, py, t, z2);
            }
            for (size_t k = 0; k < n; ++k) z[k] += z2[k];
            free(t);
            free(z2);
            break;
        }
        case K_GSTRIX:
            gstri_x(sm, sm->ws, r, z);
            break;
        case K_GSTRIY:
            gstri_y(sm, sm->ws, r, z);
            break;
    }
}

/* smooth_step, smoother.cpp:389-399: x - omega_damp * C^{-1}(Ax - b) */
static int sm_step(const smoother_t* sm, const double* x, const double* b, double omega_damp, double* out) {
    if (!(omega_damp > 0.0)) return fail(ORC_ERR_INVALID, "omega: damping must be > 0");
    const size_t n = nlev(sm->g);
    double* d = dalloc(n);
    double* z = dalloc(n);
    op_apply(sm->g, sm->A, x, d);
    for (size_t k = 0; k < n; ++k) d[k] -= b[k];
    precond(sm, d, z);
    for (size_t k = 0; k < n; ++k) out[k] = x[k] - omega_damp * z[k];
    free(d);
    free(z);
    return ORC_OK;
}

/* ---- problem ----------------------------------------------------------- */

orc_problem* orc_problem_create(int levels, int cnx, int cny, double fx, double fy, int coords,
                                double alpha, double beta) {
    if (levels < 1) { fail(ORC_ERR_INVALID, "levels: must be >= 1"); return NULL; }
    if (cnx < 1 || cny < 1) { fail(ORC_ERR_INVALID, "coarse_n: interior counts must be >= 1"); return NULL; }
    if (!(fx > 0.0) || !(fy > 0.0)) { fail(ORC_ERR_INVALID, "grading: factors must be > 0"); return NULL; }
    if (!(alpha > 0.0) || !(beta > 0.0)) { fail(ORC_ERR_INVALID, "alpha/beta must be > 0"); return NULL; }
    if (coords < CS_CART || coords > CS_POLAR) { fail(ORC_ERR_INVALID, "coords: unknown coordinate system"); return NULL; }
    if (coords == CS_POLAR && fy != 1.0) {
        fail(ORC_ERR_INVALID, "grading_y: the periodic polar theta axis must be uniform");
        return NULL;
    }
    if (coords == CS_POLAR && cny < 2) {
        fail(ORC_ERR_INVALID, "coarse_n: the periodic polar theta axis needs >= 2 nodes");
        return NULL;
    }
    orc_problem* p = (orc_problem*)calloc(1, sizeof *p);
    p->L = levels;
    p->g = (grid_t*)calloc((size_t)levels, sizeof(grid_t));
    p->op = (op_t*)calloc((size_t)levels, sizeof(op_t));
    /* build_hierarchy, mesh.cpp:103-138 */
    grid_t* f = &p->g[levels - 1];
    f->level = levels;
    f->nx = ((cnx + 1) << (levels - 1)) - 1;
    f->ny = coords == CS_POLAR ? cny << (levels - 1) : ((cny + 1) << (levels - 1)) - 1;
    f->coords = coords;
    f->per = coords == CS_POLAR;
    f->x = dalloc((size_t)f->nx + 2);
    f->y = dalloc((size_t)f->ny + 2);
    if (physical_axis(f->nx, fx, coords, 0, f->x) ||
        (!f->per && physical_axis(f->ny, fy, coords, 1, f->y))) {
        orc_problem_destroy(p);
        return NULL;
    }
    if (f->per)
        for (int q = 0; q <= f->ny + 1; ++q) f->y[q] = (double)q / (double)f->ny;
    for (int l = levels - 1; l >= 1; --l) {
        const grid_t* fg = &p->g[l];
        grid_t* cg = &p->g[l - 1];
        cg->level = l;
        cg->nx = (fg->nx - 1) / 2;
        cg->ny = fg->per ? fg->ny / 2 : (fg->ny - 1) / 2;
        cg->coords = coords;
        cg->per = fg->per;
        cg->x = dalloc((size_t)cg->nx + 2);
        cg->y = dalloc((size_t)cg->ny + 2);
        for (int q = 0; q < cg->nx + 2; ++q) cg->x[q] = fg->x[2 * q];
        if (cg->per)
            for (int q = 0; q <= cg->ny + 1; ++q) cg->y[q] = (double)q / (double)cg->ny;
        else
            for (int q = 0; q < cg->ny + 2; ++q) cg->y[q] = fg->y[2 * q];
    }
    /* MultilevelProblem, cycle.cpp:25-30 */
    for (int l = 0; l < levels; ++l) assemble(&p->g[l], alpha, beta, &p->op[l]);
    if (chol_factor(p)) {
        orc_problem_destroy(p);
        return NULL;
    }
    return p;
}

void orc_problem_destroy(orc_problem* p) {
    if (!p) return;
    for (int l = 0; l < p->L; ++l) {
        free(p->g[l].x);
        free(p->g[l].y);
        free(p->op[l].c);
        free(p->op[l].n);
        free(p->op[l].s);
        free(p->op[l].e);
        free(p->op[l].w);
    }
    free(p->g);
    free(p->op);
    free(p->band);
    free(p);
}

int orc_num_levels(const orc_problem* p) { return p->L; }

static int bad_level(const orc_problem* p, int l) { return l < 1 || l > p->L; }

int orc_level_shape(const orc_problem* p, int level, int* nx, int* ny) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "level out of range");
    *nx = p->g[level - 1].nx;
    *ny = p->g[level - 1].ny;
    return ORC_OK;
}

int orc_level_coords(const orc_problem* p, int level, double* x, double* y) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "level out of range");
    const grid_t* g = &p->g[level - 1];
    memcpy(x, g->x, ((size_t)g->nx + 2) * sizeof(double));
    memcpy(y, g->y, ((size_t)g->ny + 2) * sizeof(double));
    return ORC_OK;
}

int orc_operator(const orc_problem* p, int level, double* c, double* n, double* s, double* e, double* w) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "level out of range");
    const size_t nb = nlev(&p->g[level - 1]) * sizeof(double);
    const op_t* A = &p->op[level - 1];
    memcpy(c, A->c, nb);
    memcpy(n, A->n, nb);
    memcpy(s, A->s, nb);
    memcpy(e, A->e, nb);
    memcpy(w, A->w, nb);
    return ORC_OK;
}

int orc_apply(const orc_problem* p, int level, const double* x, double* y) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "apply: grid function does not match operator level");
    op_apply(&p->g[level - 1], &p->op[level - 1], x, y);
    return ORC_OK;
}

int orc_residual(const orc_problem* p, int level, const double* x, const double* b, double* r) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "residual: grid functions live on different levels");
    op_residual(&p->g[level - 1], &p->op[level - 1], x, b, r);
    return ORC_OK;
}

int orc_smooth_step(const orc_problem* p, int level, int kind, double somega, double damp,
                    const double* x, const double* b, double* out) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "smooth_step: level out of range");
    smoother_t sm;
    int st = sm_setup(&sm, kind, somega, &p->g[level - 1], &p->op[level - 1]);
    if (!st) st = sm_step(&sm, x, b, damp, out);
    sm_free(&sm);
    return st;
}

int orc_restriction(const orc_problem* p, int fine_level, const double* fine, double* coarse) {
    if (fine_level < 2 || fine_level > p->L) return fail(ORC_ERR_LOGIC, "restriction: levels are not parent and child");
    int st = require_nested(&p->g[fine_level - 2], &p->g[fine_level - 1]);
    if (st) return st;
    restrict_(&p->g[fine_level - 1], &p->g[fine_level - 2], fine, coarse);
    return ORC_OK;
}

int orc_prolongation(const orc_problem* p, int coarse_level, const double* coarse, double* fine) {
    if (coarse_level < 1 || coarse_level >= p->L) return fail(ORC_ERR_LOGIC, "prolongation: levels are not parent and child");
    int st = require_nested(&p->g[coarse_level - 1], &p->g[coarse_level]);
    if (st) return st;
    prolong(&p->g[coarse_level - 1], &p->g[coarse_level], coarse, fine);
    return ORC_OK;
}

/* adaptive_omega, cycle.cpp:40-51 */
static int adaptive_omega(const grid_t* g, const op_t* A, const double* d, const double* corr, double* w) {
    const size_t n = nlev(g);
    double nc = 0.0;
    for (size_t k = 0; k < n; ++k) nc += corr[k] * corr[k];
    if (nc == 0.0) {
        *w = 1.0;
        return ORC_OK;
    }
    double* ac = dalloc(n);
    op_apply(g, A, corr, ac);
    const double den = orc_dot((long long)n, ac, corr);
    free(ac);
    if (!(den > 0.0)) return fail(ORC_ERR_RUNTIME, "adaptive_omega: correction has nonpositive energy");
    *w = orc_dot((long long)n, d, corr) / den;
    return ORC_OK;
}

int orc_adaptive_omega(const orc_problem* p, int level, const double* d, const double* corr, double* omega) {
    if (bad_level(p, level)) return fail(ORC_ERR_LOGIC, "adaptive_omega: grid functions live on different levels");
    return adaptive_omega(&p->g[level - 1], &p->op[level - 1], d, corr, omega);
}

int orc_coarse_solve(const orc_problem* p, const double* b, double* x) {
    chol_solve(p, b, x);
    return ORC_OK;
}

/* ---- cycles: cycle.cpp:57-194 -------------------------------------------- */

typedef struct {
    const orc_problem* p;
    const orc_cycle* spec;
    int cycle; /* the effective cycle type (fcycle_pass forces V, cycle.cpp:129-130) */
    smoother_t* sm;
} ctx_t;

/* coarse_solve, cycle.cpp:57-65 */
static int coarse_solve(const ctx_t* c, const double* u0, const double* g, double* u) {
    const grid_t* g1 = &c->p->g[0];
    const size_t n = nlev(g1);
    if ((unsigned long long)n <= c->spec->coarse_direct_max_neq) {
        chol_solve(c->p, g, u);
        return ORC_OK;
    }
    memcpy(u, u0, n * sizeof(double));
    int steps = c->spec->pre_steps + c->spec->post_steps;
    if (steps < 1) steps = 1;
    double* t = dalloc(n);
    for (int s = 0; s < steps; ++s) {
        int st = sm_step(&c->sm[0], u, g, c->spec->smoothing_omega, t);
        if (st) { free(t); return st; }
        memcpy(u, t, n * sizeof(double));
    }
    free(t);
    return ORC_OK;
}

/* mg_cycle, cycle.cpp:69-100 */
static int mg_cycle(const ctx_t* c, int level, const double* u0, const double* g, double* uout) {
    if (level < 1 || level > c->p->L) return fail(ORC_ERR_LOGIC, "mg_cycle: missing level data");
    if (c->spec->pre_steps + c->spec->post_steps < 1)
        return fail(ORC_ERR_INVALID, "pre_steps/post_steps: at least one smoothing step per visit");
    if (level == 1) return coarse_solve(c, u0, g, uout);
    const grid_t* gr = &c->p->g[level - 1];
    const grid_t* cg = &c->p->g[level - 2];
    const op_t* A = &c->p->op[level - 1];
    const smoother_t* sm = &c->sm[level - 1];
    const size_t n = nlev(gr), nc = nlev(cg);
    double* u = dalloc(n);
    double* t = dalloc(n);
    double* d = dalloc(n);
    double* gc = dalloc(nc);
    double* uc = dalloc(nc);
    double* uc2 = dalloc(nc);
    double* corr = dalloc(n);
    int st = ORC_OK;
    memcpy(u, u0, n * sizeof(double));
    for (int s = 0; s < c->spec->pre_steps && !st; ++s) {
        st = sm_step(sm, u, g, c->spec->smoothing_omega, t);
        memcpy(u, t, n * sizeof(double));
    }
    if (!st) {
        op_residual(gr, A, u, g, d);
        restrict_(gr, cg, d, gc);
        const int reps = c->cycle == 1 ? 2 : 1;
        for (int i = 0; i < reps && !st; ++i) {
            st = mg_cycle(c, level - 1, uc, gc, uc2);
            memcpy(uc, uc2, nc * sizeof(double));
        }
    }
    if (!st) {
        prolong(cg, gr, uc, corr);
        double wl = c->spec->correction_omega;
        if (c->spec->adaptive_correction) st = adaptive_omega(gr, A, d, corr, &wl);
        if (!st) orc_axpy((long long)n, wl, corr, u);
    }
    for (int s = 0; s < c->spec->post_steps && !st; ++s) {
        st = sm_step(sm, u, g, c->spec->smoothing_omega, t);
        memcpy(u, t, n * sizeof(double));
    }
    if (!st) memcpy(uout, u, n * sizeof(double));
    free(u); free(t); free(d); free(gc); free(uc); free(uc2); free(corr);
    return st;
}

/* fcycle_pass, cycle.cpp:119-142 */
static int fcycle_pass(ctx_t* c, const double* x, const double* b, double* xout) {
    const orc_problem* p = c->p;
    const int L = p->L;
    if (L == 1) return mg_cycle(c, 1, x, b, xout);
    double** def = (double**)calloc((size_t)L + 1, sizeof(double*));
    for (int l = 1; l <= L; ++l) def[l] = dalloc(nlev(&p->g[l - 1]));
    op_residual(&p->g[L - 1], &p->op[L - 1], x, b, def[L]);
    for (int l = L; l >= 2; --l) restrict_(&p->g[l - 1], &p->g[l - 2], def[l], def[l - 1]);
    const int saved = c->cycle;
    c->cycle = 0; /* V */
    double* z1 = dalloc(nlev(&p->g[0]));
    double* e = dalloc(nlev(&p->g[0]));
    int st = mg_cycle(c, 1, z1, def[1], e);
    free(z1);
    for (int l = 2; l <= L && !st; ++l) {
        const size_t n = nlev(&p->g[l - 1]);
        double* el = dalloc(n);
        double* en = dalloc(n);
        prolong(&p->g[l - 2], &p->g[l - 1], e, el);
        st = mg_cycle(c, l, el, def[l], en);
        free(el);
        free(e);
        e = en;
    }
    c->cycle = saved;
    if (!st) {
        const size_t n = nlev(&p->g[L - 1]);
        memcpy(xout, x, n * sizeof(double));
        orc_axpy((long long)n, 1.0, e, xout);
    }
    free(e);
    for (int l = 1; l <= L; ++l) free(def[l]);
    free(def);
    return st;
}

static int setup_all(const orc_problem* p, const orc_cycle* spec, smoother_t** out) {
    smoother_t* sm = (smoother_t*)calloc((size_t)p->L, sizeof(smoother_t));
    for (int l = 0; l < p->L; ++l) {
        int st = sm_setup(&sm[l], spec->smoother_kind, spec->smoother_omega, &p->g[l], &p->op[l]);
        if (st) {
            for (int q = 0; q <= l; ++q) sm_free(&sm[q]);
            free(sm);
            return st;
        }
    }
    *out = sm;
    return ORC_OK;
}

int orc_mg_cycle(const orc_problem* p, const orc_cycle* spec, int level, const double* u0,
                 const double* g, double* u) {
    smoother_t* sm = NULL;
    int st = setup_all(p, spec, &sm);
    if (st) return st;
    ctx_t c = {p, spec, spec->cycle, sm};
    st = mg_cycle(&c, level, u0, g, u);
    for (int l = 0; l < p->L; ++l) sm_free(&sm[l]);
    free(sm);
    return st;
}

/* solve, cycle.cpp:146-194 */
int orc_solve(const orc_problem* p, const orc_cycle* spec, const double* b, double* x,
              double* hist, int* hist_len, int* iterations, int* converged) {
    const int L = p->L;
    const grid_t* g = &p->g[L - 1];
    const op_t* A = &p->op[L - 1];
    const size_t n = nlev(g);
    *hist_len = 0;
    *iterations = 0;
    *converged = 0;
    smoother_t* sm = NULL;
    int st = setup_all(p, spec, &sm);
    if (st) return st;
    ctx_t c = {p, spec, spec->cycle, sm};
    double* r = dalloc(n);
    double* xn = dalloc(n);
    op_residual(g, A, x, b, r);
    const double r0 = orc_norm_l2((long long)n, r);
    hist[(*hist_len)++] = r0;
    const double bnorm = orc_norm_l2((long long)n, b);
    const double ref = bnorm > 0.0 ? bnorm : r0;
    if (r0 <= spec->tolerance * ref) {
        *converged = 1;
        goto done;
    }
    for (int k = 1; k <= spec->max_cycles; ++k) {
        if (spec->cycle == 2)
            st = fcycle_pass(&c, x, b, xn);
        else
            st = mg_cycle(&c, L, x, b, xn);
        if (st) break;
        memcpy(x, xn, n * sizeof(double));
        op_residual(g, A, x, b, r);
        const double rk = orc_norm_l2((long long)n, r);
        hist[(*hist_len)++] = rk;
        *iterations = k;
        if (rk <= spec->tolerance * ref) {
            *converged = 1;
            break;
        }
        if (rk > 1e6 * (r0 > ref ? r0 : ref)) {
            st = fail(ORC_DIVERGED, "solve: residual grew beyond 1e6 times the initial residual");
            break;
        }
    }
done:
    free(r);
    free(xn);
    for (int l = 0; l < L; ++l) sm_free(&sm[l]);
    free(sm);
    return st;
}

/* make_start_vector, study.cpp:40-79: kind 0 zero, 1 nested (a direct level-1
 * solve of the restricted right-hand side, then prolongation + one smooth_step
 * per level, study.cpp:46-58). Continuation (kind 2) is a host copy and has no
 * arithmetic of its own. */
int orc_start_vector(const orc_problem* p, const orc_cycle* spec, int kind, const double* b, double* x) {
    const int L = p->L;
    const size_t nL = nlev(&p->g[L - 1]);
    if (kind == 0) {
        memset(x, 0, nL * sizeof(double));
        return ORC_OK;
    }
    if (kind != 1) return fail(ORC_ERR_INVALID, "start: kind must be zero or nested");
    if (L == 1) {
        chol_solve(p, b, x);
        return ORC_OK;
    }
    double** rhs = (double**)calloc((size_t)L + 1, sizeof(double*));
    rhs[L] = dalloc(nL);
    memcpy(rhs[L], b, nL * sizeof(double));
    for (int l = L; l >= 2; --l) {
        rhs[l - 1] = dalloc(nlev(&p->g[l - 2]));
        restrict_(&p->g[l - 1], &p->g[l - 2], rhs[l], rhs[l - 1]);
    }
    smoother_t* sm = NULL;
    int st = setup_all(p, spec, &sm);
    if (st) goto out;
    {
        double* u = dalloc(nlev(&p->g[0]));
        chol_solve(p, rhs[1], u);
        for (int l = 2; l <= L && !st; ++l) {
            const size_t n = nlev(&p->g[l - 1]);
            double* pu = dalloc(n);
            prolong(&p->g[l - 2], &p->g[l - 1], u, pu);
            free(u);
            u = dalloc(n);
            st = sm_step(&sm[l - 1], pu, rhs[l], spec->smoothing_omega, u);
            free(pu);
        }
        if (!st) memcpy(x, u, nL * sizeof(double));
        free(u);
    }
    for (int l = 0; l < L; ++l) sm_free(&sm[l]);
    free(sm);
out:
    for (int l = 1; l <= L; ++l) free(rhs[l]);
    free(rhs);
    return st;
}
