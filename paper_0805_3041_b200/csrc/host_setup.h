// Host-side (CPU) setup for the device problem: hierarchy + assembly for the
// standalone API, the level-1 banded Cholesky factor, operator classification
// and transfer weight tables. Setup runs once per problem and stays on the host
// (SURVEY.md §3.2); only its products are uploaded.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

namespace gmg_host {

struct Level {
    int level = 1, nx = 0, ny = 0;
    bool periodic = false;                  // y periodic (polar theta): ny nodes, no y boundary
    std::vector<double> x, y;               // nx+2 / ny+2 node coordinates
    std::vector<double> c, n, s, e, w;      // nx*ny each, reference layout
};

// gmg::build_hierarchy + gmg::assemble (mesh.cpp:48-138, stencil.cpp:49-127).
// Throws std::invalid_argument with the reference's messages.
// coords 3 (polar, no reference counterpart, BASELINE
// config 3): x = r in [0.1, 1] (Dirichlet, graded like cylindrical), y = theta
// / (2 pi) in [0, 1) periodic with coarse_ny * 2^(l-1) nodes on level l at
// y_j = (j+1)/ny (node ny-1 sits at 1 == 0); the reference's flux form with
// x-flux face weight r, y-flux face weight 1/(2 pi)^2 and transverse measures
// dy and int dr/r = log(r_e / r_w): the polar Laplacian times r, i.e. the
// variable-coefficient 5-point stencil with coefficients r and 1/r.
std::vector<Level> build_problem(int num_levels, int coarse_nx, int coarse_ny, double grading_x,
                                 double grading_y, int coords, double alpha, double beta);

// BandedCholesky ctor (stencil.cpp:155-188): band[d*n + k] = L(k, k-d),
// half bandwidth nx. Throws std::runtime_error if not SPD.
std::vector<double> cholesky_band(const double* c, const double* w, const double* s, int nx, int ny);
// The same factorization for a y-periodic level: the dense lower triangle
// (half bandwidth n-1, the wrap couplings of rows 0 and ny-1 included).
std::vector<double> cholesky_periodic(const double* c, const double* w, const double* e, const double* s,
                                      const double* n, int nx, int ny);

// Operator classification (see common.cuh).
enum CoefKind { COEF_CONST = 0, COEF_ROWX = 1, COEF_FIELD = 2, COEF_AXES = 3 };

// 1-D tables of the on-the-fly operator (common.cuh CoefAxes): per column i
// ae = alpha fw(x_e), aw = alpha fw(x_w), he, hw, mx and 1/he, 1/hw; per row j
// bn, bs, hn, hs, my and 1/hn, 1/hs, with assemble's expressions
// (stencil.cpp:49-127).
struct AxisTables {
    std::vector<double> ae, aw, he, hw, mx, rhe, rhw;
    std::vector<double> bn, bs, hn, hs, my, rhn, rhs;
};
// Builds the tables of a level of coordinate system cs and checks that the
// coefficients computed from them reproduce c, n, s, e, w bit for bit (the
// reference's arrays); false if they do not (the level then streams FIELD).
bool axis_tables(const Level& L, int cs, double alpha, double beta, const double* c, const double* n,
                 const double* s, const double* e, const double* w, AxisTables& T);
struct CoefClass {
    CoefKind kind = COEF_FIELD;
    double c = 0, w = 0, e = 0, s = 0, n = 0;            // CONST
    std::vector<double> rc, rw, re, rs, rn;              // ROWX tables (length nx)
};
// periodic: y-periodic level (s on row 0 and n on the last row couple across the wrap).
CoefClass classify(int nx, int ny, const double* c, const double* n, const double* s,
                   const double* e, const double* w, bool periodic = false);

// odd_weight (transfer.cpp:26-28) tables.
// Prolongation (fine level f from coarse cx): tx[i] for fine column i (odd node i+1).
std::vector<double> prolong_weights(const std::vector<double>& xf, const std::vector<double>& xc, int nf);
// Restriction onto coarse: per coarse column P: wxw, wxe, sx (transfer.cpp:80-85).
void restrict_weights(const std::vector<double>& xf, const std::vector<double>& xc, int nc,
                      std::vector<double>& ww, std::vector<double>& we, std::vector<double>& sw);
// require_nested (transfer.cpp:10-22); returns an error message or "".
std::string check_nested(const Level& coarse, const Level& fine);

// Polar face weight of the theta flux, 1/(2 pi)^2 (coords 3).
double polar_theta_weight();

// factor_ilu0 (smoother.cpp:187-210) on the reference arrays: lw, ls, d
// (nx*ny each; ue/un are the operator's e/n). Throws std::runtime_error
// "ilu0 factorization: nonpositive pivot".
void factor_ilu0(int nx, int ny, const double* c, const double* w, const double* e, const double* s,
                 const double* n, double* lw, double* ls, double* d);

// Row-slab partition of a hierarchy over `world` ranks (DESIGN.md §7,
// SURVEY.md §8e). Levels l >= Ls (the first level with at least min_rows
// interior rows and at least `halo` rows per rank) are split into contiguous
// row windows; coarser levels are replicated on every rank. On Ls the rows are
// divided evenly; each finer level doubles the boundaries, so a coarse row's
// restriction stencil (fine rows 2Q..2Q+2) and a fine row's prolongation
// parents stay on the owning rank up to one halo row.
// w0/w1 are [level-1][rank]; replicated levels get [0, ny) for every rank.
struct SlabPlan {
    int Ls = 0;  // first sharded level (num_levels + 1 if none)
    std::vector<std::vector<int>> w0, w1;
};
SlabPlan slab_plan(const std::vector<int>& ny, int world, int min_rows, int halo);

// CPU emulation of the device exact-order summation engine.
double seqsum_emulate(const double* terms, long long n, int threads, int ept, long long* stats);

}  // namespace gmg_host
