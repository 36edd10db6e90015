// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A flat C API over the UNMODIFIED reference library (gmg2d, built from
// /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets the
// Python tests and bench.py's reference arm call the reference's own code
// paths (gmg::solve, apply, residual, smooth_step, restriction, prolongation,
// adaptive_omega, BandedCholesky::solve) on caller-owned arrays, so that
//   * golden fixtures under tests/golden/ are produced by the reference itself
//     (oracle/make_golden.py), and
//   * the C restatement (oracle/gmg_oracle.c) is pinned against the reference.
// Status codes mirror include/gmg_b200.h so both sides map exceptions alike.
#include <chrono>
#include <cstdio>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <vector>

#include "gmg/cycle.hpp"
#include "gmg/mesh.hpp"
#include "gmg/smoother.hpp"
#include "gmg/stencil.hpp"
#include "gmg/study.hpp"
#include "gmg/transfer.hpp"

namespace {

struct RefProblem {
    gmg::GridHierarchy h;
    std::unique_ptr<gmg::MultilevelProblem> prob;
};

struct Err {
    char* buf;
    int len;
    void set(const char* m) const {
        if (buf && len > 0) std::snprintf(buf, static_cast<std::size_t>(len), "%s", m);
    }
};

// 0 ok, 1 logic_error, 2 invalid_argument, 3 runtime_error, 4 DivergenceError
template <class F>
int guarded(const Err& err, F&& f) {
    try {
        f();
        return 0;
    } catch (const gmg::DivergenceError& e) {
        err.set(e.what());
        return 4;
    } catch (const std::invalid_argument& e) {
        err.set(e.what());
        return 2;
    } catch (const std::logic_error& e) {
        err.set(e.what());
        return 1;
    } catch (const std::runtime_error& e) {
        err.set(e.what());
        return 3;
    }
}

gmg::GridFunction wrap(const gmg::LevelGrid& g, const double* v) {
    gmg::GridFunction f = gmg::GridFunction::zeros(g);
    std::memcpy(f.v.data(), v, f.v.size() * sizeof(double));
    return f;
}

void out(const gmg::GridFunction& f, double* dst) {
    std::memcpy(dst, f.v.data(), f.v.size() * sizeof(double));
}

}  // namespace

extern "C" {

struct ref_cycle {
    int cycle;  // 0 V, 1 W, 2 F (gmg::CycleType order)
    int pre_steps;
    int post_steps;
    int adaptive_correction;
    double correction_omega;
    int smoother_kind;  // gmg::SmootherKind order
    double smoother_omega;
    double smoothing_omega;
    double tolerance;
    int max_cycles;
    unsigned long long coarse_direct_max_neq;
};

void* ref_problem_create(int levels, int cnx, int cny, double fx, double fy, int coords,
                         double alpha, double beta, char* errbuf, int errlen) {
    Err err{errbuf, errlen};
    RefProblem* p = nullptr;
    int st = guarded(err, [&] {
        auto rp = std::make_unique<RefProblem>();
        rp->h = gmg::build_hierarchy(levels, cnx, cny, gmg::GradingSpec{fx, fy},
                                     static_cast<gmg::CoordinateSystem>(coords));
        rp->prob = std::make_unique<gmg::MultilevelProblem>(rp->h, gmg::AnisotropySpec{alpha, beta});
        p = rp.release();
    });
    return st == 0 ? p : nullptr;
}

void ref_problem_destroy(void* h) { delete static_cast<RefProblem*>(h); }

int ref_level_shape(void* h, int level, int* nx, int* ny) {
    auto* p = static_cast<RefProblem*>(h);
    const auto& g = p->prob->grid(level);
    *nx = g.nx;
    *ny = g.ny;
    return 0;
}

int ref_level_coords(void* h, int level, double* x, double* y) {
    auto* p = static_cast<RefProblem*>(h);
    const auto& g = p->prob->grid(level);
    std::memcpy(x, g.x.data(), g.x.size() * sizeof(double));
    std::memcpy(y, g.y.data(), g.y.size() * sizeof(double));
    return 0;
}

int ref_operator(void* h, int level, double* c, double* n, double* s, double* e, double* w) {
    auto* p = static_cast<RefProblem*>(h);
    const auto& op = p->prob->op(level);
    const std::size_t nb = op.size() * sizeof(double);
    std::memcpy(c, op.c.data(), nb);
    std::memcpy(n, op.n.data(), nb);
    std::memcpy(s, op.s.data(), nb);
    std::memcpy(e, op.e.data(), nb);
    std::memcpy(w, op.w.data(), nb);
    return 0;
}

int ref_apply(void* h, int level, const double* x, double* y) {
    auto* p = static_cast<RefProblem*>(h);
    out(gmg::apply(p->prob->op(level), wrap(p->prob->grid(level), x)), y);
    return 0;
}

int ref_residual(void* h, int level, const double* x, const double* b, double* r) {
    auto* p = static_cast<RefProblem*>(h);
    const auto& g = p->prob->grid(level);
    out(gmg::residual(p->prob->op(level), wrap(g, x), wrap(g, b)), r);
    return 0;
}

int ref_smooth_step(void* h, int level, int kind, double smoother_omega, double omega_damp,
                    const double* x, const double* b, double* y, char* errbuf, int errlen) {
    auto* p = static_cast<RefProblem*>(h);
    Err err{errbuf, errlen};
    return guarded(err, [&] {
        const auto& g = p->prob->grid(level);
        const gmg::SmootherState st = gmg::setup(
            gmg::SmootherSpec{static_cast<gmg::SmootherKind>(kind), smoother_omega}, p->prob->op(level));
        out(gmg::smooth_step(st, wrap(g, x), wrap(g, b), omega_damp), y);
    });
}

int ref_restriction(void* h, int fine_level, const double* f, double* c) {
    auto* p = static_cast<RefProblem*>(h);
    out(gmg::restriction(wrap(p->prob->grid(fine_level), f), p->prob->grid(fine_level - 1)), c);
    return 0;
}

int ref_prolongation(void* h, int coarse_level, const double* c, double* f) {
    auto* p = static_cast<RefProblem*>(h);
    out(gmg::prolongation(wrap(p->prob->grid(coarse_level), c), p->prob->grid(coarse_level + 1)), f);
    return 0;
}

int ref_adaptive_omega(void* h, int level, const double* d, const double* corr, double* omega,
                       char* errbuf, int errlen) {
    auto* p = static_cast<RefProblem*>(h);
    Err err{errbuf, errlen};
    return guarded(err, [&] {
        const auto& g = p->prob->grid(level);
        *omega = gmg::adaptive_omega(wrap(g, d), wrap(g, corr), p->prob->op(level));
    });
}

int ref_coarse_solve(void* h, const double* b, double* x) {
    auto* p = static_cast<RefProblem*>(h);
    out(p->prob->coarse_solver().solve(wrap(p->prob->grid(1), b)), x);
    return 0;
}

double ref_norm_l2(void* h, int level, const double* v) {
    auto* p = static_cast<RefProblem*>(h);
    return gmg::norm_l2(wrap(p->prob->grid(level), v));
}

double ref_dot(void* h, int level, const double* a, const double* b) {
    auto* p = static_cast<RefProblem*>(h);
    const auto& g = p->prob->grid(level);
    return gmg::dot(wrap(g, a), wrap(g, b));
}

static gmg::CycleSpec to_spec(const ref_cycle* c) {
    gmg::CycleSpec s;
    s.cycle = static_cast<gmg::CycleType>(c->cycle);
    s.pre_steps = c->pre_steps;
    s.post_steps = c->post_steps;
    s.adaptive_correction = c->adaptive_correction != 0;
    s.correction_omega = c->correction_omega;
    s.smoother = gmg::SmootherSpec{static_cast<gmg::SmootherKind>(c->smoother_kind), c->smoother_omega};
    s.smoothing_omega = c->smoothing_omega;
    s.tolerance = c->tolerance;
    s.max_cycles = c->max_cycles;
    s.coarse_direct_max_neq = static_cast<std::size_t>(c->coarse_direct_max_neq);
    return s;
}

int ref_mg_cycle(void* h, const ref_cycle* spec, int level, const double* u0, const double* g,
                 double* u, char* errbuf, int errlen) {
    auto* p = static_cast<RefProblem*>(h);
    Err err{errbuf, errlen};
    return guarded(err, [&] {
        const gmg::CycleSpec s = to_spec(spec);
        const auto sm = gmg::setup_smoothers(*p->prob, s.smoother);
        const auto& gr = p->prob->grid(level);
        out(gmg::mg_cycle(level, wrap(gr, u0), wrap(gr, g), s, *p->prob, sm), u);
    });
}

// gmg::solve. hist must hold max_cycles+1 doubles.
int ref_solve(void* h, const ref_cycle* spec, const double* b, double* x, double* hist,
              int* hist_len, int* iterations, int* converged, double* wall_seconds, char* errbuf,
              int errlen) {
    auto* p = static_cast<RefProblem*>(h);
    Err err{errbuf, errlen};
    const auto& g = p->prob->grid(p->prob->num_levels());
    gmg::GridFunction bx = wrap(g, b);
    gmg::GridFunction xx = wrap(g, x);
    gmg::SolveReport rep;
    int st = guarded(err, [&] {
        try {
            rep = gmg::solve(*p->prob, bx, to_spec(spec), xx);
        } catch (const gmg::DivergenceError& e) {
            rep = e.report();
            throw;
        }
    });
    for (std::size_t k = 0; k < rep.residual_history.size(); ++k) hist[k] = rep.residual_history[k];
    *hist_len = static_cast<int>(rep.residual_history.size());
    *iterations = rep.iterations;
    *converged = rep.converged ? 1 : 0;
    *wall_seconds = rep.wall_seconds;
    out(xx, x);
    return st;
}

// Start vector per gmg::make_start_vector (kind 0 zero, 1 nested), study.cpp:40-79.
int ref_start_vector(void* h, const ref_cycle* spec, int kind, const double* b, double* x, char* err, int len) {
    return guarded(Err{err, len}, [&] {
        auto* p = static_cast<RefProblem*>(h);
        const auto& g = p->prob->grid(p->prob->num_levels());
        gmg::StartVectorStrategy strat;
        strat.kind = static_cast<gmg::StartVectorKind>(kind);
        out(gmg::make_start_vector(strat, *p->prob, to_spec(spec), wrap(g, b)), x);
    });
}

// std::mt19937(seed) + uniform_real_distribution<double>(-1, 1), the recipe of
// tests/oracles.hpp:252-258 (random_vector).
void ref_random_vector(long long n, unsigned seed, double* v) {
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> dist(-1.0, 1.0);
    for (long long k = 0; k < n; ++k) v[k] = dist(rng);
}

}  // extern "C"
