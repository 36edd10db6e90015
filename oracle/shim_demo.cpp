// TEST INFRASTRUCTURE: the integration story end to end. Links the UNMODIFIED
// reference library (built from /root/reference/proj/src) and libgmg_b200.so,
// and runs, on the same problem objects and inputs,
//     gmg::solve        (the reference, CPU)
//     gmg_b200::solve   (include/gmg_b200.hpp -> C ABI -> B200)
// comparing iteration counts, residual histories and solutions bit for bit.
// Built by oracle/Makefile into oracle/_ref/shim_demo; run by
// tests/test_integration.py on a GPU box. Exit status 0 = identical.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "gmg/cycle.hpp"
#include "gmg_b200.hpp"

namespace {

// bitwise equality; +0 and -0 count as equal (an exact zero's sign is unobservable downstream)
bool same(double a, double b) { return (a == 0.0 && b == 0.0) || std::memcmp(&a, &b, 8) == 0; }

int run(const char* name, int levels, int cnx, int cny, gmg::CoordinateSystem cs, double alpha, double beta,
        gmg::SmootherKind kind, double tol, int seed_x) {
    const gmg::GridHierarchy h = gmg::build_hierarchy(levels, cnx, cny, {}, cs);
    const gmg::MultilevelProblem prob(h, {alpha, beta});
    const gmg::LevelGrid& f = h.finest();
    gmg::GridFunction b = gmg::GridFunction::zeros(f);
    std::mt19937 rb(1);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    for (double& v : b.v) v = U(rb);
    gmg::GridFunction x0 = gmg::GridFunction::zeros(f);
    if (seed_x) {
        std::mt19937 rx(seed_x);
        for (double& v : x0.v) v = U(rx);
    }
    gmg::CycleSpec spec;
    spec.smoother = {kind, 1.0};
    spec.tolerance = tol;
    gmg::GridFunction xr = x0, xg = x0;
    const gmg::SolveReport rr = gmg::solve(prob, b, spec, xr);
    const gmg::SolveReport rg = gmg_b200::solve(prob, b, spec, xg);
    bool ok = rr.iterations == rg.iterations && rr.converged == rg.converged &&
              rr.residual_history.size() == rg.residual_history.size();
    for (std::size_t k = 0; ok && k < rr.residual_history.size(); ++k)
        ok = same(rr.residual_history[k], rg.residual_history[k]);
    for (std::size_t k = 0; ok && k < xr.v.size(); ++k) ok = same(xr.v[k], xg.v[k]);
    std::printf("{\"case\": \"%s\", \"identical\": %s, \"cycles\": %d, \"final\": \"%.17e\", "
                "\"cpu_s\": %.4f, \"gpu_s\": %.4f}\n",
                name, ok ? "true" : "false", rg.iterations,
                rg.residual_history.empty() ? 0.0 : rg.residual_history.back(), rr.wall_seconds, rg.wall_seconds);
    gmg_b200::release(prob);
    return ok ? 0 : 1;
}

}  // namespace

int main() {
    int bad = 0;
    bad += run("C1 jacobi adaptive", 7, 1, 1, gmg::CoordinateSystem::cartesian, 1.0, 1.0,
               gmg::SmootherKind::jacobi, 1e-8, 0);
    bad += run("C3' cylindrical jacobi", 9, 1, 1, gmg::CoordinateSystem::cylindrical, 1.0, 1.0,
               gmg::SmootherKind::jacobi, 1e-8, 0);
    bad += run("aniso gauss_seidel random start", 8, 1, 1, gmg::CoordinateSystem::cartesian, 0.1, 1.0,
               gmg::SmootherKind::gauss_seidel, 1e-8, 2);
    bad += run("spherical rect jacobi", 6, 2, 3, gmg::CoordinateSystem::spherical, 1.0, 0.5,
               gmg::SmootherKind::jacobi, 1e-9, 2);
    bad += run("aniso adi random start", 7, 1, 1, gmg::CoordinateSystem::cartesian, 0.01, 1.0,
               gmg::SmootherKind::adi, 1e-8, 2);
    bad += run("cylindrical ilu0", 7, 1, 1, gmg::CoordinateSystem::cylindrical, 1.0, 1.0,
               gmg::SmootherKind::ilu0, 1e-8, 0);
    // error mapping: an invalid smoother omega must surface as std::invalid_argument
    try {
        const gmg::GridHierarchy h = gmg::build_hierarchy(3, 1, 1, {}, gmg::CoordinateSystem::cartesian);
        const gmg::MultilevelProblem prob(h, {1.0, 1.0});
        gmg::GridFunction b = gmg::GridFunction::zeros(h.finest()), x = b;
        b.v[0] = 1.0;
        gmg::CycleSpec spec;
        spec.smoother = {gmg::SmootherKind::gauss_seidel, 3.0};
        gmg_b200::solve(prob, b, spec, x);
        std::printf("{\"case\": \"error mapping\", \"identical\": false}\n");
        ++bad;
    } catch (const std::invalid_argument& e) {
        std::printf("{\"case\": \"error mapping\", \"identical\": true, \"what\": \"%s\"}\n", e.what());
    }
    return bad;
}
