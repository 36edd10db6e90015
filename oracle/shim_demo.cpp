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
#include "gmg/study.hpp"
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

bool same_vec(const std::vector<double>& a, const std::vector<double>& b) {
    if (a.size() != b.size()) return false;
    for (std::size_t k = 0; k < a.size(); ++k)
        if (!same(a[k], b[k])) return false;
    return true;
}

// The reference's callers build MultilevelProblem on the stack inside loops
// (study.cpp:162-166). Problems with different alpha and different level counts
// constructed in the same stack slot must each get their own device operators
// through the cached gmg_b200::solve(prob, ...) path (no release() between them).
int stack_slot_reuse() {
    int bad = 0;
    const void* prev = nullptr;
    int reused = 0;
    const struct { int levels; double alpha; } cases[] = {{6, 1.0}, {6, 0.1}, {6, 0.01}, {5, 0.01}, {6, 1.0}};
    for (const auto& c : cases) {
        const gmg::GridHierarchy h = gmg::build_hierarchy(c.levels, 1, 1, {}, gmg::CoordinateSystem::cartesian);
        const gmg::MultilevelProblem prob(h, {c.alpha, 1.0});
        if (&prob == prev) ++reused;
        prev = &prob;
        gmg::GridFunction b = gmg::GridFunction::zeros(h.finest());
        std::mt19937 rb(1);
        std::uniform_real_distribution<double> U(-1.0, 1.0);
        for (double& v : b.v) v = U(rb);
        gmg::CycleSpec spec;
        spec.smoother = {gmg::SmootherKind::jacobi, 1.0};
        spec.tolerance = 1e-8;
        gmg::GridFunction xr = gmg::GridFunction::zeros(h.finest()), xg = xr;
        const gmg::SolveReport rr = gmg::solve(prob, b, spec, xr);
        const gmg::SolveReport rg = gmg_b200::solve(prob, b, spec, xg);
        const bool ok = rr.iterations == rg.iterations && same_vec(rr.residual_history, rg.residual_history) &&
                        same_vec(xr.v, xg.v);
        bad += ok ? 0 : 1;
    }
    std::printf("{\"case\": \"stack-slot reuse (alpha and levels change at one address)\", \"identical\": %s, "
                "\"address_reused\": %d}\n",
                bad ? "false" : "true", reused);
    gmg_b200::release_all();
    return bad ? 1 : 0;
}

// gmg::make_start_vector (study.cpp:40-79) against gmg_b200::make_start_vector.
int start_vectors() {
    int bad = 0;
    const struct { gmg::SmootherKind kind; gmg::CoordinateSystem cs; int levels; } cases[] = {
        {gmg::SmootherKind::jacobi, gmg::CoordinateSystem::cartesian, 7},
        {gmg::SmootherKind::gauss_seidel, gmg::CoordinateSystem::cylindrical, 6},
        {gmg::SmootherKind::adi, gmg::CoordinateSystem::spherical, 5},
        {gmg::SmootherKind::ilu0, gmg::CoordinateSystem::cartesian, 1}};
    for (const auto& c : cases) {
        const gmg::GridHierarchy h = gmg::build_hierarchy(c.levels, c.levels == 1 ? 5 : 1, c.levels == 1 ? 4 : 1, {}, c.cs);
        const gmg::MultilevelProblem prob(h, {0.3, 1.0});
        gmg::GridFunction b = gmg::GridFunction::zeros(h.finest());
        std::mt19937 rb(3);
        std::uniform_real_distribution<double> U(-1.0, 1.0);
        for (double& v : b.v) v = U(rb);
        gmg::CycleSpec spec;
        spec.smoother = {c.kind, c.kind == gmg::SmootherKind::ilu0 ? 1.1 : 0.9};
        for (gmg::StartVectorKind k : {gmg::StartVectorKind::zero, gmg::StartVectorKind::nested}) {
            const gmg::GridFunction xr = gmg::make_start_vector({k, nullptr}, prob, spec, b);
            const gmg::GridFunction xg = gmg_b200::make_start_vector({k, nullptr}, prob, spec, b);
            bad += same_vec(xr.v, xg.v) ? 0 : 1;
        }
    }
    std::printf("{\"case\": \"make_start_vector zero/nested (4 smoothers, 3 coordinate systems)\", \"identical\": %s}\n",
                bad ? "false" : "true");
    gmg_b200::release_all();
    return bad ? 1 : 0;
}

// gmg::run_study (CPU) against gmg_b200::run_study (every solve, start vector and
// right-hand side on the GPU): rows and histories bit for bit.
int study(const char* name, gmg::SweepAxis axis, std::vector<std::string> values, gmg::SolverConfig base) {
    gmg::StudyConfig sc;
    sc.axis = axis;
    sc.values = std::move(values);
    sc.base = base;
    const gmg::StudyResult r = gmg::run_study(sc);
    const gmg::StudyResult g = gmg_b200::run_study(sc);
    bool ok = r.rows.size() == g.rows.size();
    for (std::size_t k = 0; ok && k < r.rows.size(); ++k) {
        const gmg::StudyRow &a = r.rows[k], &c = g.rows[k];
        ok = a.sweep_value == c.sweep_value && a.cycles == c.cycles && a.converged == c.converged &&
             same(a.final_rel_residual, c.final_rel_residual) && same(a.mean_rate, c.mean_rate) &&
             same_vec(a.history, c.history);
    }
    // the CSV a study writes, minus the wall-clock column
    auto strip = [](const std::string& csv) {
        std::string out, line;
        for (char ch : csv) {
            if (ch != '\n') {
                line += ch;
                continue;
            }
            out += line.substr(0, line.rfind(',')) + "\n";
            line.clear();
        }
        return out;
    };
    ok = ok && strip(gmg::study_csv(r)) == strip(gmg::study_csv(g));
    std::printf("{\"case\": \"study %s\", \"identical\": %s, \"rows\": %zu}\n", name, ok ? "true" : "false",
                g.rows.size());
    return ok ? 0 : 1;
}

int studies() {
    int bad = 0;
    gmg::SolverConfig base;
    base.levels = 6;
    base.tol = 1e-8;
    base.smoother = {gmg::SmootherKind::gauss_seidel, 1.0};
    bad += study("smoothing_steps", gmg::SweepAxis::smoothing_steps, {"1", "2", "3"}, base);
    bad += study("start_vector", gmg::SweepAxis::start_vector, {"zero", "nested", "continuation"}, base);
    bad += study("levels (coarse cap)", gmg::SweepAxis::levels, {"2", "4", "6"}, base);
    gmg::SolverConfig aniso = base;
    aniso.max_cycles = 12;
    bad += study("anisotropy", gmg::SweepAxis::anisotropy, {"1", "0.1", "0.001"}, aniso);
    gmg::SolverConfig sm = base;
    sm.levels = 5;
    sm.aniso.alpha = 0.01;
    bad += study("smoother", gmg::SweepAxis::smoother, {"jacobi", "sor", "ilu0", "tri_x", "gsadi", "richardson"}, sm);
    gmg::SolverConfig co = base;
    co.levels = 5;
    co.smoother = {gmg::SmootherKind::jacobi, 1.0};
    co.cycle = gmg::CycleType::W;
    bad += study("coordinates (W-cycle)", gmg::SweepAxis::coordinates, {"cartesian", "cylindrical", "spherical"}, co);
    return bad;
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
    bad += stack_slot_reuse();
    bad += start_vectors();
    bad += studies();
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
