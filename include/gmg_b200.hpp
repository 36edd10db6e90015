// gmg_b200.hpp — drop-in C++ shim for the reference gmg2d library.
//
// A maintainer of the reference adds this header (and links libgmg_b200.so)
// to run gmg::solve on a B200 with the reference's own types and exception
// behaviour:
//
//     #include "gmg/cycle.hpp"
//     #include "gmg_b200.hpp"
//     gmg::SolveReport rep = gmg_b200::solve(prob, b, spec, x);   // was gmg::solve(prob, b, spec, x)
//
// Replaces gmg::solve (include/gmg/cycle.hpp:101-106, src/cycle.cpp:146-194):
// same arguments (b read, x = start vector in / solution out), same
// SolveReport, bit-identical residual history and solution. Errors map back to
// the reference's exception types: GMG_ERR_LOGIC ->
// std::logic_error, GMG_ERR_INVALID -> std::invalid_argument, GMG_ERR_RUNTIME ->
// std::runtime_error, GMG_DIVERGED -> gmg::DivergenceError carrying the partial
// report; CUDA failures and unimplemented smoother kinds raise
// std::runtime_error.
//
// Device problem lifetime: MultilevelProblem is immutable after construction
// (cycle.hpp:59-61), so the device copy (operators of every level, transfer
// weights, level-1 factor) is built on first use and cached per
// MultilevelProblem address; gmg_b200::release(prob) frees it.
#pragma once

#include <climits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "gmg/cycle.hpp"
#include "gmg_b200.h"

namespace gmg_b200 {

namespace detail {

inline std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
inline std::map<const gmg::MultilevelProblem*, gmg_problem*>& cache() {
    static std::map<const gmg::MultilevelProblem*, gmg_problem*> c;
    return c;
}

[[noreturn]] inline void rethrow(int code, const char* what, const gmg::SolveReport* partial = nullptr) {
    const std::string msg = what ? what : "";
    switch (code) {
        case GMG_ERR_LOGIC: throw std::logic_error(msg);
        case GMG_ERR_INVALID: throw std::invalid_argument(msg);
        case GMG_DIVERGED: throw gmg::DivergenceError(msg, partial ? *partial : gmg::SolveReport{});
        default: throw std::runtime_error(msg);
    }
}

inline gmg_problem* device_problem(const gmg::MultilevelProblem& prob, int device) {
    std::lock_guard<std::mutex> lk(cache_mutex());
    auto it = cache().find(&prob);
    if (it != cache().end()) return it->second;
    std::vector<gmg_level_desc> lv(static_cast<std::size_t>(prob.num_levels()));
    for (int l = 1; l <= prob.num_levels(); ++l) {
        const gmg::LevelGrid& g = prob.grid(l);
        const gmg::StencilOperator& A = prob.op(l);
        lv[l - 1] = gmg_level_desc{l,          g.nx,       g.ny,       g.x.data(), g.y.data(),
                                   A.c.data(), A.n.data(), A.s.data(), A.e.data(), A.w.data()};
    }
    const gmg_problem_desc desc{prob.num_levels(), lv.data(), device};
    gmg_problem* p = nullptr;
    const int st = gmg_dev_problem_create(&desc, &p);
    if (st != GMG_OK) rethrow(st, gmg_last_error());
    cache().emplace(&prob, p);
    return p;
}

inline gmg_cycle_desc to_desc(const gmg::CycleSpec& s, int reduction) {
    gmg_cycle_desc d{};
    d.cycle = static_cast<int>(s.cycle);
    d.pre_steps = s.pre_steps;
    d.post_steps = s.post_steps;
    d.adaptive_correction = s.adaptive_correction ? 1 : 0;
    d.correction_omega = s.correction_omega;
    d.smoother_kind = static_cast<int>(s.smoother.kind);
    d.smoother_omega = s.smoother.omega;
    d.smoothing_omega = s.smoothing_omega;
    d.tolerance = s.tolerance;
    d.max_cycles = s.max_cycles;
    d.coarse_direct_max_neq = s.coarse_direct_max_neq > static_cast<std::size_t>(ULLONG_MAX)
                                  ? ULLONG_MAX
                                  : static_cast<unsigned long long>(s.coarse_direct_max_neq);
    d.reduction = reduction;
    return d;
}

}  // namespace detail

// gmg::solve on the GPU (device 0 unless given). reduction: GMG_REDUCE_EXACT
// (bit-identical to the reference, default) or GMG_REDUCE_FAST.
inline gmg::SolveReport solve(const gmg::MultilevelProblem& prob, const gmg::GridFunction& b,
                              const gmg::CycleSpec& spec, gmg::GridFunction& x, int device = 0,
                              int reduction = GMG_REDUCE_EXACT) {
    const gmg::LevelGrid& fine = prob.grid(prob.num_levels());
    if (b.grid == nullptr || x.grid == nullptr || b.nx() != fine.nx || b.ny() != fine.ny ||
        x.nx() != fine.nx || x.ny() != fine.ny)
        throw std::logic_error("residual: grid functions live on different levels");
    gmg_problem* p = detail::device_problem(prob, device);
    const gmg_cycle_desc d = detail::to_desc(spec, reduction);
    std::vector<double> hist(static_cast<std::size_t>(spec.max_cycles > 0 ? spec.max_cycles : 0) + 1);
    std::vector<double> fac(hist.size());
    gmg_solve_report rep{};
    rep.residual_history = hist.data();
    rep.convergence_factors = fac.data();
    const int st = gmg_dev_solve(p, &d, b.v.data(), x.v.data(), &rep);
    gmg::SolveReport out;
    out.iterations = rep.iterations;
    out.converged = rep.converged != 0;
    out.wall_seconds = rep.wall_seconds;
    out.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
    out.convergence_factors.assign(fac.begin(), fac.begin() + (rep.history_len > 0 ? rep.history_len - 1 : 0));
    if (st != GMG_OK) detail::rethrow(st, gmg_last_error(), &out);
    return out;
}

// Frees the cached device copy of prob.
inline void release(const gmg::MultilevelProblem& prob) {
    std::lock_guard<std::mutex> lk(detail::cache_mutex());
    auto it = detail::cache().find(&prob);
    if (it == detail::cache().end()) return;
    gmg_dev_problem_destroy(it->second);
    detail::cache().erase(it);
}

}  // namespace gmg_b200
