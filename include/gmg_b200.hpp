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
// The study layer (include/gmg/study.hpp) runs on the same device path:
// gmg_b200::make_start_vector, resolve_start_vector and run_study replace
// study.cpp:40-79, :139-160 and :162-217 (every solve, start vector and
// right-hand side of a sweep is computed on the GPU).
//
// Device problem lifetime. Two ways:
//   * explicit: gmg_b200::DeviceProblem dev(prob, device); solve(dev, b, spec, x);
//     owns the device copy (operators of every level, transfer weights,
//     level-1 factor) and frees it when it goes out of scope;
//   * implicit: solve(prob, ...) keeps one device copy per (MultilevelProblem
//     address, device). Every hit re-checks a content fingerprint of prob
//     (level shapes, coordinate system and node coordinates of every level, the
//     anisotropy, and sampled operator coefficients), so a new problem built at a
//     reused address (the reference's callers construct problems on the stack in
//     loops, study.cpp:162-166) never reuses a stale copy: a mismatch rebuilds it.
//     gmg_b200::release(prob) / release_all() free cached copies.
#pragma once

#include <climits>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "gmg/config.hpp"
#include "gmg/cycle.hpp"
#include "gmg/study.hpp"
#include "gmg_b200.h"

namespace gmg_b200 {

namespace detail {

[[noreturn]] inline void rethrow(int code, const char* what, const gmg::SolveReport* partial = nullptr) {
    const std::string msg = what ? what : "";
    switch (code) {
        case GMG_ERR_LOGIC: throw std::logic_error(msg);
        case GMG_ERR_INVALID: throw std::invalid_argument(msg);
        case GMG_DIVERGED: throw gmg::DivergenceError(msg, partial ? *partial : gmg::SolveReport{});
        default: throw std::runtime_error(msg);
    }
}

inline void check(int st) {
    if (st != GMG_OK) rethrow(st, gmg_last_error());
}

// Content fingerprint of a MultilevelProblem. The operators are a pure function of
// the hierarchy's node coordinates, its coordinate system and the anisotropy
// (assemble, stencil.cpp:77-127), all of which are compared in full; strided
// samples of the five coefficient arrays of every level are compared as well.
struct Fingerprint {
    std::vector<long long> ints;
    std::vector<double> vals;
    bool operator==(const Fingerprint& o) const {
        return ints == o.ints && vals.size() == o.vals.size() &&
               (vals.empty() || std::memcmp(vals.data(), o.vals.data(), vals.size() * sizeof(double)) == 0);
    }
};

inline Fingerprint fingerprint(const gmg::MultilevelProblem& prob, int device) {
    Fingerprint f;
    f.ints = {device, prob.num_levels()};
    f.vals = {prob.anisotropy().alpha, prob.anisotropy().beta};
    for (int l = 1; l <= prob.num_levels(); ++l) {
        const gmg::LevelGrid& g = prob.grid(l);
        f.ints.insert(f.ints.end(), {g.nx, g.ny, static_cast<long long>(g.coords)});
        f.vals.insert(f.vals.end(), g.x.begin(), g.x.end());
        f.vals.insert(f.vals.end(), g.y.begin(), g.y.end());
        const gmg::StencilOperator& A = prob.op(l);
        for (const std::vector<double>* a : {&A.c, &A.n, &A.s, &A.e, &A.w}) {
            f.ints.push_back(static_cast<long long>(a->size()));
            if (a->empty()) continue;
            const std::size_t stride = a->size() > 64 ? a->size() / 64 : 1;
            for (std::size_t k = 0; k < a->size(); k += stride) f.vals.push_back((*a)[k]);
            f.vals.push_back(a->back());
        }
    }
    return f;
}

inline gmg_problem* create(const gmg::MultilevelProblem& prob, int device) {
    std::vector<gmg_level_desc> lv(static_cast<std::size_t>(prob.num_levels()));
    for (int l = 1; l <= prob.num_levels(); ++l) {
        const gmg::LevelGrid& g = prob.grid(l);
        const gmg::StencilOperator& A = prob.op(l);
        lv[l - 1] = gmg_level_desc{l,          g.nx,       g.ny,       g.x.data(), g.y.data(),
                                   A.c.data(), A.n.data(), A.s.data(), A.e.data(), A.w.data()};
    }
    // the physics lets the library rebuild graded / spherical operators on the fly (checked bit for bit)
    const gmg_problem_desc desc{prob.num_levels(), lv.data(), device, 0, prob.anisotropy().alpha,
                                prob.anisotropy().beta, static_cast<int>(prob.grid(1).coords)};
    gmg_problem* p = nullptr;
    check(gmg_dev_problem_create(&desc, &p));
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

// An owned device copy of one MultilevelProblem (gmg_dev_problem_create ...
// gmg_dev_problem_destroy). The problem is immutable after construction
// (cycle.hpp:59-61), so the copy stays valid as long as the caller keeps it.
class DeviceProblem {
  public:
    explicit DeviceProblem(const gmg::MultilevelProblem& prob, int device = 0)
        : h_(detail::create(prob, device)), device_(device), num_levels_(prob.num_levels()) {}
    DeviceProblem(const DeviceProblem&) = delete;
    DeviceProblem& operator=(const DeviceProblem&) = delete;
    DeviceProblem(DeviceProblem&& o) noexcept : h_(o.h_), device_(o.device_), num_levels_(o.num_levels_) {
        o.h_ = nullptr;
    }
    ~DeviceProblem() {
        if (h_) gmg_dev_problem_destroy(h_);
    }
    gmg_problem* handle() const { return h_; }
    int device() const { return device_; }
    int num_levels() const { return num_levels_; }

  private:
    gmg_problem* h_ = nullptr;
    int device_ = 0;
    int num_levels_ = 0;
};

namespace detail {

struct CacheEntry {
    Fingerprint fp;
    std::unique_ptr<DeviceProblem> dev;
};
inline std::mutex& cache_mutex() {
    static std::mutex m;
    return m;
}
inline std::map<std::pair<const gmg::MultilevelProblem*, int>, CacheEntry>& cache() {
    static std::map<std::pair<const gmg::MultilevelProblem*, int>, CacheEntry> c;
    return c;
}

// The cached device copy of prob on `device`, rebuilt when prob's content
// fingerprint differs from the one it was built from.
inline const DeviceProblem& cached(const gmg::MultilevelProblem& prob, int device) {
    Fingerprint fp = fingerprint(prob, device);
    std::lock_guard<std::mutex> lk(cache_mutex());
    CacheEntry& e = cache()[{&prob, device}];
    if (!e.dev || !(e.fp == fp)) {
        e.dev.reset();  // free the stale copy before building the new one
        e.dev = std::make_unique<DeviceProblem>(prob, device);
        e.fp = std::move(fp);
    }
    return *e.dev;
}

inline void check_finest(const DeviceProblem& dev, const gmg::MultilevelProblem* prob, const gmg::GridFunction& v) {
    int nx = 0, ny = 0;
    check(gmg_dev_level_shape(dev.handle(), dev.num_levels(), &nx, &ny));
    if (v.grid == nullptr || v.nx() != nx || v.ny() != ny ||
        v.v.size() != static_cast<std::size_t>(nx) * static_cast<std::size_t>(ny))
        throw std::logic_error("residual: grid functions live on different levels");
    (void)prob;
}

}  // namespace detail

// gmg::solve on the GPU. reduction: GMG_REDUCE_EXACT (bit-identical to the
// reference, default) or GMG_REDUCE_FAST.
inline gmg::SolveReport solve(const DeviceProblem& dev, const gmg::GridFunction& b, const gmg::CycleSpec& spec,
                              gmg::GridFunction& x, int reduction = GMG_REDUCE_EXACT) {
    detail::check_finest(dev, nullptr, b);
    detail::check_finest(dev, nullptr, x);
    const gmg_cycle_desc d = detail::to_desc(spec, reduction);
    std::vector<double> hist(static_cast<std::size_t>(spec.max_cycles > 0 ? spec.max_cycles : 0) + 1);
    std::vector<double> fac(hist.size());
    gmg_solve_report rep{};
    rep.residual_history = hist.data();
    rep.convergence_factors = fac.data();
    const int st = gmg_dev_solve(dev.handle(), &d, b.v.data(), x.v.data(), &rep);
    gmg::SolveReport out;
    out.iterations = rep.iterations;
    out.converged = rep.converged != 0;
    out.wall_seconds = rep.wall_seconds;
    out.residual_history.assign(hist.begin(), hist.begin() + rep.history_len);
    out.convergence_factors.assign(fac.begin(), fac.begin() + (rep.history_len > 0 ? rep.history_len - 1 : 0));
    if (st != GMG_OK) detail::rethrow(st, gmg_last_error(), &out);
    return out;
}

// Drop-in: gmg::solve(prob, b, spec, x) on GPU `device` (0 unless given), with the
// fingerprint-checked cached device copy of prob.
inline gmg::SolveReport solve(const gmg::MultilevelProblem& prob, const gmg::GridFunction& b,
                              const gmg::CycleSpec& spec, gmg::GridFunction& x, int device = 0,
                              int reduction = GMG_REDUCE_EXACT) {
    const gmg::LevelGrid& fine = prob.grid(prob.num_levels());
    if (b.grid == nullptr || x.grid == nullptr || b.nx() != fine.nx || b.ny() != fine.ny ||
        x.nx() != fine.nx || x.ny() != fine.ny)
        throw std::logic_error("residual: grid functions live on different levels");
    return solve(detail::cached(prob, device), b, spec, x, reduction);
}

// Frees the cached device copies of prob (every device).
inline void release(const gmg::MultilevelProblem& prob) {
    std::lock_guard<std::mutex> lk(detail::cache_mutex());
    auto& c = detail::cache();
    for (auto it = c.begin(); it != c.end();) {
        if (it->first.first == &prob) it = c.erase(it);
        else ++it;
    }
}
inline void release_all() {
    std::lock_guard<std::mutex> lk(detail::cache_mutex());
    detail::cache().clear();
}

// gmg::apply on the finest level (stencil.cpp:129-146), on the device.
inline gmg::GridFunction apply_finest(const DeviceProblem& dev, const gmg::LevelGrid& fine, const gmg::GridFunction& v) {
    gmg::GridFunction y = gmg::GridFunction::zeros(fine);
    detail::check(gmg_dev_apply(dev.handle(), dev.num_levels(), v.v.data(), y.v.data()));
    return y;
}

// gmg::make_start_vector (study.hpp:20-21, study.cpp:40-79): zero and nested on the
// device (restriction cascade, level-1 direct solve, prolongation + one smooth_step
// per level); continuation copies the source solution as the reference does.
inline gmg::GridFunction make_start_vector(const gmg::StartVectorStrategy& strategy, const DeviceProblem& dev,
                                           const gmg::MultilevelProblem& prob, const gmg::CycleSpec& spec,
                                           const gmg::GridFunction& b) {
    const gmg::LevelGrid& finest = prob.grid(prob.num_levels());
    if (strategy.kind == gmg::StartVectorKind::continuation) {
        const gmg::GridFunction* src = strategy.continuation_source;
        if (src == nullptr) throw std::invalid_argument("start: continuation requires a source solution");
        if (src->nx() != finest.nx || src->ny() != finest.ny)
            throw std::invalid_argument("start: continuation source shape does not match");
        gmg::GridFunction u = gmg::GridFunction::zeros(finest);
        u.v = src->v;
        return u;
    }
    gmg::GridFunction u = gmg::GridFunction::zeros(finest);
    const gmg_cycle_desc d = detail::to_desc(spec, GMG_REDUCE_EXACT);
    detail::check(gmg_dev_make_start_vector(dev.handle(), &d, strategy.kind == gmg::StartVectorKind::nested ? 1 : 0,
                                            b.v.data(), u.v.data()));
    return u;
}
inline gmg::GridFunction make_start_vector(const gmg::StartVectorStrategy& strategy, const gmg::MultilevelProblem& prob,
                                           const gmg::CycleSpec& spec, const gmg::GridFunction& b, int device = 0) {
    return make_start_vector(strategy, detail::cached(prob, device), prob, spec, b);
}

// gmg::resolve_start_vector (study.cpp:139-160): continuation solves the related
// problem (alpha / 10, zero start) on the device first.
inline gmg::GridFunction resolve_start_vector(const gmg::SolverConfig& cfg, const DeviceProblem& dev,
                                              const gmg::MultilevelProblem& prob, const gmg::CycleSpec& spec,
                                              const gmg::GridFunction& b) {
    if (cfg.start != gmg::StartVectorKind::continuation)
        return make_start_vector({cfg.start, nullptr}, dev, prob, spec, b);
    gmg::SolverConfig scfg = cfg;
    scfg.aniso.alpha = cfg.aniso.alpha / 10.0;
    scfg.start = gmg::StartVectorKind::zero;
    const gmg::GridHierarchy sh = scfg.build_hierarchy();
    const gmg::MultilevelProblem sprob(sh, scfg.aniso);
    const DeviceProblem sdev(sprob, dev.device());
    const int levels = sprob.num_levels();
    const gmg::GridFunction sb = apply_finest(sdev, sprob.grid(levels), gmg::manufactured_solution(sprob.grid(levels)));
    gmg::GridFunction sx = gmg::GridFunction::zeros(sprob.grid(levels));
    try {
        solve(sdev, sb, scfg.cycle_spec(), sx);
    } catch (const gmg::DivergenceError&) {
        // keep whatever iterate the source solve reached (study.cpp:155-157)
    }
    return make_start_vector({gmg::StartVectorKind::continuation, &sx}, dev, prob, spec, b);
}

namespace detail {

// study.cpp:75 (kLevelsStudyCoarseCap)
constexpr std::size_t kLevelsStudyCoarseCap = 100;

// config_for_value, study.cpp:77-121 (the reference keeps it file-local).
inline gmg::SolverConfig config_for_value(const gmg::StudyConfig& study, const std::string& value) {
    gmg::SolverConfig cfg = study.base;
    switch (study.axis) {
        case gmg::SweepAxis::anisotropy:
            cfg.aniso.alpha = std::stod(value);
            break;
        case gmg::SweepAxis::levels: {
            const int L = std::stoi(value);
            if (L < 1) throw std::invalid_argument("values: levels must be >= 1");
            const int cells_x = (study.base.coarse_nx + 1) << (study.base.levels - 1);
            const int cells_y = (study.base.coarse_ny + 1) << (study.base.levels - 1);
            const int shift = L - 1;
            if (L > study.base.levels || (cells_x >> shift) << shift != cells_x || (cells_x >> shift) < 2 ||
                (cells_y >> shift) < 2)
                throw std::invalid_argument("values: level count incompatible with the base finest grid");
            cfg.levels = L;
            cfg.coarse_nx = (cells_x >> shift) - 1;
            cfg.coarse_ny = (cells_y >> shift) - 1;
            break;
        }
        case gmg::SweepAxis::smoothing_steps: {
            const int steps = std::stoi(value);
            if (steps < 1) throw std::invalid_argument("values: smoothing steps must be >= 1");
            cfg.pre_steps = steps;
            cfg.post_steps = steps;
            break;
        }
        case gmg::SweepAxis::coordinates:
            cfg.coords = gmg::parse_coordinate_system(value);
            break;
        case gmg::SweepAxis::smoother:
            cfg.smoother.kind = gmg::parse_smoother_kind(value);
            break;
        case gmg::SweepAxis::start_vector:
            cfg.start = gmg::parse_start_vector(value);
            break;
    }
    cfg.validate();
    return cfg;
}

inline std::string sanitize(const std::string& s) {
    std::string out = s;
    for (char& c : out)
        if (c == '/' || c == '\\' || c == ' ') c = '_';
    return out;
}

// run_one, study.cpp:162-192: right-hand side, start vector and solve on the device.
inline gmg::StudyRow run_one(const gmg::SolverConfig& cfg, const std::string& value, bool cap_coarse, int device) {
    const gmg::GridHierarchy hierarchy = cfg.build_hierarchy();
    const gmg::MultilevelProblem prob(hierarchy, cfg.aniso);
    const DeviceProblem dev(prob, device);
    gmg::CycleSpec spec = cfg.cycle_spec();
    if (cap_coarse) spec.coarse_direct_max_neq = kLevelsStudyCoarseCap;
    const int levels = prob.num_levels();
    const gmg::GridFunction b = apply_finest(dev, prob.grid(levels), gmg::manufactured_solution(prob.grid(levels)));
    gmg::GridFunction x = resolve_start_vector(cfg, dev, prob, spec, b);

    gmg::StudyRow row;
    row.sweep_value = value;
    gmg::SolveReport report;
    try {
        report = solve(dev, b, spec, x);
        row.cycles = report.converged ? report.iterations : cfg.max_cycles;
        row.converged = report.converged;
    } catch (const gmg::DivergenceError& e) {
        report = e.report();
        row.cycles = cfg.max_cycles;
        row.converged = false;
    }
    row.history = report.residual_history;
    const double r0 = report.residual_history.front();
    row.final_rel_residual = r0 == 0.0 ? 0.0 : report.residual_history.back() / r0;
    row.mean_rate = report.residual_history.size() < 2 ? 1.0 : gmg::convergence_rate(report.residual_history);
    row.wall_ms = report.wall_seconds * 1000.0;
    return row;
}

}  // namespace detail

// gmg::run_study (study.hpp:66, study.cpp:194-217) with every solve on GPU `device`:
// same rows (cycles, convergence, bit-identical histories), same CSV files.
inline gmg::StudyResult run_study(const gmg::StudyConfig& config, int device = 0) {
    if (config.values.empty()) throw std::invalid_argument("values: sweep values must be nonempty");
    config.base.validate();
    gmg::StudyResult result;
    for (const std::string& value : config.values) {
        const gmg::SolverConfig cfg = detail::config_for_value(config, value);
        result.rows.push_back(detail::run_one(cfg, value, config.axis == gmg::SweepAxis::levels, device));
    }
    if (!config.output_csv.empty()) {
        std::ofstream out(config.output_csv, std::ios::binary);
        if (!out) throw std::runtime_error("out: cannot write " + config.output_csv.string());
        out << gmg::study_csv(result);
        const auto dir = config.output_csv.parent_path();
        for (const gmg::StudyRow& row : result.rows) {
            const auto path = dir / ("history_" + detail::sanitize(row.sweep_value) + ".csv");
            std::ofstream hist(path, std::ios::binary);
            if (!hist) throw std::runtime_error("out: cannot write " + path.string());
            hist << gmg::history_csv(row);
        }
    }
    return result;
}

}  // namespace gmg_b200
