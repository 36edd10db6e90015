/*
 * gmg_b200.h — C ABI of the B200-native geometric-multigrid F-cycle
 * (libgmg_b200.so, sources in paper_0805_3041_b200/csrc/).
 *
 * This is the drop-in boundary for the reference gmg2d solver path
 * (/root/reference/proj). The reference has no FFI of its own; its boundary is
 * the free-function C++ API in namespace gmg, and each entry point below
 * replaces one of those functions behind plain pointers and sizes:
 *
 *   gmg_dev_problem_create  <- gmg::MultilevelProblem ctor   include/gmg/cycle.hpp:66 (src/cycle.cpp:25-30)
 *   gmg_dev_solve           <- gmg::solve                    include/gmg/cycle.hpp:105-106 (src/cycle.cpp:146-194)
 *   gmg_dev_mg_cycle        <- gmg::mg_cycle                 include/gmg/cycle.hpp:92-94 (src/cycle.cpp:69-100)
 *   gmg_dev_apply           <- gmg::apply                    include/gmg/stencil.hpp:44 (src/stencil.cpp:129-146)
 *   gmg_dev_residual        <- gmg::residual                 include/gmg/stencil.hpp:47 (src/stencil.cpp:148-153)
 *   gmg_dev_smooth_step     <- gmg::smooth_step (+ setup)    include/gmg/smoother.hpp:73,77-78 (src/smoother.cpp:231-276,389-399)
 *   gmg_dev_restriction     <- gmg::restriction              include/gmg/transfer.hpp:17 (src/transfer.cpp:72-101)
 *   gmg_dev_prolongation    <- gmg::prolongation             include/gmg/transfer.hpp:12 (src/transfer.cpp:32-70)
 *   gmg_dev_adaptive_omega  <- gmg::adaptive_omega           include/gmg/cycle.hpp:86-87 (src/cycle.cpp:40-51)
 *   gmg_dev_coarse_solve    <- gmg::BandedCholesky::solve    include/gmg/stencil.hpp:54 (src/stencil.cpp:190-210)
 *   gmg_dev_norm_l2/dot/axpy<- gmg::norm_l2 / dot / axpy     include/gmg/grid_function.hpp:29-34 (src/stencil.cpp:9-31)
 *   gmg_dev_make_start_vector <- gmg::make_start_vector      include/gmg/study.hpp:20-21 (src/study.cpp:40-79)
 *
 * Exceptions become status codes; the C++ shim
 * include/gmg_b200.hpp re-throws the reference's own exception types.
 *
 * Layout at the boundary: every grid function is the reference's
 * GridFunction::v — interior nodes only, row-major with x fastest,
 * k = j*nx + i (include/gmg/grid_function.hpp:10-26). Host pointers unless a
 * function name says _devptr. All arithmetic is IEEE fp64 in the reference's
 * operation order; results are bit-identical to the reference.
 */
#ifndef GMG_B200_H
#define GMG_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes -------------------------------------------------------- */
#define GMG_OK 0
#define GMG_ERR_LOGIC 1       /* std::logic_error: shape/level mismatch */
#define GMG_ERR_INVALID 2     /* std::invalid_argument: bad omega, steps, ... */
#define GMG_ERR_RUNTIME 3     /* std::runtime_error: nonpositive energy, not SPD */
#define GMG_DIVERGED 4        /* gmg::DivergenceError; report is filled */
#define GMG_ERR_CUDA 5        /* CUDA failure (no device, OOM, launch error) */
#define GMG_ERR_UNSUPPORTED 6 /* a spec this build does not implement */

/* ---- enums: same order as the reference enums ----------------------------- */
/* gmg::SmootherKind, include/gmg/smoother.hpp:13-25 */
enum gmg_smoother_kind {
    GMG_SMOOTHER_RICHARDSON = 0,
    GMG_SMOOTHER_JACOBI = 1,
    GMG_SMOOTHER_GAUSS_SEIDEL = 2,
    GMG_SMOOTHER_SOR = 3,
    GMG_SMOOTHER_ILU0 = 4,
    GMG_SMOOTHER_TRI_X = 5,
    GMG_SMOOTHER_TRI_Y = 6,
    GMG_SMOOTHER_ADI = 7,
    GMG_SMOOTHER_GSTRI_X = 8,
    GMG_SMOOTHER_GSTRI_Y = 9,
    GMG_SMOOTHER_GSADI = 10
};
/* gmg::CycleType, include/gmg/cycle.hpp:17 */
enum gmg_cycle_type { GMG_CYCLE_V = 0, GMG_CYCLE_W = 1, GMG_CYCLE_F = 2 };
/* gmg::CoordinateSystem, include/gmg/mesh.hpp:8; GMG_POLAR has no reference
 * counterpart (BASELINE config 3: r in [0.1, 1] Dirichlet, theta periodic;
 * host_setup.h documents the discretisation; only the jacobi and richardson
 * smoothers, parity against the oracle restatement, unpinned). */
enum gmg_coords { GMG_CARTESIAN = 0, GMG_CYLINDRICAL = 1, GMG_SPHERICAL = 2, GMG_POLAR = 3 };
/* how dot products / norms are summed on the device */
enum gmg_reduction {
    GMG_REDUCE_EXACT = 0, /* bit-identical to the reference's left-to-right sum */
    GMG_REDUCE_FAST = 1   /* tree reduction (not bit-identical; ~1e-13 relative) */
};

/* ---- problem description --------------------------------------------------- */
/* One level of a gmg::MultilevelProblem: LevelGrid (mesh.hpp:37-48) + StencilOperator
 * (stencil.hpp:20-34). All arrays are host memory, copied at create time. */
typedef struct gmg_level_desc {
    int level;       /* 1 = coarsest */
    int nx, ny;      /* interior points */
    const double* x; /* nx+2 node coordinates incl. boundary */
    const double* y; /* ny+2 */
    const double *c, *n, *s, *e, *w; /* nx*ny each */
} gmg_level_desc;

typedef struct gmg_problem_desc {
    int num_levels;
    const gmg_level_desc* levels; /* levels[0] = level 1 */
    int device;                   /* CUDA ordinal */
    int periodic_y;               /* 0: the reference's Dirichlet grids. 1: y periodic on every
                                     level (ny nodes, ny_l = 2 ny_(l-1); y has ny+2 entries whose
                                     first and last are the wrapped neighbours), the operator's
                                     s on row 0 and n on row ny-1 couple across the wrap */
    /* Optional: the physics the operators were assembled from (AnisotropySpec and
     * LevelGrid::coords, cycle.hpp:62-78). With alpha > 0, levels whose arrays are
     * not constant or x-only are rebuilt on the fly from 1-D tables (0 B/DOF of
     * coefficient traffic) when the tables reproduce every given coefficient bit
     * for bit; otherwise (alpha <= 0, or a mismatch) the five arrays are streamed. */
    double alpha, beta;
    int coords;                   /* gmg_coords */
} gmg_problem_desc;

/* gmg::CycleSpec, include/gmg/cycle.hpp:23-39 (+ SmootherSpec) */
typedef struct gmg_cycle_desc {
    int cycle;               /* gmg_cycle_type */
    int pre_steps;
    int post_steps;
    int adaptive_correction; /* 1: energy-norm minimiser (adaptive_omega) */
    double correction_omega;
    int smoother_kind;       /* gmg_smoother_kind */
    double smoother_omega;
    double smoothing_omega;  /* outer damping of each smooth_step */
    double tolerance;
    int max_cycles;
    unsigned long long coarse_direct_max_neq; /* ULLONG_MAX = unlimited */
    int reduction;           /* gmg_reduction */
} gmg_cycle_desc;

/* gmg::SolveReport, include/gmg/cycle.hpp:41-47. Buffers are caller-owned. */
typedef struct gmg_solve_report {
    int iterations;
    int converged;
    double wall_seconds;
    double* residual_history;    /* capacity >= max_cycles + 1 */
    double* convergence_factors; /* capacity >= max_cycles, may be NULL */
    int history_len;
    char message[256];
} gmg_solve_report;

typedef struct gmg_problem gmg_problem;

/* Row-slab distribution. Levels with at least
 * min_rows interior rows (and 4 rows per rank) are split into contiguous row
 * slabs, coarser levels are replicated. rank < 0: all `world` slabs live in
 * this process on one device (virtual ranks, exchanges are device copies);
 * rank >= 0: this process's slab of an NCCL group, nccl_id from
 * gmg_dist_unique_id on rank 0 (128 bytes). No reference counterpart: the
 * reference is single-threaded; results are bit-identical to gmg::solve. */
typedef struct gmg_slab_desc {
    int world;
    int rank;
    int min_rows;
    const unsigned char* nccl_id;
} gmg_slab_desc;

/* Thread-local text of the last failure (exception message in the reference). */
const char* gmg_last_error(void);
/* Library build string (arch, reduction engine version). */
const char* gmg_version(void);

/* ---- problem lifecycle ----------------------------------------------------- */
int gmg_dev_problem_create(const gmg_problem_desc* desc, gmg_problem** out);
int gmg_dev_problem_destroy(gmg_problem* p);
int gmg_dev_num_levels(const gmg_problem* p);
int gmg_dev_level_shape(const gmg_problem* p, int level, int* nx, int* ny);
/* operator storage chosen at create: 0 = constant 5-point, 1 = x-varying rows, 2 = full
 * field (five streamed arrays), 3 = computed on the fly from 1-D axis tables */
int gmg_dev_level_coef_kind(const gmg_problem* p, int level);
/* Row-slab problems (see gmg_slab_desc). Only gmg_dev_solve / _solve_devptr and
 * the queries below accept such a handle; the Jacobi smoother is sharded. */
int gmg_dev_problem_create_slabs(const gmg_problem_desc* desc, const gmg_slab_desc* slabs,
                                 gmg_problem** out);
int gmg_dist_unique_id(unsigned char* id128);
/* rank, world and the first sharded level (num_levels + 1: none) of a handle */
int gmg_dev_dist_info(const gmg_problem* p, int* rank, int* world, int* first_sharded_level);
/* rows [w0, w1) of `level` this slab owns ([0, ny) when the level is replicated) */
int gmg_dev_level_window(const gmg_problem* p, int level, int* w0, int* w1);

/* ---- the hot path ---------------------------------------------------------- */
/* gmg::solve: b read, x_inout carries the start vector in and the solution out.
 * Host pointers (nx*ny doubles, reference layout); pinned, registered or pageable
 * (large pageable vectors are staged through a pinned ring by a few host threads). */
int gmg_dev_solve(gmg_problem* p, const gmg_cycle_desc* spec, const double* b, double* x_inout,
                  gmg_solve_report* report);
/* Same, with b and x already resident on the device (reference layout, nx*ny
 * doubles each). Used by the benchmark's device-resident leg. */
int gmg_dev_solve_devptr(gmg_problem* p, const gmg_cycle_desc* spec, const double* b_dev,
                         double* x_dev, gmg_solve_report* report);
/* gmg::mg_cycle on level `level` (u0, g in, u out; host pointers). */
int gmg_dev_mg_cycle(gmg_problem* p, const gmg_cycle_desc* spec, int level, const double* u0,
                     const double* g, double* u);

/* gmg::make_start_vector (study.cpp:40-79) on the finest level: kind 0 zero,
 * 1 nested (restrict b to level 1, direct solve, then per level prolongation
 * and one smooth_step of spec's smoother). b, x: host arrays of the finest
 * level. Continuation (kind 2) is a host copy of another solution and has no
 * device counterpart: GMG_ERR_INVALID. */
int gmg_dev_make_start_vector(gmg_problem* p, const gmg_cycle_desc* spec, int kind, const double* b, double* x);

/* ---- per-operator entry points (host arrays; unit parity) ------------------- */
int gmg_dev_apply(gmg_problem* p, int level, const double* x, double* y);
int gmg_dev_residual(gmg_problem* p, int level, const double* x, const double* b, double* r);
int gmg_dev_smooth_step(gmg_problem* p, int level, int smoother_kind, double smoother_omega,
                        double omega_damp, const double* x, const double* b, double* out);
int gmg_dev_restriction(gmg_problem* p, int fine_level, const double* fine, double* coarse);
int gmg_dev_prolongation(gmg_problem* p, int coarse_level, const double* coarse, double* fine);
int gmg_dev_adaptive_omega(gmg_problem* p, int level, const double* defect,
                           const double* correction, double* omega);
int gmg_dev_coarse_solve(gmg_problem* p, const double* b, double* x);
int gmg_dev_norm_l2(gmg_problem* p, long long n, const double* v, int reduction, double* out);
int gmg_dev_dot(gmg_problem* p, long long n, const double* a, const double* b, int reduction,
                double* out);
int gmg_dev_axpy(gmg_problem* p, long long n, double alpha, const double* x, double* y);

/* ---- measurement hooks (bench.py) ------------------------------------------ */
/* Times `reps` back-to-back launches of the finest-level Jacobi smoother kernel
 * exactly as the F-cycle launches it, with CUDA events on the solver stream.
 * variant 0: pre-smoothing of the top visit (u0 = P e streamed from the coarse
 * level; 18 B/DOF algorithmic: g in, coarse e in, u out), 1: post-smoothing
 * (u + omega P uc; 26 B/DOF: u, g in, coarse uc in, u out), 2: plain smoother
 * from u (24 B/DOF). Writes the average ms per launch and the algorithmic
 * bytes per launch. */
int gmg_dev_time_smoother(gmg_problem* p, const gmg_cycle_desc* spec, int variant, int reps,
                          double* ms_per_launch, double* bytes_per_launch);
/* Exact-order summation engine counters accumulated since the last reset:
 * [0] sums, [1] records, [2] chain SM cycles, [3] of which re-walks,
 * [4] break adds, [5] re-walked ranges, [6] terms re-walked, [7] chunks,
 * [8..12] walk-kernel SM cycles per phase (load, prefix look-back, thread walk,
 * block merge, run/offset look-back), [13] walk CTAs, [14] literal (dense-break)
 * chunks among [5], [15] their cycles. out16 holds 16 values. */
int gmg_dev_seqsum_stats(gmg_problem* p, int reset, unsigned long long* out16);
/* Cycle skip+1 of a solve from b_dev, x_dev (device, reference layout) run
 * outside the CUDA graph with CUDA events around every launch (on the solver
 * stream): per launch the kernel family, the level it works on, its algorithmic
 * bytes (SURVEY.md §8d per-DOF bytes x the level's DOFs; 0 for the exact-sum
 * chains and the one-CTA coarse V-cycles) and its duration. The first `skip`
 * cycles replay the solve's graph unprofiled. count = launches (entries beyond
 * cap dropped). */
typedef struct gmg_prof_entry {
    char kernel[48];
    int level;
    double bytes;
    double ms;
} gmg_prof_entry;
int gmg_dev_profile_cycle(gmg_problem* p, const gmg_cycle_desc* spec, const double* b_dev, const double* x_dev,
                          int skip, int cap, gmg_prof_entry* out, int* count);
/* Number of kernels one solver cycle launches (from the captured graph). */
int gmg_dev_cycle_kernel_count(gmg_problem* p, const gmg_cycle_desc* spec, int* count);

/* ---- host-side setup helpers (no device work) ------------------------------ */
/* gmg::build_hierarchy + gmg::assemble (mesh.cpp:103-138, stencil.cpp:77-127)
 * followed by gmg_dev_problem_create. */
int gmg_host_problem_create(int num_levels, int coarse_nx, int coarse_ny, double grading_x,
                            double grading_y, int coords, double alpha, double beta, int device,
                            gmg_problem** out);
/* gmg_host_problem_create for row slabs. */
int gmg_host_problem_create_slabs(int num_levels, int coarse_nx, int coarse_ny, double grading_x,
                                  double grading_y, int coords, double alpha, double beta, int device,
                                  const gmg_slab_desc* slabs, gmg_problem** out);
/* The row-slab partition (no device work): first sharded level and, per level
 * and rank, the owned rows; w0/w1 are [num_levels][world], level-major. */
int gmg_host_slab_plan(int num_levels, const int* ny, int world, int min_rows, int halo, int* first_sharded,
                       int* w0, int* w1);
/* std::mt19937(seed) + uniform_real_distribution<double>(-1,1), the reference test
 * recipe (tests/oracles.hpp:252-258). */
void gmg_host_random_vector(long long n, unsigned seed, double* out);
/* Host emulation of the device exact-order summation engine (same chunking,
 * speculation and record chain), for CPU tests of its logic. */
int gmg_host_seqsum_emulate(long long n, const double* terms, int threads_per_chunk,
                            int elems_per_thread, double* out, long long* stats);

#ifdef __cplusplus
}
#endif
#endif
