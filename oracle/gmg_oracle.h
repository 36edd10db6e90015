/* TEST INFRASTRUCTURE ONLY — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline/reference legs may load it, and only as the checker.
 *
 * Plain-C restatement of the reference gmg2d F-cycle path (/root/reference/proj):
 * hierarchy + assembly (mesh.cpp, stencil.cpp), apply/residual/norm/dot/axpy
 * (stencil.cpp), the 11 preconditioned-Richardson smoothers (smoother.cpp),
 * transfers (transfer.cpp), banded Cholesky (stencil.cpp), adaptive omega,
 * V/W recursion, F-cycle and the outer solve loop (cycle.cpp). Every function
 * cites the reference file:line it follows. Operation order matches the
 * reference term by term; build with -ffp-contract=off (oracle/Makefile).
 *
 * Parity pin: tests/test_oracle_pin.py checks this restatement bit-for-bit
 * against the reference itself (oracle/_ref, built from the reference sources)
 * and against the committed golden fixtures tests/golden/ (*.json).
 */
#ifndef GMG_ORACLE_H
#define GMG_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

/* status codes: same meaning as include/gmg_b200.h */
#define ORC_OK 0
#define ORC_ERR_LOGIC 1
#define ORC_ERR_INVALID 2
#define ORC_ERR_RUNTIME 3
#define ORC_DIVERGED 4

typedef struct orc_problem orc_problem;

typedef struct orc_cycle {
    int cycle; /* 0 V, 1 W, 2 F */
    int pre_steps;
    int post_steps;
    int adaptive_correction;
    double correction_omega;
    int smoother_kind; /* reference SmootherKind order */
    double smoother_omega;
    double smoothing_omega;
    double tolerance;
    int max_cycles;
    unsigned long long coarse_direct_max_neq;
} orc_cycle;

const char* orc_last_error(void);

orc_problem* orc_problem_create(int levels, int coarse_nx, int coarse_ny, double grading_x,
                                double grading_y, int coords, double alpha, double beta);
void orc_problem_destroy(orc_problem* p);
int orc_num_levels(const orc_problem* p);
int orc_level_shape(const orc_problem* p, int level, int* nx, int* ny);
int orc_level_coords(const orc_problem* p, int level, double* x, double* y);
int orc_operator(const orc_problem* p, int level, double* c, double* n, double* s, double* e,
                 double* w);

int orc_apply(const orc_problem* p, int level, const double* x, double* y);
int orc_residual(const orc_problem* p, int level, const double* x, const double* b, double* r);
int orc_smooth_step(const orc_problem* p, int level, int kind, double smoother_omega,
                    double omega_damp, const double* x, const double* b, double* out);
int orc_restriction(const orc_problem* p, int fine_level, const double* fine, double* coarse);
int orc_prolongation(const orc_problem* p, int coarse_level, const double* coarse, double* fine);
int orc_adaptive_omega(const orc_problem* p, int level, const double* d, const double* corr,
                       double* omega);
int orc_coarse_solve(const orc_problem* p, const double* b, double* x);
double orc_norm_l2(long long n, const double* v);
double orc_dot(long long n, const double* a, const double* b);
void orc_axpy(long long n, double alpha, const double* x, double* y);

int orc_mg_cycle(const orc_problem* p, const orc_cycle* spec, int level, const double* u0,
                 const double* g, double* u);
int orc_solve(const orc_problem* p, const orc_cycle* spec, const double* b, double* x,
              double* history, int* history_len, int* iterations, int* converged);

/* make_start_vector (study.cpp:40-79): kind 0 zero, 1 nested */
int orc_start_vector(const orc_problem* p, const orc_cycle* spec, int kind, const double* b, double* x);

void orc_random_vector(long long n, unsigned seed, double* out);

#ifdef __cplusplus
}
#endif
#endif
