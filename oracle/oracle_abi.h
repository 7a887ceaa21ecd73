/*
 * TEST INFRASTRUCTURE ONLY — not part of the product path.
 *
 * Common C-ABI of the two CPU oracles for the GaBP hot path:
 *   - oracle/liboracle.so          : own restatement (oracle/gabp_restate.cpp), always built
 *   - oracle/_ref/libbelief_ref.so : the reference's own sources compiled from /root/reference
 *                                    (oracle/ref_shim.cpp over belief::GabpEngine; see oracle/Makefile)
 * Both export exactly these symbols so the tests can run the same case through either and
 * require bitwise agreement between them before trusting the restatement as the checker.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load these libraries.  The CUDA product never links or calls them.
 *
 * Schedule kinds (shared with include/gabp_b200.h):
 *   0 ParallelFlood              Schedule::parallel_flood()            schedule.cpp:51-55
 *   1 SequentialLexicographic    Schedule::sequential(n)               schedule.cpp:57-63
 *   2 RedBlack (grid)            Schedule::red_black_grid(nx, ny)      schedule.cpp:78-83
 *   3 FourColor (grid)           Schedule::four_color_grid(nx, ny)     schedule.cpp:85-91
 *   4 CustomOrder                Schedule::custom(order)               schedule.cpp:65-76
 *   5 RedBlack (greedy)          Schedule::red_black(A)                schedule.cpp:93-97
 *   6 FourColor (greedy)         Schedule::four_color(A)               schedule.cpp:99-103
 * Return codes: 1 ok, 0 pivot breakdown (err filled), -1 invalid argument (err filled).
 */
#ifndef GABP_ORACLE_ABI_H
#define GABP_ORACLE_ABI_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct orc_matrix orc_matrix;
typedef struct orc_engine orc_engine;
typedef struct orc_mg orc_mg;

typedef struct {
    int kind;
    int nx, ny;        /* grid kinds */
    const int* order;  /* custom kind: permutation of 0..n-1 */
} orc_sched;

/* ---- sparse storage (sparse.cpp) ---- */
orc_matrix* orc_make_csr(int n, long ntrip, const int* rows, const int* cols, const double* vals,
                         char* err, size_t errlen);
/* canonical CSR given directly; transpose_pos is recomputed as make_csr does (sparse.cpp:70-74) */
orc_matrix* orc_matrix_from_csr(int n, const int* row_offsets, const int* col_indices,
                                const double* values);
void orc_matrix_free(orc_matrix* A);
int orc_matrix_n(const orc_matrix* A);
long orc_matrix_nnz(const orc_matrix* A);
void orc_matrix_export(const orc_matrix* A, int* row_offsets, int* col_indices, double* values,
                       int* transpose_pos);
double orc_residual_inf_norm(const orc_matrix* A, const double* x, const double* b);
double orc_inf_norm(const double* v, long n);

/* ---- schedules (schedule.cpp) ---- */
int orc_schedule_order(orc_sched s, const orc_matrix* A, int* order_out, int* color_out,
                       int* num_colors);

/* ---- GaBP engine (gabp.cpp) ---- */
orc_engine* orc_engine_create(const orc_matrix* A, char* err, size_t errlen);
void orc_engine_free(orc_engine* e);
long orc_engine_num_edges(const orc_engine* e);
double orc_sweep_flops(const orc_engine* e);
/* state arrays lam/m are length nnz, CSR-position indexed (gabp.hpp:31-35) */
int orc_sweep(const orc_engine* e, const double* b, orc_sched s, double* lam, double* m, double* x,
              char* err, size_t errlen);
int orc_solve(const orc_engine* e, const double* b, orc_sched s, double tol, int max_iter,
              int stop_kind, double divergence_factor, double* x_out, double* history,
              int* iterations, int* status, double* flops, char* detail, size_t detaillen);
int orc_set_threads(int k); /* OpenMP threads of the restatement (1 in the reference build) */
/* BASELINE.json configs 3-5 (restatement only): matrix, b into b_out */
orc_matrix* orc_config3(int N, double pe_cell, double theta, unsigned seed, double* b_out);
orc_matrix* orc_config4(int N, double wx, double wy, double wz, unsigned seed, double* b_out);
orc_matrix* orc_config5_level(int J, int k, unsigned seed, double sigma, double* b_out);
int orc_set_damping(orc_engine* e, double alpha); /* restatement only (no reference damping) */
int orc_precompute_lambda(const orc_engine* e, orc_sched s, double tol, int max_iter,
                          double* lam_out, double* sigma_out, int* converged, int* iterations);
int orc_correction_sweeps(const orc_engine* e, const double* r, orc_sched s, const double* lam,
                          const double* sigma, int sweeps, double* e_out);
int orc_error_correction_apply_frozen(const orc_engine* e, const double* b, const double* x0,
                                      int sweeps, orc_sched s, const double* lam,
                                      const double* sigma, double* x_out);
int orc_error_correction_apply_cold(const orc_engine* e, const double* b, const double* x0,
                                    int sweeps, orc_sched s, double* x_out, char* err,
                                    size_t errlen);
int orc_solve_error_correction(const orc_engine* e, const double* b, orc_sched s, int sweeps,
                               const double* lam, const double* sigma, double tol, int max_iter,
                               double divergence_factor, double* x_out, double* history,
                               int* iterations, int* status, double* flops, char* detail,
                               size_t detaillen);
void orc_node_precisions(const orc_engine* e, const double* lam, const double* m, double* beta);

/* computation-tree oracle (analysis.cpp:160-215); returns 0 on error (err filled) */
int orc_computation_tree_solve(const orc_matrix* A, const double* b, int root, int depth,
                               long node_cap, double* out, char* err, size_t errlen);

/* ---- multigrid restatement (multigrid.cpp:54-318, Eigen-free) ---- */
/* smoother: 0 GabpSequential 1 GabpRedBlack 2 GabpFourColor 3 GabpFlood 6 GsLex 7 GsRedBlack
 * (numbering = belief::MgSmoother, multigrid.hpp:17-31) */
orc_mg* orc_mg_create(int nlevels, const orc_matrix* const* levels, const int* nx, int smoother,
                      char* err, size_t errlen);
void orc_mg_free(orc_mg* h);
int orc_mg_num_levels(const orc_mg* h);
int orc_mg_level_frozen_ok(const orc_mg* h, int k);
int orc_mg_vcycle(orc_mg* h, int pre, int post, int frozen, const double* b, double* x, char* err,
                  size_t errlen);
int orc_mg_solve(orc_mg* h, int pre, int post, int frozen, const double* b, double tol,
                 int max_cycles, double divergence_factor, double* x_out, double* history,
                 int* iterations, int* status, double* flops, int* hist_len, char* detail, size_t detaillen);
/* Hierarchy::cycle_flops_per_unknown (multigrid.cpp:240-274) and flop_table (analysis.cpp:135-154) */
double orc_mg_cycle_flops(const orc_mg* h, int pre, int post);
double orc_flop_table(int stencil, int smoother, int sweeps, char* err, size_t errlen);
void orc_mg_restrict(const double* fine, int mf, double* out);
void orc_mg_prolong(const double* coarse, int mc, double* out);
/* Gauss-Seidel in schedule order (classic.cpp:16-30) — comparison smoother */
int orc_gs_sweeps(const orc_matrix* A, const double* b, double* x, orc_sched s, int sweeps,
                  char* err, size_t errlen);

/* ---- dense partial-pivot LU (stands in for Eigen PartialPivLU, oracles.hpp:23-27) ---- */
int orc_dense_solve(const orc_matrix* A, const double* b, double* x);

/* ---- seeded test-input generators (restated from proj/tests/oracles.hpp; restatement lib only) */
typedef struct orc_rng orc_rng;
orc_rng* orc_rng_new(unsigned seed);
void orc_rng_free(orc_rng* r);
int orc_rng_uniform_int(orc_rng* r, int lo, int hi);
void orc_random_vector(orc_rng* r, int n, double* out);
orc_matrix* orc_random_diag_dominant(orc_rng* r, int n, int symmetric, double edge_prob);
orc_matrix* orc_random_tree(orc_rng* r, int n, int* edges_out /* 2*(n-1) or NULL */);
orc_matrix* orc_random_cycle_chords(orc_rng* r, int n);
orc_matrix* orc_poisson5(int nx, int ny);
orc_matrix* orc_example7x7(void);
int orc_tree_diameter(int n, const int* edges);

/* ---- region (line) GaBP restatement (region.cpp, region_gabp.cpp; see region_restate.inc) ---- */
typedef struct orc_region orc_region;
orc_region* orc_region_create(const orc_matrix* A, int nlarge, const int* offs, const int* idx, char* err,
                              size_t errlen);
void orc_region_free(orc_region* h);
int orc_region_num_edges(const orc_region* h);
int orc_region_num_small(const orc_region* h);
long orc_region_state_size(const orc_region* h, long* m_size);
void orc_region_edges(const orc_region* h, int* edge_large, int* edge_small);
long orc_region_small(const orc_region* h, int* offs, int* vars, int* poffs, int* parents, int* counting);
int orc_region_sweep(const orc_region* h, const double* b, int mode, double* lam, double* m, double* x, char* err,
                     size_t errlen);
int orc_region_solve(const orc_region* h, const double* b, double tol, int max_iter, int mode,
                     double divergence_factor, double* x_out, double* history, int* iterations, int* status,
                     double* flops, char* detail, size_t detaillen);
int orc_region_direct_message(const orc_region* h, const double* b, const double* lam, const double* m, int edge,
                              double* lam_out, double* m_out, char* err, size_t errlen);
double orc_region_flops(const orc_region* h, int per_child);

#ifdef __cplusplus
}
#endif
#endif
