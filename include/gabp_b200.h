/*
 * gabp_b200.h — C-ABI of the B200 (sm_100a) GaBP hot path.
 *
 * This is the drop-in boundary for the reference's solver and smoother entry points in
 * proj/core (paths below are relative to /root/reference/proj/core).  Plain pointers and sizes,
 * no exceptions, no C++ or torch types.  A handle owns its device copy of the matrix, the
 * device message layout, the message buffers and one CUDA stream; it is not re-entrant, but
 * separate handles may be used concurrently from different threads.
 *
 * Host buffers are used by every call that has no `_device` suffix; those calls copy inputs to
 * the device, run, and copy results back before returning.  `_device` calls take device
 * pointers, enqueue on the handle's stream and return without synchronising unless stated.
 *
 * Return codes: BGABP_OK (0), BGABP_EINVAL (1, the reference throws std::invalid_argument),
 * BGABP_EPIVOT (2, the reference returns false / Diverged with the same message text),
 * BGABP_ECUDA (3), BGABP_ERUNTIME (4, the reference throws std::runtime_error).
 * Every call taking (err, errlen) writes the reference's message text there.
 */
#ifndef GABP_B200_H
#define GABP_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { BGABP_OK = 0, BGABP_EINVAL = 1, BGABP_EPIVOT = 2, BGABP_ECUDA = 3, BGABP_ERUNTIME = 4 };

/* ScheduleKind (schedule.hpp:9-15) + constructor used (schedule.cpp:51-103) */
enum {
    BGABP_SCHED_FLOOD = 0,           /* Schedule::parallel_flood()                         */
    BGABP_SCHED_SEQUENTIAL = 1,      /* Schedule::sequential(n)                            */
    BGABP_SCHED_RED_BLACK_GRID = 2,  /* Schedule::red_black_grid(nx, ny)                   */
    BGABP_SCHED_FOUR_COLOR_GRID = 3, /* Schedule::four_color_grid(nx, ny)                  */
    BGABP_SCHED_CUSTOM = 4,          /* Schedule::custom(order)                            */
    BGABP_SCHED_RED_BLACK = 5,       /* Schedule::red_black(A)  (greedy)                   */
    BGABP_SCHED_FOUR_COLOR = 6       /* Schedule::four_color(A) (greedy)                   */
};

/* SolveStatus (report.hpp:10) and StopCriterion (gabp.hpp:37) */
enum { BGABP_CONVERGED = 0, BGABP_DIVERGED = 1, BGABP_MAX_ITER = 2 };
enum { BGABP_STOP_RESIDUAL = 0, BGABP_STOP_MESSAGE_DELTA = 1 };

/* device message layout chosen at create time */
enum { BGABP_LAYOUT_AUTO = 0, BGABP_LAYOUT_DIA = 1, BGABP_LAYOUT_CSR = 2 };

typedef struct {
    int kind;
    int nx, ny;       /* grid kinds */
    const int* order; /* BGABP_SCHED_CUSTOM: permutation of 0..n-1 (host) */
} bgabp_schedule;

/* GabpOptions (gabp.hpp:39-45); pivot_floor is not a field: the reference never reads it
 * (gabp.hpp:43 vs the engine's private 1e-300, gabp.hpp:110) */
typedef struct {
    double tol;               /* absolute inf-norm tolerance (reference default 2e-4) */
    int max_iter;             /* reference default 20000 */
    int stop;                 /* BGABP_STOP_* */
    double divergence_factor; /* reference default 1e12 */
} bgabp_options;

/* SolveReport (report.hpp:21-28) minus the vectors, which are caller buffers */
typedef struct {
    int status;
    int iterations;
    double flop_estimate;
} bgabp_report;

typedef struct {
    int n;
    long long nnz;
    long long num_edges;          /* MessageGraph::num_edges (gabp.cpp:22) */
    int layout;                   /* BGABP_LAYOUT_DIA or BGABP_LAYOUT_CSR */
    int num_slots;                /* DIA: slots (distinct neighbour offsets) per node */
    int symmetric_values;         /* 1 if A == A^T bit for bit (residual reuses the sweep coefficients) */
    double bytes_per_sweep;       /* algorithmic B_sweep = 40 E + 24 n */
    double bytes_per_residual;    /* algorithmic B_res = 8 nnz + 16 n */
    long long device_bytes;       /* device memory held by the handle */
    int uniform_coefficients;     /* DIA constant-coefficient stencil: coefficients and diagonal are
                                     kernel parameters, not arrays (the solve step reads 32 E + 28 n) */
    long long sell_slots;         /* CSR layout: slots of the padded SELL solve layout (0 for DIA) */
} bgabp_info;

typedef struct bgabp_engine bgabp_engine;

/* ---- engine lifetime: GabpEngine::GabpEngine(const SparseMatrix&) (gabp.cpp:29-33) ----------
 * Input is canonical CSR (sparse.hpp:10-27: strictly increasing columns per row).  The reverse
 * edge index (SparseMatrix::transpose_pos, sparse.cpp:70-74) is rebuilt internally.
 * EINVAL "gabp: matrix has a structurally zero diagonal entry" as gabp.cpp:30-32. */
int bgabp_create(int n, const int* row_offsets, const int* col_indices, const double* values,
                 int layout, bgabp_engine** out, char* err, size_t errlen);
void bgabp_destroy(bgabp_engine* e);
int bgabp_get_info(const bgabp_engine* e, bgabp_info* info);
/* diagnostic: FNV-1a digest of the device layout (DIA mask/coefficients/diagonal, the CSR-position
 * slot map) and of the facts derived from it.  The layout is built by kernels from the uploaded
 * CSR; with the environment variable BGABP_HOST_BUILD set it is built on the host instead, and
 * the two digests of one matrix must be equal. */
int bgabp_layout_digest(bgabp_engine* e, unsigned long long* out);
/* the handle's CUDA stream (cudaStream_t), for callers that time or order work around it */
void* bgabp_stream(bgabp_engine* e);

/* ---- message state: MessageState (gabp.hpp:31-35) ----------------------------------------------
 * CSR-position indexed arrays of length nnz; diagonal slots read back as 0. */
int bgabp_reset_state(bgabp_engine* e); /* make_state(): zeros (gabp.cpp:35-40) */
int bgabp_set_state(bgabp_engine* e, const double* lambda_tilde, const double* m);
int bgabp_get_state(bgabp_engine* e, double* lambda_tilde, double* m);

/* ---- one sweep: GabpEngine::sweep(b, sched, state, x, &err) (gabp.cpp:42-47) ------------------
 * Advances the handle's state.  x is in/out (n): the sequential and coloured schedules write
 * every node they visit, flood writes all of x from the new messages (gabp.cpp:141-160).
 * EPIVOT with "zero pivot on edge j->i" / "zero pivot at node i" as gabp.cpp:71-74,83-87,126-130,
 * 155-158 (state contents after a breakdown are not contractual). */
int bgabp_sweep(bgabp_engine* e, const double* b, const bgabp_schedule* sched, double* x,
                char* err, size_t errlen);

/* node_precisions(state) (gabp.cpp:403-419) of the handle's current state */
int bgabp_node_precisions(bgabp_engine* e, double* beta);
/* Optional message damping of the flood sweep (BASELINE.json north_star; the reference has none,
 * SPEC.md:197): from now on every message the handle's flood sweeps and solves compute becomes
 * (1 - alpha) * new + alpha * old on its edge (products rounded before the add).  alpha = 0 (the
 * default) is the reference's update bit for bit.  EINVAL unless 0 <= alpha < 1; with alpha != 0
 * ordered schedules and sharded solves return EINVAL. */
int bgabp_set_damping(bgabp_engine* e, double alpha);
double bgabp_sweep_flops(const bgabp_engine* e); /* gabp.cpp:165-172 */

/* ---- solve(b, sched, opt) (gabp.cpp:174-219) ------------------------------------------------------
 * Starts from make_state() and leaves the handle's state at the last sweep run.  x_out (n) gets
 * the solution, history (max_iter+1, nullable) the residual history -- iterations + 1 entries, or
 * iterations on a pivot stop (detail "zero pivot ...": the failed sweep has no residual,
 * gabp.cpp:193-199; the buffer's next entry is then unspecified); detail gets
 * SolveReport::detail.  Iteration counts, statuses, details, histories and x follow the reference
 * exactly -- on a pivot stop x is the reference's partly updated x (gabp.cpp:71-87, 126-130,
 * 155-158).  b and x_out may be pageable (staged copies) or pinned (direct copies). */
int bgabp_solve(bgabp_engine* e, const double* b, const bgabp_schedule* sched,
                const bgabp_options* opt, bgabp_report* rep, double* x_out, double* history,
                char* detail, size_t detaillen);

/* Device-resident stepping form of bgabp_solve for drivers that keep b and x in HBM:
 *   begin: reset state, r0 = ||b||_inf (device b), arm the stop logic;
 *   steps: enqueue `nsteps` solve iterations (sweep + residual check + stop test) without
 *          synchronising; iterations after the stop decision are no-ops on the device;
 *   end:   synchronise and fill the report; x_dev (n) receives the solution, history_dev
 *          (max_iter+1) the residual history (both device pointers, nullable). */
int bgabp_solve_device_begin(bgabp_engine* e, const double* b_dev, const bgabp_schedule* sched,
                             const bgabp_options* opt);
int bgabp_solve_device_steps(bgabp_engine* e, int nsteps);
int bgabp_solve_device_end(bgabp_engine* e, bgabp_report* rep, double* x_dev, double* history_dev,
                           char* detail, size_t detaillen);
/* Same as bgabp_solve_device_steps, launched without graphs and with a CUDA event pair around
 * the hot kernel of every iteration (the fused flood sweep + residual for DIA flood solves);
 * synchronises and returns the summed device time of those launches in *hot_ms. */
int bgabp_solve_device_steps_timed(bgabp_engine* e, int nsteps, double* hot_ms);
/* `nsweeps` bare flood sweeps on device b (no residual, no stop logic; x of the previous sweep
 * is written to the handle's x buffer): the sweep kernel alone. */
int bgabp_flood_sweeps_device(bgabp_engine* e, const double* b_dev, int nsweeps);

/* ---- sharded flood solve (one contiguous row block per rank; no reference counterpart: the
 * reference is single-process, gabp.cpp:174-219 is the loop these steps split) -----------------
 * The handle holds the block's local matrix (owned rows + ghost rows, DIA layout).  set_range
 * restricts the fused step to the owned local nodes [own_lo, own_hi) and adds gofs (the global
 * index of local node 0) to the pivot keys.  Per iteration the driver calls step_compute, MAX
 * all-reduces the 4 int64 words at reduce_buffer across ranks, calls step_decide (the reference's
 * stop rule on the combined words, identical on every rank), then exchanges halos:
 * pack(which = t&1) the in-slot messages of the neighbour's nodes, unpack them on the neighbour
 * (only slots whose sender lies in [sender_lo, sender_hi)), and copy x buffer (t-1)&1 of owned
 * nodes into the neighbour's ghost range.  Every call is stream-ordered on bgabp_stream(e); r0 is
 * the global ||b||_inf.  End with bgabp_solve_device_end.  Pointers are device pointers. */
int bgabp_shard_set_range(bgabp_engine* e, int own_lo, int own_hi, int gofs);
/* DIA neighbour offsets of the handle (ascending; returns the slot count, -1 for the CSR layout).
 * Shards exchange halos slot by slot, so neighbouring shards must hold identical offsets
 * (shard.py checks this before wiring peers or starting a sharded solve). */
int bgabp_dia_offsets(const bgabp_engine* e, int* off, int cap);
int bgabp_shard_solve_begin(bgabp_engine* e, const double* b_dev, const bgabp_options* opt, double r0);
int bgabp_shard_step_compute(bgabp_engine* e);
void* bgabp_shard_reduce_buffer(bgabp_engine* e);
int bgabp_shard_step_decide(bgabp_engine* e);
void* bgabp_shard_msg(bgabp_engine* e, int which);
void* bgabp_shard_x(bgabp_engine* e, int which);
int bgabp_shard_pack(bgabp_engine* e, int which, int lo, int len, void* out_dev);
int bgabp_shard_unpack(bgabp_engine* e, int which, const void* recv_dev, int lo, int len, int sender_lo,
                       int sender_hi);
int bgabp_shard_state(bgabp_engine* e, int* done, int* step);
/* Peer-memory variant (direct peer stores instead of pack / collective / unpack).
 * The fused step stores the messages it computes for a neighbour's owned nodes straight into that
 * neighbour's message buffer (and x(t-1) of the neighbour's ghost nodes into its x slot), and the
 * fold writes the four reduction words into slot [rank][t & 1] of every shard; each shard then
 * waits for every other shard's step (bgabp_shard_p2p_wait) and decides on the MAX of the slots.
 * lower / upper = {msg buffer 0, msg buffer 1, x slot 0, x slot 1} device pointers of the
 * neighbour (bgabp_shard_msg / bgabp_shard_x; peer-mapped between GPUs), or NULL at the ends;
 * *_n = the neighbour's local node count, *_delta = its local index minus ours for the same
 * global node; own local nodes j < xlo_end are the lower neighbour's ghosts, j >= xhi_begin the
 * upper's; slots[q] = shard q's bgabp_shard_peer_slots array.  1 <= nranks <= 8. */
int bgabp_shard_peer_slots(bgabp_engine* e, void** slots);
int bgabp_shard_set_peers(bgabp_engine* e, int nranks, int rank, void* const* lower, int lower_n, int lower_delta,
                          void* const* upper, int upper_n, int upper_delta, int xlo_end, int xhi_begin,
                          void* const* slots);
int bgabp_shard_p2p_compute(bgabp_engine* e);
int bgabp_shard_p2p_wait(bgabp_engine* e, bgabp_engine* other);
/* spin = 0: the caller ordered this stream after every other shard's step (bgabp_shard_p2p_wait,
 * shards of one process); spin = 1: wait on the device for the other shards' step flags (shards
 * in other processes, slot arrays mapped with bgabp_ipc_*; ~20 s timeout -> Diverged "peer shard
 * timeout") */
int bgabp_shard_p2p_decide(bgabp_engine* e, int spin);
/* nsteps iterations of the peer-memory solve for the shards of one process (event-ordered);
 * use_graph: replay 16-iteration chunks from a CUDA graph captured across the shards' streams */
int bgabp_shard_p2p_steps(bgabp_engine* const* shards, int count, int nsteps, int use_graph);
/* one shard per process (peers mapped by CUDA IPC): nsteps iterations of p2p_compute followed by a
 * decision that waits on the peers' step flags on the device (spin), no host synchronisation */
int bgabp_shard_p2p_steps_ipc(bgabp_engine* e, int nsteps);
/* CUDA IPC of device allocations (64-byte handles) for shards in different processes */
int bgabp_ipc_get(const void* dev_ptr, void* handle_out);
int bgabp_ipc_open(const void* handle, void** dev_ptr);
int bgabp_ipc_close(void* dev_ptr);

/* residual_inf_norm(A, x, b) (sparse.cpp:104-115) on the handle's matrix */
int bgabp_residual_inf_norm(bgabp_engine* e, const double* x, const double* b, double* out);

/* ---- frozen-precision path (gabp.cpp:221-401) ------------------------------------------------------
 * precompute_lambda keeps the result on the device for the correction calls; lambda_out (nnz,
 * CSR order) and sigma_out (n) are nullable host copies.  set_frozen loads a FrozenLambda. */
int bgabp_precompute_lambda(bgabp_engine* e, const bgabp_schedule* sched, double tol, int max_iter,
                            double* lambda_out, double* sigma_out, int* converged, int* iterations);
int bgabp_set_frozen(bgabp_engine* e, const double* lambda_tilde, const double* sigma);
int bgabp_correction_sweeps(bgabp_engine* e, const double* r, const bgabp_schedule* sched,
                            int sweeps, double* e_out);
int bgabp_error_correction_apply(bgabp_engine* e, const double* b, const double* x0, int sweeps,
                                 const bgabp_schedule* sched, int use_frozen, double* x_out,
                                 char* err, size_t errlen);
int bgabp_solve_error_correction(bgabp_engine* e, const double* b, const bgabp_schedule* sched,
                                 int sweeps, const bgabp_options* opt, bgabp_report* rep,
                                 double* x_out, double* history, char* detail, size_t detaillen);

/* ---- line GaBP: region GaBP over grid lines (region_gabp.hpp:41-94, region_gabp.cpp:30-198 with
 * grid_line_regions, region.cpp:208-221) ---------------------------------------------------------
 * RegionGabpEngine(A, build_two_layer_region_graph(A, grid_line_regions(nx, ny))) for a 5-point
 * operator on an nx x ny grid (x fastest): large regions are the rows then the columns, children
 * the single nodes; bglin_create rejects the inputs build_two_layer_region_graph rejects, with its
 * messages.  Block messages are scalars, 2n edges in the reference's edge order (row edges by node,
 * then column edges column by column).  mode: 0 RegionSweepMode::Sequential, 1 Flood.  Local
 * systems are solved in O(N) per line (tridiagonal) instead of the reference's dense FullPivLU,
 * so results agree to rounding, not bitwise. */
typedef struct bglin_engine bglin_engine;
typedef struct {
    double tol;               /* RegionSolveOptions (region_gabp.hpp:25-30): default 2e-4 */
    int max_iter;             /* default 10000 */
    int mode;                 /* default 0 (Sequential) */
    double divergence_factor; /* default 1e12 */
} bglin_options;
int bglin_create(int n, const int* row_offsets, const int* col_indices, const double* values, int nx, int ny,
                 bglin_engine** out, char* err, size_t errlen);
void bglin_destroy(bglin_engine* e);
int bglin_num_edges(const bglin_engine* e);
double bglin_sweep_flops(const bglin_engine* e); /* flop_count_region(SharedInverse) */
void* bglin_stream(bglin_engine* e);
int bglin_reset_state(bglin_engine* e);
int bglin_set_state(bglin_engine* e, const double* lambda, const double* m);
int bglin_get_state(bglin_engine* e, double* lambda, double* m);
/* RegionGabpEngine::sweep: BGABP_EPIVOT with the reference's message on a singular local system */
int bglin_sweep(bglin_engine* e, const double* b, int mode, double* x, char* err, size_t errlen);
int bglin_solve(bglin_engine* e, const double* b, const bglin_options* opt, bgabp_report* rep, double* x_out,
                double* history, char* detail, size_t detaillen);

/* ---- multigrid with the GaBP smoother (multigrid.hpp:17-103, multigrid.cpp:54-318) ----------------
 * Levels are supplied by the caller finest first (the reference rediscretises a named problem per
 * level, multigrid.cpp:79-83; bgmg_create_named does that with the built-in assembly).  Smoother
 * numbering = MgSmoother (multigrid.hpp:17-31): 0 GabpSequential 1 GabpRedBlack 2 GabpFourColor
 * 3 GabpFlood 4 GabpLine 5 Jacobi 6 GsLex 7 GsRedBlack 8 GsFourColor.  Coarsening stops where the
 * sweeps_expand probe fires (multigrid.cpp:54-70, 89-93); the coarsest level is solved directly. */
typedef struct bgmg bgmg;
typedef struct {
    int pre, post; /* CycleSpec (multigrid.hpp:33-40) */
    int frozen;
} bgmg_cycle;
typedef struct {
    double tol;               /* MgSolveOptions (multigrid.hpp:96-100): absolute, default 2e-4 */
    int max_cycles;           /* default 200 */
    double divergence_factor; /* default 1e6 */
} bgmg_options;

int bgmg_create(int nlevels, const int* n, const int* const* row_offsets,
                const int* const* col_indices, const double* const* values, const int* nx,
                int smoother, bgmg** out, char* err, size_t errlen);
int bgmg_create_named(const char* problem, int J1, int J2, int nparam, const char* const* keys,
                      const double* vals, int smoother, bgmg** out, char* err, size_t errlen);
void bgmg_destroy(bgmg* h);
int bgmg_num_levels(const bgmg* h);
int bgmg_level_frozen_ok(const bgmg* h, int k);
int bgmg_level_n(const bgmg* h, int k);
int bgmg_level_nx(const bgmg* h, int k); /* grid points per axis of level k (GridLevel::prob.grid) */
/* Hierarchy::cycle_flops_per_unknown (multigrid.hpp:71-73, multigrid.cpp:240-274): the analytic
 * flop_table (analysis.cpp:135-154) of the pre + post sweeps, by the fine centre row's population */
int bgmg_cycle_flops_per_unknown(const bgmg* h, const bgmg_cycle* spec, double* out, char* err,
                                 size_t errlen);
/* fine-level right-hand side of a named hierarchy (Hierarchy::fine_rhs, multigrid.hpp:62) */
int bgmg_fine_rhs(const bgmg* h, double* b_out);
/* Hierarchy::v_cycle (multigrid.cpp:234-238): x updated in place; on a smoother breakdown returns
 * BGABP_ERUNTIME with the reference's message and x holding the updates made before it. */
int bgmg_vcycle(bgmg* h, const bgmg_cycle* spec, const double* b, double* x, char* err,
                size_t errlen);
/* mg_solve (multigrid.cpp:276-318).  rep->flop_estimate = cycle_flops_per_unknown * n per
 * completed cycle.  history (max_cycles + 1) receives iterations + 1 residuals, or iterations when
 * the last cycle ended in a smoother breakdown (status Diverged, detail other than "residual
 * blowup": that cycle has no residual, multigrid.cpp:288-297); x_out is then the reference's
 * partly cycled x (the level-0 updates made before the breakdown). */
int bgmg_solve(bgmg* h, const bgmg_cycle* spec, const double* b, const bgmg_options* opt,
               bgabp_report* rep, double* x_out, double* history, char* detail, size_t detaillen);
/* device-resident mg_solve: b_dev / x_dev device pointers; synchronises at every cycle's stop test */
int bgmg_solve_device(bgmg* h, const bgmg_cycle* spec, const double* b_dev,
                      const bgmg_options* opt, bgabp_report* rep, double* x_dev, double* history,
                      char* detail, size_t detaillen);
void* bgmg_stream(bgmg* h);
/* transfer operators on host buffers, run on the device (multigrid.cpp:111-161) */
int bgmg_restrict(const double* fine, int mf, double* coarse_out);
int bgmg_prolong(const double* coarse, int mc, double* fine_out);

/* ---- problem assembly (input generation; host only, no device work) ----------------------------
 * Named problems restate assemble(name, J, params) (problems.cpp:161-226); the config generators
 * are the BASELINE.json workloads the reference cannot assemble. */
typedef struct bgabp_problem bgabp_problem;
bgabp_problem* bgabp_problem_named(const char* name, int J, int nparam, const char* const* keys,
                                   const double* vals, char* err, size_t errlen);
bgabp_problem* bgabp_problem_poisson5(int nx, int ny);          /* tests/oracles.hpp:140-152 */
/* load_matrix_market (sparse.cpp:123-180): coordinate real general|symmetric; NULL + err on error */
bgabp_problem* bgabp_problem_matrix_market(const char* path, char* err, size_t errlen);
bgabp_problem* bgabp_problem_config(int config, int size, unsigned seed); /* configs 2..5 */
/* config-5 coarse level: same K field rule, level `k` below the finest (k=0 finest) */
bgabp_problem* bgabp_problem_config5_level(int J_fine, int k, unsigned seed);
/* the same family with another log-K standard deviation (config 5 uses sigma = 2) */
bgabp_problem* bgabp_problem_varcoef2d_level(int J_fine, int k, unsigned seed, double sigma);
/* the same with another coarse-K rule: 0 = full-weighted log K, 1 = full-weighted K (the
 * generator's: the rule with which the sigma = 2 V-cycle converges), 2 = full-weighted 1/K,
 * 3 = injection (tools/config5_coarse_rules.py compares them) */
bgabp_problem* bgabp_problem_varcoef2d_rule(int J_fine, int k, unsigned seed, double sigma, int rule);
void bgabp_problem_free(bgabp_problem* p);
int bgabp_problem_n(const bgabp_problem* p);
long long bgabp_problem_nnz(const bgabp_problem* p);
int bgabp_problem_nx(const bgabp_problem* p);
const int* bgabp_problem_row_offsets(const bgabp_problem* p);
const int* bgabp_problem_col_indices(const bgabp_problem* p);
const double* bgabp_problem_values(const bgabp_problem* p);
const double* bgabp_problem_rhs(const bgabp_problem* p);   /* b (n) */
const double* bgabp_problem_exact(const bgabp_problem* p); /* manufactured solution or NULL */

/* Give the idle device blocks of the process-wide block cache back to the driver (engine
 * allocations are cached for reuse by later handles; an allocation failure trims automatically). */
void bgabp_trim_cache(void);

/* library build tag (sm arch, git-independent) */
const char* bgabp_version(void);

#ifdef __cplusplus
}
#endif
#endif
