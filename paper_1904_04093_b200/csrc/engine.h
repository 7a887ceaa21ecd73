// Internal host-side declarations of the B200 GaBP engine (not part of the C-ABI).
#pragma once

#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/gabp_b200.h"
#include "kernels.cuh"
#include "rb_kernels.cuh"
#include "seq_kernels.cuh"
#include "seqpipe_kernels.cuh"
#include "sell_kernels.cuh"

namespace bgabp {

struct InvalidArg : std::invalid_argument {
    using std::invalid_argument::invalid_argument;
};
struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

void put_err(char* err, size_t len, const std::string& s);
void trim_block_cache();  // idle cached device blocks back to the driver (memory.cu)

// makes `dev` current for its lifetime (a handle's work runs on the device it was built on)
struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        if (dev < 0) return;
        cudaGetDevice(&prev);
        if (prev != dev) cudaSetDevice(dev);
        else prev = -1;
    }
    ~DeviceGuard() {
        if (prev >= 0) cudaSetDevice(prev);
    }
};
void release_block(void* p);  // engine device blocks back to the cache (memory.cu)
struct Engine;
void p2p_forget(Engine* e);  // drop captured multi-shard graphs that use this engine
// host <-> device copies of caller buffers: direct when pinned, staged (parallel) when pageable
void host_to_device(void* dst, const void* src, size_t bytes, cudaStream_t st);
void device_to_host(void* dst, const void* src, size_t bytes, cudaStream_t st);
void ck(cudaError_t e, const char* what);

inline double bits2d(unsigned long long b) {
    double d;
    std::memcpy(&d, &b, sizeof d);
    return d;
}

// dependency levels of one schedule's visit order (see k_level_dia)
struct Levels {
    std::vector<int> ptr;    // level l = nodes[ptr[l] .. ptr[l+1])
    std::vector<int> order;  // the schedule's visit order (for pivot messages)
    int* d_nodes = nullptr;
    int* d_npos = nullptr;   // position of each node in `order`
};

struct Engine {
    // matrix (host copy, canonical CSR) and message graph facts
    int n = 0;
    long long nnz = 0, num_edges = 0;
    std::vector<int> ro, ci;
    std::vector<double> val;
    std::vector<long long> tpos;
    bool symmetric = false;
    std::vector<int> uptr, unbr;  // union neighbour lists
    int layout = BGABP_LAYOUT_DIA, S = 0;
    long long nslots = 0;
    long long msg_cap = 0;  // elements of each d_msg buffer (>= nslots)
    DiaP dia{};
    CsrP csr{};
    std::vector<long long> csr2slot;

    // device state
    int device = -1;  // the device the handle was built on (build())
    long long peer_gen = 0;  // bumped when shard range / peers change (captured multi-shard graphs)
    cudaStream_t st = nullptr;
    bool own_stream = true;
    Ctrl* d_ctrl = nullptr;
    Ctrl* h_ctrl = nullptr;
    long long* d_csr2slot = nullptr;
    void ensure_csr2slot();
    // the matrix in HBM (canonical CSR); the host copies above exist once host_ready is set
    int* d_ro = nullptr;
    int* d_ci = nullptr;
    double* d_val = nullptr;
    bool host_ready = false;
    void ensure_host();  // ro/ci/val/tpos/uptr/unbr from the device CSR, on first use

    double2* d_msg[2] = {nullptr, nullptr};
    int cur = 0;
    double *d_b = nullptr, *d_x = nullptr, *d_r = nullptr, *d_e = nullptr, *d_aux = nullptr;
    double* d_hist = nullptr;
    double* d_xf = nullptr;          // fused flood solve: x(k) in ring slot k % kXRing ([kXRing][n])
    double* d_xord = nullptr;        // ordered solves: x(k) in slot k & 1 ([2][n]); pivot stops compose

    unsigned long long* d_spread = nullptr;  // per-warp max slots of the fused solve step
    long long hist_cap = 0;
    long long hist_gen = 0;  // bumped when d_hist is reallocated (captured graphs hold the pointer)
    void drop_graphs();
    double *d_lam = nullptr, *d_lsrc = nullptr, *d_sigma = nullptr;
    bool has_frozen = false;
    std::vector<void*> allocs;
    long long device_bytes = 0;
    std::map<std::string, std::unique_ptr<Levels>> level_cache;
    std::map<std::string, cudaGraphExec_t> graphs;

    // device-resident solve loop
    bool solve_flood = true;
    bool solve_fused = false;
    PeerP peer{};               // sharded solve: peer-memory halos and reduction slots
    bool peer_on = false;
    unsigned long long* d_slots = nullptr;  // [kMaxShards][2][4] reduction words of every shard
    cudaEvent_t step_ev = nullptr;          // recorded after each p2p step
    const Levels* solve_levels = nullptr;
    bool solve_rb = false;
    bool solve_seq = false;
    const double* solve_b = nullptr;
    int solve_stop = 0, solve_max_iter = 0;
    long long steps_enqueued = 0;
    int* h_poll = nullptr;  // pinned stop flags of the two chunks in flight (solve_run_to_end)
    cudaEvent_t poll_ev[2] = {nullptr, nullptr};
    std::vector<cudaEvent_t>* timed_events = nullptr;  // bgabp_solve_device_steps_timed
    int timed_index = 0;

    ~Engine();
    void* dalloc(size_t bytes);
    void dfree(void* p);
    template <class T>
    T* upload(const std::vector<T>& v);

    void build(int n, const int* ro, const int* ci, const double* v, int layout,
               cudaStream_t shared_stream = nullptr);
    void build_dia_device(const int* ro, const int* ci, const double* v);
    void build_dia_host();
    void build_ucsr_host();
    // general sparsity: SELL layout of the union graph for the fused solve step (sell.cu)
    static constexpr int kSellBuckets = 4;
    SellP sell[kSellBuckets]{};  // chunks of <= 8 / <= 16 / <= 32 slot rows (TMA-staged), wider (registers)
    unsigned sell_grid[6] = {0, 0, 0, 0, 0, 0};  // persistent grids of the TMA-staged kernel variants
    int sell_variant = 1;  // BGABP_SELL_TMA: 0 double-buffered, 1 single buffer / more warps (default)
    bool sell_reg = false;  // BGABP_SELL_KIND=reg: the register-cached kernels for every bucket (A/B)
    void sell_tma_setup();
    bool sell_ready = false;
    bool use_ucsr_solve = false;  // BGABP_UCSR_SOLVE=1: the three-launch union-CSR solve loop instead
    long long sell_slots = 0;
    void build_sell(const std::vector<uint8_t>& flg, const std::vector<double>& uc, const std::vector<double>& urow,
                    const std::vector<int>& urev, const double* d_diag);
    void launch_sell_step(bool dl);
    void host_graph(const int* ro, const int* ci, const double* v);
    void upload_host(void* dst, const void* src, size_t bytes);
    long long find_pos(int r, int c) const;
    std::vector<int> schedule_order(const bgabp_schedule& s);
    // validates the schedule (reference exceptions) and caches its levels
    void schedule_order_check(const bgabp_schedule& s) {
        if (s.kind != BGABP_SCHED_FLOOD) (void)levels_for(s);
    }
    const Levels& levels_for(const bgabp_schedule& s);

    void launch_flood(const double* b, double2* m0, double2* m1, double* x, int mode, bool delta,
                      long long xstride = 0);
    void launch_aggregate(const double* b, const double2* msg, double* x, double* beta, unsigned long long* npiv);
    // DIA only: rb_nx > 0, r written colour-compact for rb_smooth_add(r, ..., true); rpart, one
    // max |r| per 256-node block (residual_blocks() entries) instead of the atomic into rmax
    void launch_residual(const double* b, const double* x, double* r, unsigned long long* rmax, int mode,
                         long long xstride = 0, int rb_nx = 0, unsigned long long* rpart = nullptr);
    unsigned residual_blocks() const { return (unsigned)((n + 255) / 256); }
    void launch_levels(const Levels& L, const double* b, double2* msg, double* x, bool delta,
                       unsigned long long* dslot, int mode, long long xstride = 0);
    void launch_gs_levels(const Levels& L, const double* b, double* x);
    void launch_jacobi(const double* b, const double* x, double* xn);

    // colour-compact red-black path (rb_kernels.cuh) for 5-point grids with odd nx
    bool rb_ready = false;
    int rb_nx = 0;
    RbP rb{};
    double2* d_rbmsg = nullptr;
    bool rb_applicable(const bgabp_schedule& s) const;
    void rb_build(int nx, bool msgs = true);  // msgs: also the colour-compact message buffers
    void launch_gs_rb(const double* b, double* x);
    void launch_rb_sweep(const double* b, double* x, bool cold, bool delta, unsigned long long* dslot, int mode,
                         long long xstride = 0);
    void rb_state(bool to_compact, double2* natural);
    // cold smoothing with recorded lambda / sigma per sweep (multigrid smoother fast path)
    std::vector<double*> rb_lamrec, rb_sigrec;
    int rb_pre_sweeps = 0;
    bool rb_pre_failed = false;
    bool rb_precompute(int sweeps);
    void rb_smooth_add(const double* r, int sweeps, double* x, bool r_compact = false);
    // pipelined lexicographic sweep on 5-point grids (seq_kernels.cuh)
    bool grid5 = false;  // DIA offsets {-nx,-1,+1,+nx} with no wrap-around edges at row ends
    int grid5_nx = 0;
    bool grid5_full = false;  // ... and every in-grid neighbour entry is present (both directions)
    int* d_progress = nullptr;
    bool seq_applicable(const bgabp_schedule& s) const {
        return grid5 && s.kind == BGABP_SCHED_SEQUENTIAL && n > 0;
    }
    void launch_seq_sweep(const double* b, double2* msg, double* x, bool delta, unsigned long long* dslot, int mode,
                          long long xstride = 0);
    // pipelined lexicographic sweeps (seqpipe_kernels.cuh): many sweeps per launch
    double* d_xring = nullptr;   // [kPipeR][pipe_sn] x(t) of the solve, lane-skewed
    double2* d_pmsg = nullptr;   // [4][pipe_sn] the pipeline's in-slot messages, lane-skewed
    const double* pipe_x_out(int slot, int oslot, long long p);  // natural-order x of a ring slot
    unsigned long long* d_pprog = nullptr;
    PipeRed* d_pred = nullptr;
    int* d_pint = nullptr;  // [0] ticket, [1] decided
    int pipe_strips = 0, pipe_next = 1;
    std::map<int, int*> pipe_orders;  // ticket orders per batch size
    // lane-skewed copies of the pipeline's read-only node operands (seqpipe_kernels.cuh): element
    // (strip k, step s, lane i) = node (row 32k + i, column s - i), so the 32 lanes of a strip
    // read 32 consecutive elements at every step
    long long pipe_sn = 0;            // elements per skewed array (strips x (nx + 31) x 32)
    uint32_t* d_skmask = nullptr;     // [sn]
    double* d_skc = nullptr;          // [4][sn] out-edge coefficients (general coefficients only)
    double* d_skrow = nullptr;        // [4][sn] row coefficients (A not bit-symmetric)
    double* d_skdiag = nullptr;       // [sn]
    double* d_skb = nullptr;          // [sn] b of the current launch
    void pipe_setup(bool ring);
    bool pipe_fits() const { return (n / std::max(grid5_nx, 1) + 31) / 32 + 1 < 2 * kPipeR; }
    bool solve_pipe = false;  // the sequential solve runs pipelined (else one k_seq_grid5 per sweep)
    void pipe_reset();
    void launch_pipe(const double* b, double* x, int t0, int nsweeps, bool solve, bool delta);

    void reset_ctrl();
    void read_ctrl();
    std::string ordered_detail(const std::vector<int>& order, unsigned long long key) const;
    std::string decode_failure(const Ctrl& c, const std::vector<int>* order) const;

    int sweep(const double* b, const bgabp_schedule& s, double* x, std::string& err);

    void solve_begin(const double* b_dev, const bgabp_schedule& s, const bgabp_options& o,
                     const double* r0_override = nullptr);
    void enqueue_step();
    void enqueue_fused_kernel();  // the fused DIA flood step alone (solve loop and sharded steps)
    void enqueue_step_other();
    unsigned long long* d_red4 = nullptr;  // sharded solve: this rank's four reduction words
    void* d_pack = nullptr;
    long long pack_cap = 0;
    void solve_steps(int nsteps);
    double damping = 0.0;  // flood message damping (bgabp_set_damping); 0 = the reference's update
    void set_damping(double a);
    void check_damping(const bgabp_schedule& s) const;
    static constexpr int kChunk = 16;  // solve iterations per captured graph
    bool chunk_graph_eligible() const;
    cudaGraphExec_t chunk_graph(int len);
    bool solve_done();
    void solve_run_to_end();
    void solve_report(bgabp_report& rep, std::string& detail);
    const double* solve_x();  // after solve_report (composes the node-pivot x on the fused path)
    double sweep_flops() const;

    void ensure_frozen_buffers();
    void frozen_finish();
    void precompute_lambda(const bgabp_schedule& s, double tol, int max_iter, int& converged, int& iters);
    void correction_sweeps_dev(const double* r_dev, const bgabp_schedule& s, int sweeps, double* e_dev);
    int cold_sweeps_dev(const double* r_dev, const bgabp_schedule& s, int sweeps, double* e_dev, std::string& err,
                        bool check, int seq = 0);
    // probe of multigrid.cpp:54-70 on the device
    bool sweeps_expand(const bgabp_schedule& s);
};

unsigned nblk_host(long long n, int t = 256);

template <class T>
inline T* Engine::upload(const std::vector<T>& v) {
    T* d = static_cast<T*>(dalloc(sizeof(T) * v.size()));
    if (!v.empty()) ck(cudaMemcpyAsync(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice, st), "H2D");
    return d;
}


}  // namespace bgabp

// the C-ABI handle
struct bgabp_engine {
    bgabp::Engine E;
};

#define ABI_GUARD(ERRBUF, ERRLEN, ...)                           \
    try {                                                        \
        __VA_ARGS__                                              \
    } catch (const InvalidArg& ex) {                             \
        put_err(ERRBUF, ERRLEN, ex.what());                      \
        return BGABP_EINVAL;                                     \
    } catch (const CudaError& ex) {                              \
        put_err(ERRBUF, ERRLEN, ex.what());                      \
        return BGABP_ECUDA;                                      \
    } catch (const std::exception& ex) {                         \
        put_err(ERRBUF, ERRLEN, ex.what());                      \
        return BGABP_ERUNTIME;                                   \
    }


