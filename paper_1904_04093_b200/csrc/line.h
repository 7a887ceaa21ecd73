// Host side of line GaBP (line_kernels.cuh): the region GaBP engine of region_gabp.cpp for the
// grid-line regions of a 5-point operator, device-resident.
#pragma once

#include <string>
#include <vector>

#include "engine.h"
#include "line_kernels.cuh"

namespace bgabp {

struct LineEngine {
    int n = 0, nx = 0, ny = 0;
    long long nnz = 0;
    cudaStream_t st = nullptr;
    bool own_stream = false;
    LineP P{};
    // block messages, one scalar (Lambda, m) per (line -> node) edge: row edges and column edges
    // indexed by node, double-buffered for flood sweeps
    double *lr[2] = {}, *mr[2] = {}, *lc[2] = {}, *mc[2] = {};
    int cur = 0;
    double *d_fd = nullptr, *d_fy = nullptr, *d_x = nullptr, *d_b = nullptr, *d_hist = nullptr;
    long long hist_cap = 0;
    unsigned long long* d_fail = nullptr;
    LineCtrl* d_ctrl = nullptr;
    LineCtrl* h_ctrl = nullptr;
    std::vector<void*> allocs;

    ~LineEngine();
    void* dalloc(size_t bytes);
    // validates the grid-line region graph the way build_two_layer_region_graph does
    // (region.cpp:64-127) and uploads the couplings
    void build(int n, const int* ro, const int* ci, const double* v, int nx, int ny, cudaStream_t shared = nullptr);
    void reset_state();
    // one sweep on device b; x (device, nullable) receives the column-phase solution
    void sweep(const double* b, int mode, double* x, const int* done = nullptr);
    // first failure of the last sweep(s) (kNone if none), and its message (region_gabp.cpp:97-100,115-119)
    unsigned long long read_fail();
    std::string fail_message(unsigned long long key) const;
    void clear_fail();
    // flop_count_region(SharedInverse) (region_gabp.cpp:305-326)
    double sweep_flops() const;
    void set_state(const double* lam, const double* m);  // host, reference edge order
    void get_state(double* lam, double* m);
    // multigrid smoothing fast path: the factors of `sweeps` cold sweeps recorded once (false if
    // the recursion breaks down within them: the full sweep then reports it), then mean-only
    // sweeps on r with x += e folded into the last column phase
    std::vector<LineRec> rec_rows, rec_cols;
    int rec_sweeps = 0;
    bool rec_failed = false;
    bool record(int sweeps);
    void smooth_add(const double* r, int sweeps, double* x);
};

}  // namespace bgabp
