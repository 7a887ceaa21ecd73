// Host side of the B200 GaBP engine behind include/gabp_b200.h.
//
// Replaces GabpEngine (proj/core/include/belief/gabp.hpp:58-111, src/gabp.cpp) with a handle that
// owns the device layout of the message graph, the message buffers and a CUDA stream.  This file
// holds the schedules (dependency levels), the sweep / solve loops and the C-ABI; construction is
// in build.cu, device memory and caller-buffer copies in memory.cu, the sharded solve in
// shard.cu.  Every sweep, residual and reduction runs in the kernels of kernels.cuh (and
// rb_ / seq_ / seqpipe_kernels.cuh).  There is no CPU fallback: a failed CUDA call is
// BGABP_ECUDA.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "engine.h"
#include "dia_tma_kernels.cuh"
#include "build_kernels.cuh"

namespace bgabp {

const char* kVersion = "gabp_b200 sm_100a";

// ---------------------------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------------------------
void put_err(char* err, size_t len, const std::string& s) {
    if (err && len) std::snprintf(err, len, "%s", s.c_str());
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
}

void Engine::drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second);
    graphs.clear();
    p2p_forget(this);
}

Engine::~Engine() {
    DeviceGuard g(device);  // the engine's device, not whichever one is current
    if (st) cudaStreamSynchronize(st);
    drop_graphs();
    if (!allocs.empty()) {
        // no kernel still uses the blocks: this device's, and a peer shard's on another device
        // (peers store into these buffers)
        cudaDeviceSynchronize();
        if (peer_on) {
            int nd = 0;
            cudaGetDeviceCount(&nd);
            for (int d = 0; d < nd; ++d)
                if (d != device) {
                    DeviceGuard gd(d);
                    cudaDeviceSynchronize();
                }
        }
    }
    for (void* p : allocs) release_block(p);
    if (h_ctrl) cudaFreeHost(h_ctrl);
    if (h_poll) cudaFreeHost(h_poll);
    if (step_ev) cudaEventDestroy(step_ev);
    for (auto& e : poll_ev)
        if (e) cudaEventDestroy(e);
    if (st && own_stream) cudaStreamDestroy(st);
}

// ---------------------------------------------------------------------------------------------
// schedules: node order (schedule.cpp) -> dependency levels over the union graph
// ---------------------------------------------------------------------------------------------
std::vector<int> Engine::schedule_order(const bgabp_schedule& s) {
    std::vector<int> order;
    auto grouped = [&](std::vector<int> colour) {  // schedule.cpp:11-22 (stable, ascending in colour)
        std::vector<int> o(colour.size());
        std::iota(o.begin(), o.end(), 0);
        std::stable_sort(o.begin(), o.end(), [&](int a, int b) { return colour[a] < colour[b]; });
        return o;
    };
    switch (s.kind) {
        case BGABP_SCHED_SEQUENTIAL:
            order.resize(n);
            std::iota(order.begin(), order.end(), 0);
            break;
        case BGABP_SCHED_RED_BLACK_GRID:
        case BGABP_SCHED_FOUR_COLOR_GRID: {
            if (s.nx < 0 || s.ny < 0) throw InvalidArg("gabp: bad grid shape");
            std::vector<int> col((size_t)s.nx * s.ny);
            for (int iy = 0; iy < s.ny; ++iy)
                for (int ix = 0; ix < s.nx; ++ix)
                    col[(size_t)iy * s.nx + ix] =
                        s.kind == BGABP_SCHED_RED_BLACK_GRID ? (ix + iy) % 2 : 2 * (iy % 2) + (ix % 2);
            order = grouped(std::move(col));
            break;
        }
        case BGABP_SCHED_CUSTOM: {  // schedule.cpp:65-76
            if (!s.order && n > 0) throw InvalidArg("Schedule::custom: order is not a permutation");
            order.assign(s.order, s.order + n);
            std::vector<char> seen(n, 0);
            for (int v : order) {
                if (v < 0 || v >= n || seen[v]) throw InvalidArg("Schedule::custom: order is not a permutation");
                seen[v] = 1;
            }
            break;
        }
        case BGABP_SCHED_RED_BLACK:
        case BGABP_SCHED_FOUR_COLOR: {  // greedy first fit over the undirected structure (schedule.cpp:25-47)
            ensure_host();
            std::vector<std::vector<int>> adj(n);
            for (int i = 0; i < n; ++i)
                for (int p = ro[i]; p < ro[i + 1]; ++p) {
                    const int j = ci[p];
                    if (j == i) continue;
                    adj[i].push_back(j);
                    adj[j].push_back(i);
                }
            std::vector<int> col(n, -1);
            int nc = 1;
            std::vector<char> used;
            for (int i = 0; i < n; ++i) {
                used.assign(nc + 1, 0);
                for (int j : adj[i])
                    if (col[j] >= 0 && col[j] < (int)used.size()) used[col[j]] = 1;
                int c = 0;
                while (c < (int)used.size() && used[c]) ++c;
                col[i] = c;
                nc = std::max(nc, c + 1);
            }
            order = grouped(std::move(col));
            break;
        }
        default:
            throw InvalidArg("gabp: unknown schedule kind " + std::to_string(s.kind));
    }
    if ((int)order.size() != n) throw InvalidArg("gabp: schedule order does not cover every node");
    return order;
}

const Levels& Engine::levels_for(const bgabp_schedule& s) {
    // the cache key needs no O(n log n) order build except for custom orders (the multigrid
    // smoother looks its levels up on every smoothing call)
    std::string key = std::to_string(s.kind) + ":" + std::to_string(s.nx) + "x" + std::to_string(s.ny);
    if (s.kind == BGABP_SCHED_CUSTOM) {  // FNV-1a of the order; a hit is confirmed element-wise
        unsigned long long hsh = 1469598103934665603ull;
        for (int q = 0; q < n && s.order; ++q) hsh = (hsh ^ (unsigned)s.order[q]) * 1099511628211ull;
        key += ":" + std::to_string(hsh);
    }
    auto it = level_cache.find(key);
    if (it != level_cache.end()) {
        if (s.kind != BGABP_SCHED_CUSTOM || (s.order && std::equal(s.order, s.order + n, it->second->order.begin())))
            return *it->second;
        drop_graphs();  // graphs captured with these levels (their key is the Levels address)
        level_cache.erase(it);
    }
    std::vector<int> order = schedule_order(s);
    ensure_host();
    std::vector<int> pos(n), lev(n, 0);
    for (int q = 0; q < n; ++q) pos[order[q]] = q;
    int nlev = 0;
    for (int q = 0; q < n; ++q) {
        const int j = order[q];
        int L = 0;
        for (long long s2 = uptr[j]; s2 < uptr[j + 1]; ++s2) {
            const int k = unbr[s2];
            if (pos[k] < q) L = std::max(L, lev[k] + 1);
        }
        lev[j] = L;
        nlev = std::max(nlev, L + 1);
    }
    auto lv = std::make_unique<Levels>();
    lv->ptr.assign(nlev + 1, 0);
    for (int j = 0; j < n; ++j) lv->ptr[lev[j] + 1]++;
    for (int l = 0; l < nlev; ++l) lv->ptr[l + 1] += lv->ptr[l];
    std::vector<int> nodes(n), npos(n);
    std::vector<int> fillp(lv->ptr.begin(), lv->ptr.end() - 1);
    for (int q = 0; q < n; ++q) {  // visit order kept within each level
        const int j = order[q];
        const int at = fillp[lev[j]]++;
        nodes[at] = j;
        npos[at] = q;
    }
    lv->order = order;
    lv->d_nodes = upload(nodes);
    lv->d_npos = upload(npos);
    ck(cudaStreamSynchronize(st), "levels sync");
    auto& ref = *lv;
    level_cache[key] = std::move(lv);
    return ref;
}

// ---------------------------------------------------------------------------------------------
// kernel launchers
// ---------------------------------------------------------------------------------------------
#define DIA_SWITCH(S_, ...)                                   \
    switch (S_) {                                             \
        case 2: { constexpr int SS = 2; __VA_ARGS__; } break; \
        case 4: { constexpr int SS = 4; __VA_ARGS__; } break; \
        case 6: { constexpr int SS = 6; __VA_ARGS__; } break; \
        case 8: { constexpr int SS = 8; __VA_ARGS__; } break; \
        default: throw InvalidArg("gabp: unsupported DIA slot count"); \
    }

unsigned nblk_host(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }
static inline unsigned nblk(long long n, int t = 256) { return nblk_host(n, t); }

void Engine::launch_flood(const double* b, double2* m0, double2* m1, double* x, int mode, bool delta,
                          long long xstride) {
    if (n == 0) return;
    const unsigned g = nblk(n);
    const bool damp = damping != 0.0;
    if (layout == BGABP_LAYOUT_DIA) {
        if (damp) {
            DIA_SWITCH(S, if (delta) k_flood_dia<SS, true, true><<<g, 256, 0, st>>>(dia, b, m0, m1, x, d_ctrl, mode);
                       else k_flood_dia<SS, false, true><<<g, 256, 0, st>>>(dia, b, m0, m1, x, d_ctrl, mode));
        } else {
            DIA_SWITCH(S, if (delta) k_flood_dia<SS, true><<<g, 256, 0, st>>>(dia, b, m0, m1, x, d_ctrl, mode);
                       else k_flood_dia<SS, false><<<g, 256, 0, st>>>(dia, b, m0, m1, x, d_ctrl, mode));
        }
    } else {
        if (delta && damp)
            k_flood_csr<true, true><<<g, 256, 0, st>>>(csr, b, m0, m1, x, d_ctrl, mode, xstride);
        else if (damp)
            k_flood_csr<false, true><<<g, 256, 0, st>>>(csr, b, m0, m1, x, d_ctrl, mode, xstride);
        else if (delta)
            k_flood_csr<true><<<g, 256, 0, st>>>(csr, b, m0, m1, x, d_ctrl, mode, xstride);
        else
            k_flood_csr<false><<<g, 256, 0, st>>>(csr, b, m0, m1, x, d_ctrl, mode, xstride);
    }
}

void Engine::launch_aggregate(const double* b, const double2* msg, double* x, double* beta,
                              unsigned long long* npiv) {
    if (n == 0) return;
    const unsigned g = nblk(n);
    if (layout == BGABP_LAYOUT_DIA) {
        DIA_SWITCH(S, k_aggregate_dia<SS><<<g, 256, 0, st>>>(dia, b, msg, x, beta, npiv));
    } else {
        k_aggregate_csr<<<g, 256, 0, st>>>(csr, b, msg, x, beta, npiv);
    }
}

void Engine::launch_residual(const double* b, const double* x, double* r, unsigned long long* rmax, int mode,
                             long long xstride, int rb_nx, unsigned long long* rpart) {
    if (n == 0) return;
    const unsigned g = nblk(n);
    if (layout == BGABP_LAYOUT_DIA) {
        if (dia.uniform) {
            DIA_SWITCH(S, k_residual_dia<SS, true, true><<<g, 256, 0, st>>>(dia, b, x, r, rmax, d_ctrl, mode, xstride, rb_nx, rpart));
        } else if (symmetric) {
            DIA_SWITCH(S, k_residual_dia<SS, true><<<g, 256, 0, st>>>(dia, b, x, r, rmax, d_ctrl, mode, xstride, rb_nx, rpart));
        } else {
            DIA_SWITCH(S, k_residual_dia<SS><<<g, 256, 0, st>>>(dia, b, x, r, rmax, d_ctrl, mode, xstride, rb_nx, rpart));
        }
    } else {
        k_residual_csr<<<g, 256, 0, st>>>(csr, b, x, r, rmax, d_ctrl, mode, xstride);
    }
}

void Engine::launch_levels(const Levels& L, const double* b, double2* msg, double* x, bool delta,
                           unsigned long long* dslot, int mode, long long xstride) {
    for (size_t l = 0; l + 1 < L.ptr.size(); ++l) {
        const int cnt = L.ptr[l + 1] - L.ptr[l];
        const int* nodes = L.d_nodes + L.ptr[l];
        const int* npos = L.d_npos + L.ptr[l];
        const unsigned g = nblk(cnt);
        if (layout == BGABP_LAYOUT_DIA) {
            DIA_SWITCH(S, if (delta) k_level_dia<SS, true><<<g, 256, 0, st>>>(dia, b, msg, x, nodes, npos, cnt, d_ctrl, dslot, mode, xstride);
                       else k_level_dia<SS, false><<<g, 256, 0, st>>>(dia, b, msg, x, nodes, npos, cnt, d_ctrl, dslot, mode, xstride));
        } else {
            if (delta)
                k_level_csr<true><<<g, 256, 0, st>>>(csr, b, msg, x, nodes, npos, cnt, d_ctrl, dslot, mode, xstride);
            else
                k_level_csr<false><<<g, 256, 0, st>>>(csr, b, msg, x, nodes, npos, cnt, d_ctrl, dslot, mode, xstride);
        }
    }
}

void Engine::launch_gs_levels(const Levels& L, const double* b, double* x) {
    for (size_t l = 0; l + 1 < L.ptr.size(); ++l) {
        const int cnt = L.ptr[l + 1] - L.ptr[l];
        const int* nodes = L.d_nodes + L.ptr[l];
        const int* npos = L.d_npos + L.ptr[l];
        if (layout == BGABP_LAYOUT_DIA) {
            DIA_SWITCH(S, k_gs_level_dia<SS><<<nblk(cnt), 256, 0, st>>>(dia, b, x, nodes, npos, cnt, d_ctrl));
        } else {
            k_gs_level_csr<<<nblk(cnt), 256, 0, st>>>(csr, b, x, nodes, npos, cnt, d_ctrl);
        }
    }
}

void Engine::launch_jacobi(const double* b, const double* x, double* xn) {
    if (n == 0) return;
    if (layout == BGABP_LAYOUT_DIA) {
        DIA_SWITCH(S, k_jacobi_dia<SS><<<nblk(n), 256, 0, st>>>(dia, b, x, xn, d_ctrl));
    } else {
        k_jacobi_csr<<<nblk(n), 256, 0, st>>>(csr, b, x, xn, d_ctrl);
    }
}

void Engine::reset_ctrl() {
    Ctrl c;
    std::memset(&c, 0, sizeof(c));
    for (int q = 0; q < 4; ++q) {
        c.epiv[q] = kNone;
        c.npiv[q] = kNone;
    }
    c.opiv = kNone;
    ck(cudaMemcpyAsync(d_ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, st), "ctrl reset");
    ck(cudaStreamSynchronize(st), "ctrl sync");
}

void Engine::read_ctrl() {
    ck(cudaMemcpyAsync(h_ctrl, d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "ctrl D2H");
    ck(cudaStreamSynchronize(st), "ctrl sync");
}

std::string Engine::ordered_detail(const std::vector<int>& order, unsigned long long key) const {
    const int pos = (int)(key >> 32);
    const unsigned sub = (unsigned)(key & 0xffffffffu);
    const int j = order[pos];
    if (sub == 0) return "zero pivot at node " + std::to_string(j);
    return "zero pivot on edge " + std::to_string(j) + "->" + std::to_string((int)sub - 1);
}

// ---------------------------------------------------------------------------------------------
// one sweep (gabp.cpp:42-47)
// ---------------------------------------------------------------------------------------------
void Engine::set_damping(double a) {
    if (!(a >= 0.0 && a < 1.0)) throw InvalidArg("gabp: damping must lie in [0, 1)");
    if (a == damping) return;
    ck(cudaStreamSynchronize(st), "sync");
    drop_graphs();  // captured solve chunks hold the undamped (or damped) kernels
    damping = a;
    dia.damp = csr.damp = a;
    dia.undamp = csr.undamp = 1.0 - a;
}

void Engine::check_damping(const bgabp_schedule& s) const {
    if (damping != 0.0 && s.kind != BGABP_SCHED_FLOOD)
        throw InvalidArg("gabp: message damping applies to the parallel flood schedule only");
}

int Engine::sweep(const double* b, const bgabp_schedule& s, double* x, std::string& err) {
    check_damping(s);
    if (s.kind == BGABP_SCHED_FLOOD) {
        if (n == 0) return BGABP_OK;
        reset_ctrl();
        ck(cudaMemcpyAsync(d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D b");
        launch_flood(d_b, d_msg[cur], d_msg[cur ^ 1], nullptr, MODE_PLAIN, false);
        cur ^= 1;
        launch_aggregate(d_b, d_msg[cur], d_x, nullptr, &d_ctrl->npiv[0]);
        ck(cudaGetLastError(), "flood launch");
        read_ctrl();
        if (h_ctrl->epiv[1] != kNone) {  // edge stage failed: x untouched (gabp.cpp:126-130)
            const unsigned long long k = h_ctrl->epiv[1];
            err = "zero pivot on edge " + std::to_string(k >> 32) + "->" + std::to_string(k & 0xffffffffu);
            return BGABP_EPIVOT;
        }
        if (h_ctrl->npiv[0] != kNone) {  // the x-stage stopped at the pivot node (gabp.cpp:155-158)
            const unsigned long long piv = h_ctrl->npiv[0];
            if (piv > 0) ck(cudaMemcpyAsync(x, d_x, sizeof(double) * (size_t)piv, cudaMemcpyDeviceToHost, st), "D2H x");
            ck(cudaStreamSynchronize(st), "sync");
            err = "zero pivot at node " + std::to_string(piv);
            return BGABP_EPIVOT;
        }
        ck(cudaMemcpyAsync(x, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H x");
        ck(cudaStreamSynchronize(st), "sync");
        return BGABP_OK;
    }
    const Levels& L = levels_for(s);
    if (n == 0) return BGABP_OK;
    reset_ctrl();
    ck(cudaMemcpyAsync(d_b, b, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D b");
    ck(cudaMemcpyAsync(d_x, x, sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D x");
    if (rb_applicable(s)) {  // same visit, colour-compact storage (state converted around it)
        rb_build(s.nx);
        rb_state(true, d_msg[cur]);
        launch_rb_sweep(d_b, d_x, false, false, nullptr, MODE_PLAIN);
        rb_state(false, d_msg[cur]);
    } else if (seq_applicable(s)) {  // lexicographic order on a 5-point grid: one pipelined launch
        launch_seq_sweep(d_b, d_msg[cur], d_x, false, nullptr, MODE_PLAIN);
    } else {
        launch_levels(L, d_b, d_msg[cur], d_x, false, nullptr, MODE_PLAIN);
    }
    ck(cudaGetLastError(), "level launch");
    read_ctrl();
    if (h_ctrl->opiv != kNone) {
        // the visit stopped at position p (gabp.cpp:71-87): nodes visited before it (and the
        // pivot node on an edge pivot, whose x was written) take the new x, the rest keep the caller's
        const unsigned long long key = h_ctrl->opiv;
        const long long p = (long long)(key >> 32) + ((key & 0xffffffffu) ? 1 : 0);
        std::vector<double> xn((size_t)n);
        ck(cudaMemcpyAsync(xn.data(), d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H x");
        ck(cudaStreamSynchronize(st), "sync");
        for (long long q = 0; q < p && q < n; ++q) x[L.order[q]] = xn[L.order[q]];
        err = ordered_detail(L.order, key);
        return BGABP_EPIVOT;
    }
    ck(cudaMemcpyAsync(x, d_x, sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H x");
    ck(cudaStreamSynchronize(st), "sync");
    return BGABP_OK;
}

// ---------------------------------------------------------------------------------------------
// solve (gabp.cpp:174-219): device-resident loop, stop logic in k_solve_finalize*
// ---------------------------------------------------------------------------------------------
void Engine::solve_begin(const double* b_dev, const bgabp_schedule& s, const bgabp_options& o,
                         const double* r0_override) {
    check_damping(s);
    if (damping != 0.0 && r0_override) throw InvalidArg("gabp: message damping is not supported by sharded solves");
    solve_flood = s.kind == BGABP_SCHED_FLOOD;
    // the fused step: DIA stencils, or the SELL layout for general sparsity (not sharded)
    solve_fused = solve_flood && (layout == BGABP_LAYOUT_DIA || (sell_ready && !r0_override && !use_ucsr_solve));
    solve_levels = solve_flood ? nullptr : &levels_for(s);
    solve_rb = !solve_flood && rb_applicable(s);
    solve_seq = !solve_flood && !solve_rb && seq_applicable(s);
    if (solve_rb) rb_build(s.nx);
    solve_b = b_dev;
    solve_stop = o.stop;
    solve_max_iter = o.max_iter;
    if (hist_cap < (long long)std::max(o.max_iter, 0) + 2) {
        hist_cap = (long long)std::max(o.max_iter, 0) + 2;
        // captured solve graphs hold the old history pointer: drop them with it
        ck(cudaStreamSynchronize(st), "sync");
        drop_graphs();
        if (d_hist) dfree(d_hist);
        d_hist = static_cast<double*>(dalloc(sizeof(double) * hist_cap));
        ++hist_gen;
    }
    Ctrl c;
    std::memset(&c, 0, sizeof(c));
    c.tol = o.tol;
    c.divergence = o.divergence_factor;
    c.stop = o.stop;
    c.max_iter = o.max_iter;
    ck(cudaMemcpyAsync(d_ctrl, &c, sizeof(Ctrl), cudaMemcpyHostToDevice, st), "ctrl");
    for (int k = 0; k < 2; ++k)
        ck(cudaMemsetAsync(d_msg[k], 0, sizeof(double2) * (size_t)std::max<long long>(msg_cap, 1), st), "memset");
    ck(cudaMemsetAsync(d_x, 0, sizeof(double) * std::max(n, 1), st), "memset x");
    if (!solve_fused && !(solve_seq && pipe_fits())) {  // ordered (not pipelined), or union-CSR flood
        if (!d_xord) d_xord = static_cast<double*>(dalloc(sizeof(double) * 2 * (size_t)std::max(n, 1)));
        ck(cudaMemsetAsync(d_xord, 0, sizeof(double) * 2 * (size_t)std::max(n, 1), st), "memset x ring");
    }
    if (solve_fused) {
        if (!d_xf) d_xf = static_cast<double*>(dalloc(sizeof(double) * kXRing * (size_t)std::max(n, 1)));
        ck(cudaMemsetAsync(d_xf, 0, sizeof(double) * kXRing * (size_t)std::max(n, 1), st), "memset x ring");
    }
    ck(cudaMemsetAsync(d_spread, 0, sizeof(unsigned long long) * 8 * kSpread, st), "memset");
    if (d_slots)  // peer-memory shards: words and step flags of the previous solve
        ck(cudaMemsetAsync(d_slots, 0, sizeof(unsigned long long) * (kSlotWords + kMaxShards), st), "memset");
    if (solve_rb) ck(cudaMemsetAsync(d_rbmsg, 0, sizeof(double2) * 4 * (size_t)std::max(n, 2), st), "memset");
    solve_pipe = solve_seq && pipe_fits();
    if (solve_pipe) {  // pipelined lexicographic sweeps: x(0) = 0 in ring slot 0
        pipe_setup(true);
        pipe_reset();
        ck(cudaMemsetAsync(d_xring, 0, sizeof(double) * (size_t)pipe_sn, st), "memset ring");
        pipe_next = 1;
    }
    cur = 0;
    if (r0_override) {  // sharded solve: ||b||_inf over all ranks, supplied by the driver
        unsigned long long bits;
        std::memcpy(&bits, r0_override, sizeof bits);
        ck(cudaMemcpyAsync(&d_ctrl->red[0], &bits, sizeof bits, cudaMemcpyHostToDevice, st), "r0");
        ck(cudaStreamSynchronize(st), "sync");
    } else if (n > 0) {
        k_inf_norm<<<std::min<unsigned>(nblk(n), 1184), 256, 0, st>>>(b_dev, n, &d_ctrl->red[0]);
    }
    k_solve_arm<<<1, 1, 0, st>>>(d_ctrl, d_hist);
    ck(cudaGetLastError(), "solve arm");
    steps_enqueued = 0;
    // capture (not run) the iteration chunk now, so the first steps call replays it instead of
    // paying capture + instantiation inside the caller's loop; shard solves use their own graphs
    if (!r0_override && chunk_graph_eligible())
        for (int len = kChunk; len >= 1; len >>= 1) chunk_graph(len);
}

void Engine::enqueue_step() {
    if (solve_fused) {
        enqueue_fused_kernel();
        k_solve_decide_lag2<<<1, kSpread, 0, st>>>(d_ctrl, d_hist, d_spread);
        return;
    }
    enqueue_step_other();
}

// the sharded fused step (runtime node range / global pivot keys), with or without peer halos
template <int SS, int MB, bool DF>
static void launch_sharded_step(Engine& E, unsigned g, bool dl) {
    double *x0 = E.d_xf, *x1 = E.d_xf + E.n;
#define SHARDED_STEP(DL_, SYM_, PEER_, UNIF_)                                                                   \
    k_flood_solve_dia<SS, DL_, SYM_, MB, DF, true, UNIF_, true, PEER_><<<g, 256, 0, E.st>>>(                   \
        E.dia, E.solve_b, E.d_msg[0], E.d_msg[1], x0, x1, E.d_ctrl, E.d_spread, E.peer)
    if (E.peer_on && E.dia.uniform) {  // constant stencil: coefficients and diagonal as parameters
        if (dl) SHARDED_STEP(true, true, true, true); else SHARDED_STEP(false, true, true, true);
    } else if (E.peer_on) {
        if (E.symmetric) {
            if (dl) SHARDED_STEP(true, true, true, false); else SHARDED_STEP(false, true, true, false);
        } else {
            if (dl) SHARDED_STEP(true, false, true, false); else SHARDED_STEP(false, false, true, false);
        }
    } else {
        if (E.symmetric) {
            if (dl) SHARDED_STEP(true, true, false, false); else SHARDED_STEP(false, true, false, false);
        } else {
            if (dl) SHARDED_STEP(true, false, false, false); else SHARDED_STEP(false, false, false, false);
        }
    }
#undef SHARDED_STEP
}

// The bulk-copy staged step (dia_tma_kernels.cuh): persistent warps, one grid per SM count x
// resident blocks.  BGABP_DIA_TMA=0 keeps the one-thread-per-node step (A/B).
template <int S, bool DL, bool SYM, bool UNIF, int WPB, int NPL, int MINB>
static void launch_dia_tma_t(Engine& E) {
    constexpr size_t smem = dia_tma_smem<S, NPL, WPB>();
    auto kfn = k_flood_solve_dia_tma<S, DL, SYM, UNIF, WPB, NPL, MINB>;
    static int grids[64] = {};  // per device: the attribute is set per device context
    const int dev = std::min(std::max(E.device, 0), 63);
    int& grid = grids[dev];
    if (!grid) {
        DeviceGuard g(E.device);
        ck(cudaFuncSetAttribute(kfn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem), "dia tma smem");
        int bps = 1, sms = 148;
        ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, kfn, 32 * WPB, smem), "occupancy");
        ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, E.device), "sm count");
        grid = sms * std::max(bps, 1);
    }
    kfn<<<grid, 32 * WPB, smem, E.st>>>(E.dia, E.solve_b, E.d_msg[0], E.d_msg[1], E.d_xf, E.d_xf + E.n, E.d_ctrl,
                                        E.d_spread);
}

// Two nodes per lane, 4 blocks of 4 warps per SM (16 warps, 124 registers).  Measured on config 2
// (ms per step): 2 blocks of 8 warps 0.1075, 4 of 4 0.1072; one node per lane with 24 warps
// (80 registers, small spills) 0.1092, with 32 warps (64 registers, spills) 0.1440.
template <int S, bool DL>
static void launch_dia_tma_v(Engine& E) {
    launch_dia_tma_t<S, DL, true, true, 4, 2, 4>(E);
}

template <int S>
static void launch_dia_tma_s(Engine& E, bool dl) {  // constant stencils only (see enqueue_fused_kernel)
    if (dl) launch_dia_tma_v<S, true>(E); else launch_dia_tma_v<S, false>(E);
}

static bool dia_tma_enabled() {
    static const bool on = !(getenv("BGABP_DIA_TMA") && std::string(getenv("BGABP_DIA_TMA")) == "0");
    return on;
}

void Engine::enqueue_fused_kernel() {
    if (layout != BGABP_LAYOUT_DIA) {  // general sparsity: the SELL step
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index], st), "event");
        launch_sell_step(solve_stop == BGABP_STOP_MESSAGE_DELTA);
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index + 1], st), "event");
        return;
    }
    {
        const bool dl = solve_stop == BGABP_STOP_MESSAGE_DELTA;
        const unsigned g = nblk(std::max(dia.j1 - dia.j0, 1));
        const bool sharded = dia.j0 != 0 || dia.j1 != n || dia.gofs != 0;
        // constant stencils (config 2): the bulk-copy staged step, 1-5 % faster than the
        // one-thread-per-node step depending on the box; with coefficient columns to gather
        // (configs 3, 4) the thread-per-node step is faster (0.041 vs 0.051 ms, 0.72 vs 0.83 ms)
        if (!sharded && damping == 0.0 && dia.uniform && n > 0 && n % kTmaTile == 0 && dia_tma_enabled()) {
            if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index], st), "event");
            switch (S) {
                case 2: launch_dia_tma_s<2>(*this, dl); break;
                case 4: launch_dia_tma_s<4>(*this, dl); break;
                case 6: launch_dia_tma_s<6>(*this, dl); break;
                case 8: launch_dia_tma_s<8>(*this, dl); break;
                default: throw InvalidArg("gabp: unsupported DIA slot count");
            }
            ck(cudaGetLastError(), "dia tma step");
            if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index + 1], st), "event");
            return;
        }
        // register cap per slot count: 4 resident blocks for 2-4 slots, fewer for 6-8 (no spills)
#define FUSED(SS_, MB_, DF_, MBU_, DFU_)                                                                            \
    if (sharded) {                                                                                                 \
        launch_sharded_step<SS_, MB_, DF_>(*this, g, dl);                                                          \
    } else if (damping != 0.0) {  /* damped messages: the general-coefficient step (c arrays exist) */           \
        if (symmetric) {                                                                                           \
            if (dl) k_flood_solve_dia<SS_, true, true, MB_, DF_, true, false, false, false, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
            else k_flood_solve_dia<SS_, false, true, MB_, DF_, true, false, false, false, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
        } else {                                                                                                   \
            if (dl) k_flood_solve_dia<SS_, true, false, MB_, DF_, true, false, false, false, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
            else k_flood_solve_dia<SS_, false, false, MB_, DF_, true, false, false, false, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
        }                                                                                                          \
    } else if (dia.uniform) {                                                                                      \
        if (dl) k_flood_solve_dia<SS_, true, true, MBU_, DFU_, true, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
        else k_flood_solve_dia<SS_, false, true, MBU_, DFU_, true, true><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
    } else if (symmetric) {                                                                                        \
        if (dl) k_flood_solve_dia<SS_, true, true, MB_, DF_><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
        else k_flood_solve_dia<SS_, false, true, MB_, DF_><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
    } else {                                                                                                       \
        if (dl) k_flood_solve_dia<SS_, true, false, MB_, DF_><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
        else k_flood_solve_dia<SS_, false, false, MB_, DF_><<<g, 256, 0, st>>>(dia, solve_b, d_msg[0], d_msg[1], d_xf, d_xf + n, d_ctrl, d_spread); \
    }
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index], st), "event");
        // (resident blocks, deferred x loads) per slot count, from tools/exp_flood.cu on the B200:
        // S=4 2048^2: (3, early) 133 us vs (4, deferred) 135; S=6 256^3: (4, deferred) 696 us vs (3, early) 725
        // uniform-coefficient variants (no coefficient / diagonal loads): S=4 2048^2 112.6 us with
        // (4, early), S=6 256^3 602 us with (4, deferred)
        switch (S) {
            case 2: FUSED(2, 4, true, 4, true) break;
            case 4: FUSED(4, 3, false, 4, false) break;
            case 6: FUSED(6, 4, true, 4, true) break;
            case 8: FUSED(8, 2, true, 2, true) break;
            default: throw InvalidArg("gabp: unsupported DIA slot count");
        }
#undef FUSED
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index + 1], st), "event");
    }
}

void Engine::enqueue_step_other() {
    if (solve_flood) {
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index], st), "event");
        // x(k) in slot k & 1 of d_xord: a node-pivot stop composes the partly updated x
        launch_flood(solve_b, d_msg[0], d_msg[1], d_xord, MODE_SOLVE, solve_stop == BGABP_STOP_MESSAGE_DELTA, n);
        if (timed_events) ck(cudaEventRecord((*timed_events)[2 * timed_index + 1], st), "event");
        launch_residual(solve_b, d_xord, nullptr, nullptr, MODE_SOLVE, n);
        k_solve_finalize<<<1, 1, 0, st>>>(d_ctrl, d_hist);
    } else if (solve_pipe) {  // one pipelined sweep (the timed path; solve_steps batches them)
        if (pipe_next <= solve_max_iter) {
            launch_pipe(solve_b, d_xring, pipe_next, 1, true, solve_stop == BGABP_STOP_MESSAGE_DELTA);
            ++pipe_next;
        }
    } else {
        // x(t) goes to slot t & 1 of d_xord (the kernels pick the slot from the device's step), so a
        // pivot stop still has x(t-1) for the reference's partly updated x (solve_x)
        if (solve_rb)
            launch_rb_sweep(solve_b, d_xord, false, solve_stop == BGABP_STOP_MESSAGE_DELTA, &d_ctrl->delta[0], MODE_SOLVE,
                            n);
        else if (solve_seq)  // grids too tall for the pipeline's x ring
            launch_seq_sweep(solve_b, d_msg[0], d_xord, solve_stop == BGABP_STOP_MESSAGE_DELTA, &d_ctrl->delta[0],
                             MODE_SOLVE, n);
        else
            launch_levels(*solve_levels, solve_b, d_msg[0], d_xord, solve_stop == BGABP_STOP_MESSAGE_DELTA,
                          &d_ctrl->delta[0], MODE_SOLVE, n);
        launch_residual(solve_b, d_xord, nullptr, nullptr, MODE_SOLVE_ORDERED, n);
        k_solve_finalize_ordered<<<1, 1, 0, st>>>(d_ctrl, d_hist);
    }
}

bool Engine::chunk_graph_eligible() const {
    const size_t per_step = solve_fused ? 2 : solve_flood ? 3 : solve_levels->ptr.size() + 1;
    return per_step * kChunk <= 4096 && n > 0 && !solve_seq;  // cooperative launches stay out of graphs
}

// The captured graph of `len` iterations of the current solve (len = kChunk or a power of two
// below it for the remainder of a steps call).  Captured on first use; capture records the
// launches without running them, so solve_begin takes them all outside the caller's loop.
cudaGraphExec_t Engine::chunk_graph(int len) {
    const std::string key = std::string(solve_fused ? "F" : solve_flood ? "f" : "o") +
                            std::to_string(solve_stop) + ":" +
                            std::to_string((long long)(uintptr_t)solve_b) + ":" +
                            std::to_string((long long)(uintptr_t)solve_levels) + ":" + std::to_string(len);
    auto it = graphs.find(key);
    if (it == graphs.end()) {
        cudaGraph_t g;
        ck(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal), "capture");
        for (int k = 0; k < len; ++k) enqueue_step();
        ck(cudaStreamEndCapture(st, &g), "capture end");
        cudaGraphExec_t ge;
        ck(cudaGraphInstantiate(&ge, g, 0), "graph instantiate");
        cudaGraphDestroy(g);
        ck(cudaGraphUpload(ge, st), "graph upload");  // the first launch then pays no upload
        it = graphs.emplace(key, ge).first;
    }
    return it->second;
}

void Engine::solve_steps(int nsteps) {
    if (nsteps <= 0) return;
    if (solve_pipe) {  // one launch carries all of them, pipelined (seqpipe_kernels.cuh)
        const int k = std::min(nsteps, solve_max_iter - pipe_next + 1);
        if (k > 0) launch_pipe(solve_b, d_xring, pipe_next, k, true, solve_stop == BGABP_STOP_MESSAGE_DELTA);
        pipe_next += std::max(k, 0);
        steps_enqueued += nsteps;
        return;
    }
    // graph-replay chunks of iterations: the kernels read their step index from the device,
    // so one captured chunk is valid for any position in the loop
    const bool use_graph = chunk_graph_eligible();
    int left = nsteps;
    while (left > 0) {
        // kChunk-iteration graphs, then the remainder as power-of-two graphs (16 + 4 for 20)
        int chunk = left;
        if (use_graph) {
            chunk = kChunk;
            while (chunk > left) chunk >>= 1;
        }
        if (use_graph) {
            ck(cudaGraphLaunch(chunk_graph(chunk), st), "graph launch");
        } else {
            for (int k = 0; k < chunk; ++k) enqueue_step();
        }
        left -= chunk;
        steps_enqueued += chunk;
    }
    ck(cudaGetLastError(), "solve steps");
}

bool Engine::solve_done() {
    read_ctrl();
    return h_ctrl->done != 0;
}

void Engine::solve_run_to_end() {
    // Enqueue growing chunks until the device has decided (at most max_iter + 2 iterations).
    // Two chunks stay queued: the host reads chunk k's stop flag (a 4-byte copy behind it) while
    // chunk k+1 runs, so the GPU never idles on the poll.
    if (!h_poll) {
        ck(cudaMallocHost((void**)&h_poll, 2 * sizeof(int)), "cudaMallocHost");
        for (auto& e : poll_ev) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
    }
    read_ctrl();
    if (h_ctrl->done) return;
    const long long total = (long long)solve_max_iter + (solve_fused ? 2 : 1);
    // The pipelined sequential solve fills and drains its wavefront once per launch (~7 ms at
    // 2048^2), while the sweeps of a launch that start after the decision exit at their gate
    // check: it runs kPipeChunk sweeps per launch from the start.
    const int cap = solve_pipe ? kPipeChunk : 512;
    int chunk = solve_pipe ? kPipeChunk : 16, inflight = 0, oldest = 0;
    while (true) {
        while (inflight < 2 && steps_enqueued < total) {
            solve_steps((int)std::min<long long>(chunk, total - steps_enqueued));
            const int sl = (oldest + inflight) & 1;
            ck(cudaMemcpyAsync(&h_poll[sl], &d_ctrl->done, sizeof(int), cudaMemcpyDeviceToHost, st), "poll");
            ck(cudaEventRecord(poll_ev[sl], st), "event");
            ++inflight;
            chunk = std::min(chunk * 2, cap);
        }
        if (inflight == 0) throw CudaError("solve loop did not terminate");
        ck(cudaEventSynchronize(poll_ev[oldest]), "poll sync");
        --inflight;
        if (h_poll[oldest]) {
            ck(cudaStreamSynchronize(st), "sync");
            return;
        }
        oldest ^= 1;
    }
}

void Engine::solve_report(bgabp_report& rep, std::string& detail) {
    if (solve_rb) {  // the handle's state stays in the natural layout between calls
        rb_state(false, d_msg[0]);
        cur = 0;
    }
    read_ctrl();
    const Ctrl& c = *h_ctrl;
    rep.status = c.status;
    rep.iterations = c.iterations;
    detail.clear();
    bool pivot = false;
    if (c.status == BGABP_DIVERGED) {
        switch (c.detail_kind) {
            case 1: detail = "zero pivot at node " + std::to_string(c.detail_key); pivot = true; break;
            case 2:
                detail = "zero pivot on edge " + std::to_string(c.detail_key >> 32) + "->" +
                         std::to_string(c.detail_key & 0xffffffffu);
                pivot = true;
                break;
            case 3: detail = "residual blowup"; break;
            case 5: detail = "peer shard timeout"; break;
            case 4: detail = ordered_detail(solve_levels->order, c.detail_key); pivot = true; break;
        }
    }
    const double per_iter = sweep_flops() + 2.0 * (double)nnz;  // gabp.cpp:200-202
    rep.flop_estimate = 0.0;
    for (int k = 0; k < c.iterations - (pivot ? 1 : 0); ++k) rep.flop_estimate += per_iter;
}

const double* Engine::solve_x() {
    if (solve_pipe) {
        const Ctrl& c = *h_ctrl;  // read by solve_report
        if (n == 0) return d_aux;
        const int xs = c.solx % kPipeR;
        if (c.status == BGABP_DIVERGED && c.detail_kind == 4) {
            // the reference's sweep stopped at visit position p: x(k) before it (and at it for an
            // edge pivot, whose x-stage ran), x(k-1) from there on; positions are node ids here
            const long long p = (long long)(c.detail_key >> 32) + ((c.detail_key & 0xffffffffu) ? 1 : 0);
            return pipe_x_out(xs, (c.solx + kPipeR - 1) % kPipeR, p);
        }
        return pipe_x_out(xs, xs, (long long)n);
    }
    if (!solve_fused && solve_flood) {  // union-CSR flood: x(k) in slot k & 1 of d_xord
        const Ctrl& c = *h_ctrl;
        if (c.status == BGABP_DIVERGED && c.detail_kind == 2)  // failed edge stage: x of the sweep before
            return d_xord + (size_t)((c.iterations + 1) & 1) * n;
        const double* xs = d_xord + (size_t)(c.iterations & 1) * n;
        if (c.status == BGABP_DIVERGED && c.detail_kind == 1 && n > 0) {  // x-stage stopped at the pivot node
            k_compose_pivot_x<<<nblk(n), 256, 0, st>>>(xs, d_xord + (size_t)((c.iterations + 1) & 1) * n, d_aux, n,
                                                       (long long)c.detail_key);
            ck(cudaGetLastError(), "compose x");
            return d_aux;
        }
        return xs;
    }
    if (!solve_fused) {  // ordered (levels / red-black): x(k) in slot k & 1 of d_xord
        const Ctrl& c = *h_ctrl;  // read by solve_report
        const double* xs = d_xord + (size_t)(c.iterations & 1) * n;
        if (c.status == BGABP_DIVERGED && c.detail_kind == 4 && n > 0 && solve_levels) {
            // the reference's sweep stopped at visit position p (gabp.cpp:71-87): nodes visited
            // before it (and the pivot node itself on an edge pivot, whose x-stage ran) hold x(k),
            // the rest x(k-1)
            const double* xo = d_xord + (size_t)((c.iterations + 1) & 1) * n;
            std::vector<int> pos(n);
            for (int q = 0; q < n; ++q) pos[solve_levels->order[q]] = q;
            int* dpos = static_cast<int*>(dalloc(sizeof(int) * (size_t)n));
            ck(cudaMemcpyAsync(dpos, pos.data(), sizeof(int) * (size_t)n, cudaMemcpyHostToDevice, st), "H2D");
            const long long p = (long long)(c.detail_key >> 32) + ((c.detail_key & 0xffffffffu) ? 1 : 0);
            k_compose_pos_x<<<nblk(n), 256, 0, st>>>(xs, xo, dpos, d_aux, n, p);
            ck(cudaGetLastError(), "compose x");
            ck(cudaStreamSynchronize(st), "sync");
            dfree(dpos);
            return d_aux;
        }
        return xs;
    }
    const Ctrl& c = *h_ctrl;  // read by solve_report
    const int ring = kXRing;
    const double* xs = d_xf + (size_t)(c.solx & (ring - 1)) * n;
    if (c.status == BGABP_DIVERGED && c.detail_kind == 1 && n > 0) {
        // the reference stops its x-stage at the pivot node: x(k) below it, x(k-1) from it on
        const double* xo = d_xf + (size_t)((c.solx - 1) & (ring - 1)) * n;
        k_compose_pivot_x<<<nblk(n), 256, 0, st>>>(xs, xo, d_aux, n, (long long)c.detail_key - dia.gofs);
        ck(cudaGetLastError(), "compose x");
        return d_aux;
    }
    return xs;
}

double Engine::sweep_flops() const {  // gabp.cpp:165-172
    const double e = (double)num_edges;
    return n + 3.0 * e + 4.0 * e;
}

// ---------------------------------------------------------------------------------------------
// frozen-precision path (gabp.cpp:221-401)
// ---------------------------------------------------------------------------------------------
void Engine::ensure_frozen_buffers() {
    if (d_lam) return;
    const size_t sb = sizeof(double) * (size_t)std::max<long long>(nslots, 1);
    d_lam = static_cast<double*>(dalloc(sb));
    d_lsrc = static_cast<double*>(dalloc(sb));
    d_sigma = static_cast<double*>(dalloc(sizeof(double) * std::max(n, 1)));
}

void Engine::frozen_finish() {  // sigma and the source-major lambda copy from d_lam
    if (n == 0) return;
    const unsigned g = nblk(n);
    if (layout == BGABP_LAYOUT_DIA) {
        DIA_SWITCH(S, k_sigma_dia<SS><<<g, 256, 0, st>>>(dia, d_lam, d_sigma);
                   k_lambda_by_source_dia<SS><<<g, 256, 0, st>>>(dia, d_lam, d_lsrc));
    } else {
        k_sigma_csr<<<g, 256, 0, st>>>(csr, d_lam, d_sigma);
        k_lambda_by_source_csr<<<g, 256, 0, st>>>(csr, d_lam, d_lsrc);
    }
    has_frozen = true;
}

void Engine::precompute_lambda(const bgabp_schedule& s, double tol, int max_iter, int& converged, int& iters) {
    const bool flood = s.kind == BGABP_SCHED_FLOOD;
    const Levels* L = flood ? nullptr : &levels_for(s);
    ensure_frozen_buffers();
    const size_t sb = sizeof(double) * (size_t)std::max<long long>(nslots, 1);
    double* lb[2] = {d_lam, reinterpret_cast<double*>(d_msg[0])};  // flood ping-pong scratch
    ck(cudaMemsetAsync(lb[0], 0, sb, st), "memset");
    ck(cudaMemsetAsync(lb[1], 0, sb, st), "memset");
    converged = 0;
    iters = 0;
    int curb = 0;
    const unsigned g = nblk(n);
    for (int it = 1; it <= max_iter; ++it) {
        reset_ctrl();
        unsigned long long* ds = &d_ctrl->red[1];
        if (n > 0) {
            if (flood) {
                if (layout == BGABP_LAYOUT_DIA) {
                    DIA_SWITCH(S, k_lambda_flood_dia<SS><<<g, 256, 0, st>>>(dia, lb[curb], lb[curb ^ 1], d_ctrl, ds));
                } else {
                    k_lambda_flood_csr<<<g, 256, 0, st>>>(csr, lb[curb], lb[curb ^ 1], d_ctrl, ds);
                }
                curb ^= 1;
            } else {
                for (size_t l = 0; l + 1 < L->ptr.size(); ++l) {
                    const int cnt = L->ptr[l + 1] - L->ptr[l];
                    const int* nodes = L->d_nodes + L->ptr[l];
                    if (layout == BGABP_LAYOUT_DIA) {
                        DIA_SWITCH(S, k_lambda_level_dia<SS><<<nblk(cnt), 256, 0, st>>>(dia, lb[0], nodes, cnt, d_ctrl, ds));
                    } else {
                        k_lambda_level_csr<<<nblk(cnt), 256, 0, st>>>(csr, lb[0], nodes, cnt, d_ctrl, ds);
                    }
                }
            }
        }
        ck(cudaGetLastError(), "lambda sweep");
        read_ctrl();
        iters = it;
        if (h_ctrl->opiv != kNone) {  // breakdown: not converged, no sigma (gabp.cpp:238-243)
            if (curb) ck(cudaMemcpyAsync(d_lam, lb[1], sb, cudaMemcpyDeviceToDevice, st), "copy");
            ck(cudaMemsetAsync(d_sigma, 0, sizeof(double) * std::max(n, 1), st), "memset");
            converged = 0;
            has_frozen = false;
            cudaMemsetAsync(d_msg[0], 0, sb, st);
            return;
        }
        const double delta = bits2d(h_ctrl->red[1]);
        if (delta <= tol) {
            converged = 1;
            break;
        }
        if (!std::isfinite(delta)) break;
    }
    if (curb) ck(cudaMemcpyAsync(d_lam, lb[1], sb, cudaMemcpyDeviceToDevice, st), "copy");
    ck(cudaMemsetAsync(d_msg[0], 0, sizeof(double2) * (size_t)std::max<long long>(nslots, 1), st), "memset");
    frozen_finish();
    ck(cudaStreamSynchronize(st), "sync");
}

void Engine::correction_sweeps_dev(const double* r_dev, const bgabp_schedule& s, int sweeps, double* e_dev) {
    // mean-only sweeps (gabp.cpp:289-325), cold messages, frozen lambda/sigma on the device
    const bool flood = s.kind == BGABP_SCHED_FLOOD;
    const Levels* L = flood ? nullptr : &levels_for(s);
    const size_t sb = sizeof(double) * (size_t)std::max<long long>(nslots, 1);
    double* mb[2] = {reinterpret_cast<double*>(d_msg[0]), reinterpret_cast<double*>(d_msg[1])};
    ck(cudaMemsetAsync(mb[0], 0, sb, st), "memset");
    ck(cudaMemsetAsync(e_dev, 0, sizeof(double) * std::max(n, 1), st), "memset");
    if (n == 0) return;
    const unsigned g = nblk(n);
    int curb = 0;
    for (int k = 0; k < sweeps; ++k) {
        if (flood) {
            if (layout == BGABP_LAYOUT_DIA) {
                DIA_SWITCH(S, k_corr_flood_dia<SS><<<g, 256, 0, st>>>(dia, r_dev, d_lsrc, mb[curb], mb[curb ^ 1]));
            } else {
                k_corr_flood_csr<<<g, 256, 0, st>>>(csr, r_dev, d_lsrc, mb[curb], mb[curb ^ 1]);
            }
            curb ^= 1;
        } else {
            for (size_t l = 0; l + 1 < L->ptr.size(); ++l) {
                const int cnt = L->ptr[l + 1] - L->ptr[l];
                const int* nodes = L->d_nodes + L->ptr[l];
                if (layout == BGABP_LAYOUT_DIA) {
                    DIA_SWITCH(S, k_corr_level_dia<SS><<<nblk(cnt), 256, 0, st>>>(dia, r_dev, d_lsrc, d_sigma, mb[0], e_dev, nodes, cnt));
                } else {
                    k_corr_level_csr<<<nblk(cnt), 256, 0, st>>>(csr, r_dev, d_lsrc, d_sigma, mb[0], e_dev, nodes, cnt);
                }
            }
        }
    }
    if (flood) {
        if (layout == BGABP_LAYOUT_DIA) {
            DIA_SWITCH(S, k_corr_final_dia<SS><<<g, 256, 0, st>>>(dia, r_dev, d_sigma, mb[curb], e_dev));
        } else {
            k_corr_final_csr<<<g, 256, 0, st>>>(csr, r_dev, d_sigma, mb[curb], e_dev);
        }
    }
    ck(cudaGetLastError(), "correction sweeps");
}

// cold sweeps on A e = r from zero messages (gabp.cpp:343-361, multigrid.cpp:180-187).  Failures
// are promoted on the device (k_plain_check) so a multigrid cycle never synchronises; with
// check=true the call synchronises and returns BGABP_EPIVOT with the reference's message.
int Engine::cold_sweeps_dev(const double* r_dev, const bgabp_schedule& s, int sweeps, double* e_dev,
                            std::string& err, bool check, int seq) {
    const bool flood = s.kind == BGABP_SCHED_FLOOD;
    const bool rbp = rb_applicable(s) && n > 0 && sweeps > 0;
    const Levels* L = (flood || (rbp && !check)) ? nullptr : &levels_for(s);
    if (check) reset_ctrl();
    k_plain_reset<<<1, 1, 0, st>>>(d_ctrl);
    if (rbp) {
        // colour-compact red-black: the cold first red phase reads no message, every later read
        // slot has been written by then, and every sweep writes all of e -- nothing to clear
        rb_build(s.nx);
        for (int k = 0; k < sweeps; ++k) launch_rb_sweep(r_dev, e_dev, k == 0, false, nullptr, MODE_PLAIN);
    } else {
        if (!seq_applicable(s))  // the pipeline zeroes its own (lane-skewed) messages
            for (int k = 0; k < 2; ++k)
                ck(cudaMemsetAsync(d_msg[k], 0, sizeof(double2) * (size_t)std::max<long long>(nslots, 1), st), "memset");
        ck(cudaMemsetAsync(e_dev, 0, sizeof(double) * std::max(n, 1), st), "memset");
        cur = 0;
        if (n == 0 || sweeps <= 0) return BGABP_OK;
        if (flood) {
            for (int k = 0; k < sweeps; ++k) {
                launch_flood(r_dev, d_msg[cur], d_msg[cur ^ 1], nullptr, k == 0 ? MODE_PLAIN : MODE_PLAIN_X, false);
                cur ^= 1;
                k_plain_check<<<1, 1, 0, st>>>(d_ctrl, seq, 4);
            }
            launch_aggregate(r_dev, d_msg[cur], e_dev, nullptr, &d_ctrl->npiv[0]);
        } else if (seq_applicable(s)) {  // all sweeps in one pipelined launch, e = x of the last
            pipe_setup(false);
            pipe_reset();
            launch_pipe(r_dev, e_dev, 1, sweeps, false, false);
        } else {
            for (int k = 0; k < sweeps; ++k) launch_levels(*L, r_dev, d_msg[cur], e_dev, false, nullptr, MODE_PLAIN);
        }
    }
    k_plain_check<<<1, 1, 0, st>>>(d_ctrl, seq, 4);
    ck(cudaGetLastError(), "cold sweeps");
    if (!check) return BGABP_OK;
    read_ctrl();
    if (h_ctrl->halt) {
        err = decode_failure(*h_ctrl, L ? &L->order : nullptr);
        return BGABP_EPIVOT;
    }
    return BGABP_OK;
}

// sweeps_expand (multigrid.cpp:54-70): 30 cold sweeps on r = 1; expand if any sweep breaks down,
// if max|m| is non-finite after any sweep, or if it grows more than 6.19x from sweep 20 to 30.
bool Engine::sweeps_expand(const bgabp_schedule& s) {
    if (n == 0) return false;
    const bool timing = getenv("BGABP_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* what) {
        if (!timing) return;
        ck(cudaStreamSynchronize(st), "sync");
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[probe] n=%d %-18s %8.2f ms\n", n, what,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    const bool flood = s.kind == BGABP_SCHED_FLOOD;
    const bool rbp = rb_applicable(s);
    if (rbp) rb_build(s.nx);
    phase("layout");
    const Levels* L = (flood || rbp) ? nullptr : &levels_for(s);
    unsigned long long* d_norms = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long) * 32));
    ck(cudaMemsetAsync(d_norms, 0, sizeof(unsigned long long) * 32, st), "memset");
    double* d_ones = static_cast<double*>(dalloc(sizeof(double) * (size_t)n));
    k_fill_value<<<std::min<unsigned>(nblk(n), 148u * 8u), 256, 0, st>>>(d_ones, n, 1.0);
    reset_ctrl();
    for (int k = 0; k < 2; ++k)
        ck(cudaMemsetAsync(d_msg[k], 0, sizeof(double2) * (size_t)std::max<long long>(nslots, 1), st), "memset");
    ck(cudaMemsetAsync(d_e, 0, sizeof(double) * n, st), "memset");
    cur = 0;
    const unsigned gr = std::min<unsigned>(nblk(nslots), 1184);
    phase("buffers");
    for (int k = 0; k < 30; ++k) {
        if (flood) {
            launch_flood(d_ones, d_msg[cur], d_msg[cur ^ 1], nullptr, k == 0 ? MODE_PLAIN : MODE_PLAIN_X, false);
            cur ^= 1;
        } else if (rbp) {  // colour-compact: max |m| over the same values, permuted
            launch_rb_sweep(d_ones, d_e, k == 0, false, nullptr, MODE_PLAIN);
        } else {
            launch_levels(*L, d_ones, d_msg[cur], d_e, false, nullptr, MODE_PLAIN);
        }
        k_plain_check<<<1, 1, 0, st>>>(d_ctrl, k, 4);
        if (flood) {  // the x-stage of this sweep belongs to this sweep (gabp.cpp:141-160)
            launch_aggregate(d_ones, d_msg[cur], d_e, nullptr, &d_ctrl->npiv[0]);
            k_plain_check<<<1, 1, 0, st>>>(d_ctrl, k, 4);
        }
        k_max_abs_m<<<gr, 256, 0, st>>>(rbp ? d_rbmsg : d_msg[cur], nslots, d_norms + k);
    }
    ck(cudaGetLastError(), "probe");
    phase("30 sweeps");
    unsigned long long hn[32];
    ck(cudaMemcpyAsync(hn, d_norms, sizeof(hn), cudaMemcpyDeviceToHost, st), "D2H");
    read_ctrl();
    for (int k = 0; k < 2; ++k)
        ck(cudaMemsetAsync(d_msg[k], 0, sizeof(double2) * (size_t)std::max<long long>(nslots, 1), st), "memset");
    ck(cudaStreamSynchronize(st), "sync");
    dfree(d_ones);
    dfree(d_norms);
    phase("read back");
    if (h_ctrl->halt) return true;
    for (int k = 0; k < 30; ++k)
        if (!std::isfinite(bits2d(hn[k]))) return true;
    const double mid = bits2d(hn[19]), end = bits2d(hn[29]);
    return mid > 0.0 && end > 6.19 * mid;
}

std::string Engine::decode_failure(const Ctrl& c, const std::vector<int>* order) const {
    switch (c.detail_kind) {
        case 1: return "zero pivot at node " + std::to_string(c.detail_key);
        case 2:
            return "zero pivot on edge " + std::to_string(c.detail_key >> 32) + "->" +
                   std::to_string(c.detail_key & 0xffffffffu);
        case 3: return "residual blowup";
        case 4: return order ? ordered_detail(*order, c.detail_key) : "zero pivot";
        case 5: {  // relax: gs_pass / jacobi_pass (classic.cpp:27,43)
            const int pos = (int)(c.detail_key >> 32);
            return "relax: zero diagonal at " + std::to_string(order ? (*order)[pos] : pos);
        }
    }
    return "breakdown";
}

}  // namespace bgabp

// =============================================================================================
// C-ABI
// =============================================================================================
using namespace bgabp;

extern "C" {

const char* bgabp_version(void) { return kVersion; }

int bgabp_create(int n, const int* row_offsets, const int* col_indices, const double* values, int layout,
                 bgabp_engine** out, char* err, size_t errlen) {
    *out = nullptr;
    auto h = std::make_unique<bgabp_engine>();
    ABI_GUARD(err, errlen, {
        h->E.build(n, row_offsets, col_indices, values, layout);
        *out = h.release();
        return BGABP_OK;
    })
}

void bgabp_destroy(bgabp_engine* e) { delete e; }

int bgabp_get_info(const bgabp_engine* h, bgabp_info* info) {
    const Engine& E = h->E;
    info->n = E.n;
    info->nnz = E.nnz;
    info->num_edges = E.num_edges;
    info->layout = E.layout;
    info->num_slots = E.S;
    info->symmetric_values = E.symmetric ? 1 : 0;
    info->bytes_per_sweep = 40.0 * (double)E.num_edges + 24.0 * E.n;
    info->uniform_coefficients = (E.layout == BGABP_LAYOUT_DIA && E.dia.uniform) ? 1 : 0;
    info->bytes_per_residual = 8.0 * (double)E.nnz + 16.0 * E.n;
    info->device_bytes = E.device_bytes;
    info->sell_slots = E.sell_slots;
    return BGABP_OK;
}

// FNV-1a over the device layout and the facts derived from it (diagnostic: the device and the
// host build of the same matrix must agree bit for bit)
int bgabp_layout_digest(bgabp_engine* h, unsigned long long* out) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        unsigned long long f = 1469598103934665603ull;
        auto mix = [&](const void* p, size_t bytes) {
            const unsigned char* c = static_cast<const unsigned char*>(p);
            for (size_t i = 0; i < bytes; ++i) f = (f ^ c[i]) * 1099511628211ull;
        };
        auto mix_dev = [&](const void* d, size_t bytes) {
            std::vector<unsigned char> t(bytes);
            if (bytes) ck(cudaMemcpy(t.data(), d, bytes, cudaMemcpyDeviceToHost), "D2H");
            mix(t.data(), bytes);
        };
        const int flags[6] = {E.layout, E.S, E.symmetric ? 1 : 0, E.grid5 ? 1 : 0, E.grid5 ? E.grid5_nx : 0,
                              E.layout == BGABP_LAYOUT_DIA ? E.dia.uniform : 0};
        mix(flags, sizeof flags);
        ck(cudaStreamSynchronize(E.st), "sync");
        if (E.layout == BGABP_LAYOUT_DIA) {
            mix(E.dia.off, sizeof(int) * E.S);
            mix(E.dia.rev, sizeof(int) * E.S);
            if (E.dia.uniform) {
                mix(E.dia.cu, sizeof(double) * E.S);
                mix(&E.dia.du, sizeof(double));
            }
            mix_dev(E.dia.mask, sizeof(uint32_t) * (size_t)E.n);
            mix_dev(E.dia.c, sizeof(double) * (size_t)E.nslots);
            mix_dev(E.dia.rowv, sizeof(double) * (size_t)E.nslots);
            mix_dev(E.dia.diag, sizeof(double) * (size_t)E.n);
        }
        E.ensure_csr2slot();
        ck(cudaStreamSynchronize(E.st), "sync");  // built on the handle's (non-blocking) stream
        mix_dev(E.d_csr2slot, sizeof(long long) * (size_t)E.nnz);
        *out = f;
        return BGABP_OK;
    })
}

void* bgabp_stream(bgabp_engine* h) { return (void*)h->E.st; }

int bgabp_reset_state(bgabp_engine* h) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        for (int k = 0; k < 2; ++k)
            ck(cudaMemsetAsync(E.d_msg[k], 0, sizeof(double2) * (size_t)std::max<long long>(E.nslots, 1), E.st), "memset");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_set_state(bgabp_engine* h, const double* lam, const double* m) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (E.nnz == 0) return BGABP_OK;
        double *dl = nullptr, *dm = nullptr;
        ck(cudaMallocAsync((void**)&dl, sizeof(double) * E.nnz, E.st), "malloc");
        ck(cudaMallocAsync((void**)&dm, sizeof(double) * E.nnz, E.st), "malloc");
        ck(cudaMemcpyAsync(dl, lam, sizeof(double) * E.nnz, cudaMemcpyHostToDevice, E.st), "H2D");
        ck(cudaMemcpyAsync(dm, m, sizeof(double) * E.nnz, cudaMemcpyHostToDevice, E.st), "H2D");
        ck(cudaMemsetAsync(E.d_msg[E.cur], 0, sizeof(double2) * (size_t)E.nslots, E.st), "memset");
        E.ensure_csr2slot();
        k_state_scatter<<<nblk(E.nnz), 256, 0, E.st>>>(E.d_msg[E.cur], E.d_csr2slot, E.nnz, dl, dm);
        ck(cudaFreeAsync(dl, E.st), "free");
        ck(cudaFreeAsync(dm, E.st), "free");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_get_state(bgabp_engine* h, double* lam, double* m) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (E.nnz == 0) return BGABP_OK;
        double *dl = nullptr, *dm = nullptr;
        ck(cudaMallocAsync((void**)&dl, sizeof(double) * E.nnz, E.st), "malloc");
        ck(cudaMallocAsync((void**)&dm, sizeof(double) * E.nnz, E.st), "malloc");
        E.ensure_csr2slot();
        k_state_gather<<<nblk(E.nnz), 256, 0, E.st>>>(E.d_msg[E.cur], E.d_csr2slot, E.nnz, dl, dm);
        ck(cudaMemcpyAsync(lam, dl, sizeof(double) * E.nnz, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaMemcpyAsync(m, dm, sizeof(double) * E.nnz, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaFreeAsync(dl, E.st), "free");
        ck(cudaFreeAsync(dm, E.st), "free");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_sweep(bgabp_engine* h, const double* b, const bgabp_schedule* s, double* x, char* err, size_t errlen) {
    ABI_GUARD(err, errlen, {
        std::string msg;
        int rc = h->E.sweep(b, *s, x, msg);
        if (rc != BGABP_OK) put_err(err, errlen, msg);
        return rc;
    })
}

int bgabp_node_precisions(bgabp_engine* h, double* beta) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (E.n == 0) return BGABP_OK;
        E.launch_aggregate(nullptr, E.d_msg[E.cur], nullptr, E.d_aux, nullptr);
        ck(cudaMemcpyAsync(beta, E.d_aux, sizeof(double) * E.n, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

double bgabp_sweep_flops(const bgabp_engine* h) { return h->E.sweep_flops(); }

int bgabp_set_damping(bgabp_engine* h, double alpha) {
    ABI_GUARD(nullptr, 0, {
        h->E.set_damping(alpha);
        return BGABP_OK;
    })
}

int bgabp_solve(bgabp_engine* h, const double* b, const bgabp_schedule* s, const bgabp_options* opt,
                bgabp_report* rep, double* x_out, double* history, char* detail, size_t dl) {
    ABI_GUARD(detail, dl, {
        Engine& E = h->E;
        E.schedule_order_check(*s);
        host_to_device(E.d_b, b, sizeof(double) * E.n, E.st);
        E.solve_begin(E.d_b, *s, *opt);
        E.solve_run_to_end();
        std::string d;
        E.solve_report(*rep, d);
        if (x_out && E.n > 0) device_to_host(x_out, E.solve_x(), sizeof(double) * E.n, E.st);
        if (history)
            ck(cudaMemcpyAsync(history, E.d_hist, sizeof(double) * (rep->iterations + 1), cudaMemcpyDeviceToHost, E.st),
               "D2H hist");
        ck(cudaStreamSynchronize(E.st), "sync");
        put_err(detail, dl, d);
        return BGABP_OK;
    })
}

int bgabp_solve_device_begin(bgabp_engine* h, const double* b_dev, const bgabp_schedule* s, const bgabp_options* opt) {
    ABI_GUARD(nullptr, 0, {
        h->E.schedule_order_check(*s);
        h->E.solve_begin(b_dev, *s, *opt);
        return BGABP_OK;
    })
}

int bgabp_solve_device_steps(bgabp_engine* h, int nsteps) {
    ABI_GUARD(nullptr, 0, {
        h->E.solve_steps(nsteps);
        return BGABP_OK;
    })
}

int bgabp_solve_device_end(bgabp_engine* h, bgabp_report* rep, double* x_dev, double* history_dev, char* detail,
                           size_t dl) {
    ABI_GUARD(detail, dl, {
        Engine& E = h->E;
        std::string d;
        E.solve_report(*rep, d);
        if (x_dev && E.n > 0)
            ck(cudaMemcpyAsync(x_dev, E.solve_x(), sizeof(double) * E.n, cudaMemcpyDeviceToDevice, E.st), "D2D x");
        if (history_dev)
            ck(cudaMemcpyAsync(history_dev, E.d_hist, sizeof(double) * (rep->iterations + 1), cudaMemcpyDeviceToDevice,
                               E.st),
               "D2D hist");
        ck(cudaStreamSynchronize(E.st), "sync");
        put_err(detail, dl, d);
        return BGABP_OK;
    })
}

int bgabp_solve_device_steps_timed(bgabp_engine* h, int nsteps, double* hot_ms) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        const int launches = nsteps;  // one event pair per launch
        std::vector<cudaEvent_t> ev(2 * (size_t)std::max(launches, 0));
        for (auto& e : ev) ck(cudaEventCreate(&e), "event");
        E.timed_events = &ev;
        for (int k = 0; k < launches; ++k) {
            E.timed_index = k;
            E.enqueue_step();
        }
        E.timed_events = nullptr;
        ck(cudaGetLastError(), "timed steps");
        ck(cudaStreamSynchronize(E.st), "sync");
        double total = 0.0;
        for (int k = 0; k < launches; ++k) {
            float ms = 0.f;
            ck(cudaEventElapsedTime(&ms, ev[2 * k], ev[2 * k + 1]), "elapsed");
            total += ms;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        E.steps_enqueued += launches;
        *hot_ms = total;
        return BGABP_OK;
    })
}

int bgabp_flood_sweeps_device(bgabp_engine* h, const double* b_dev, int nsweeps) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        for (int k = 0; k < nsweeps; ++k) {
            E.launch_flood(b_dev, E.d_msg[E.cur], E.d_msg[E.cur ^ 1], E.d_x, MODE_PLAIN, false);
            E.cur ^= 1;
        }
        ck(cudaGetLastError(), "flood sweeps");
        return BGABP_OK;
    })
}

int bgabp_residual_inf_norm(bgabp_engine* h, const double* x, const double* b, double* out) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        *out = 0.0;
        if (E.n == 0) return BGABP_OK;
        E.reset_ctrl();
        ck(cudaMemcpyAsync(E.d_b, b, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        ck(cudaMemcpyAsync(E.d_aux, x, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        E.launch_residual(E.d_b, E.d_aux, nullptr, &E.d_ctrl->red[2], MODE_PLAIN);
        E.read_ctrl();
        *out = bits2d(E.h_ctrl->red[2]);
        return BGABP_OK;
    })
}

int bgabp_precompute_lambda(bgabp_engine* h, const bgabp_schedule* s, double tol, int max_iter, double* lam_out,
                            double* sigma_out, int* converged, int* iterations) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        int cv = 0, it = 0;
        E.precompute_lambda(*s, tol, max_iter, cv, it);
        if (converged) *converged = cv;
        if (iterations) *iterations = it;
        if (lam_out && E.nnz > 0) {
            double* dl = nullptr;
            ck(cudaMallocAsync((void**)&dl, sizeof(double) * E.nnz, E.st), "malloc");
            E.ensure_csr2slot();
            k_lambda_gather<<<nblk(E.nnz), 256, 0, E.st>>>(E.d_lam, E.d_csr2slot, E.nnz, dl);
            ck(cudaMemcpyAsync(lam_out, dl, sizeof(double) * E.nnz, cudaMemcpyDeviceToHost, E.st), "D2H");
            ck(cudaFreeAsync(dl, E.st), "free");
        }
        if (sigma_out && E.n > 0)
            ck(cudaMemcpyAsync(sigma_out, E.d_sigma, sizeof(double) * E.n, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_set_frozen(bgabp_engine* h, const double* lam, const double* sigma) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        E.ensure_frozen_buffers();
        ck(cudaMemsetAsync(E.d_lam, 0, sizeof(double) * (size_t)std::max<long long>(E.nslots, 1), E.st), "memset");
        if (E.nnz > 0) {
            double* dl = nullptr;
            ck(cudaMallocAsync((void**)&dl, sizeof(double) * E.nnz, E.st), "malloc");
            ck(cudaMemcpyAsync(dl, lam, sizeof(double) * E.nnz, cudaMemcpyHostToDevice, E.st), "H2D");
            E.ensure_csr2slot();
            k_lambda_scatter<<<nblk(E.nnz), 256, 0, E.st>>>(E.d_lam, E.d_csr2slot, E.nnz, dl);
            ck(cudaFreeAsync(dl, E.st), "free");
        }
        E.frozen_finish();
        if (E.n > 0)  // the caller's sigma wins over the recomputed one (FrozenLambda carries both)
            ck(cudaMemcpyAsync(E.d_sigma, sigma, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_correction_sweeps(bgabp_engine* h, const double* r, const bgabp_schedule* s, int sweeps, double* e_out) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        E.schedule_order_check(*s);
        if (!E.has_frozen) throw InvalidArg("gabp: no frozen precisions (call precompute_lambda or set_frozen)");
        if (E.n == 0) return BGABP_OK;
        ck(cudaMemcpyAsync(E.d_r, r, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        E.correction_sweeps_dev(E.d_r, *s, sweeps, E.d_e);
        ck(cudaMemcpyAsync(e_out, E.d_e, sizeof(double) * E.n, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

int bgabp_error_correction_apply(bgabp_engine* h, const double* b, const double* x0, int sweeps,
                                 const bgabp_schedule* s, int use_frozen, double* x_out, char* err, size_t errlen) {
    ABI_GUARD(err, errlen, {
        Engine& E = h->E;
        E.schedule_order_check(*s);
        if (use_frozen && !E.has_frozen) throw InvalidArg("gabp: no frozen precisions");
        if (E.n == 0) return BGABP_OK;
        ck(cudaMemcpyAsync(E.d_b, b, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        ck(cudaMemcpyAsync(E.d_aux, x0, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
        E.launch_residual(E.d_b, E.d_aux, E.d_r, nullptr, MODE_PLAIN);  // gabp.cpp:327-335
        if (use_frozen) {
            E.correction_sweeps_dev(E.d_r, *s, sweeps, E.d_e);
        } else {
            std::string msg;
            if (E.cold_sweeps_dev(E.d_r, *s, sweeps, E.d_e, msg, true) != BGABP_OK)
                throw std::runtime_error("gabp error correction: " + msg);
        }
        k_axpy1<<<nblk(E.n), 256, 0, E.st>>>(E.d_aux, E.d_e, E.n);
        ck(cudaMemcpyAsync(x_out, E.d_aux, sizeof(double) * E.n, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaStreamSynchronize(E.st), "sync");
        return BGABP_OK;
    })
}

// gabp.cpp:363-401; the outer loop stays on the host (one residual read per iteration)
int bgabp_solve_error_correction(bgabp_engine* h, const double* b, const bgabp_schedule* s, int sweeps,
                                 const bgabp_options* o, bgabp_report* rep, double* x_out, double* history,
                                 char* detail, size_t dl) {
    ABI_GUARD(detail, dl, {
        Engine& E = h->E;
        E.schedule_order_check(*s);
        if (!E.has_frozen) throw InvalidArg("gabp: no frozen precisions");
        std::vector<double> hist;
        double r0 = 0.0;
        for (int i = 0; i < E.n; ++i) r0 = std::max(r0, std::abs(b[i]));
        hist.push_back(r0);
        rep->status = BGABP_MAX_ITER;
        rep->iterations = 0;
        rep->flop_estimate = 0.0;
        std::string d;
        if (E.n > 0) {
            ck(cudaMemcpyAsync(E.d_b, b, sizeof(double) * E.n, cudaMemcpyHostToDevice, E.st), "H2D");
            ck(cudaMemsetAsync(E.d_aux, 0, sizeof(double) * E.n, E.st), "memset");
        }
        const double ee = (double)E.num_edges;
        const double per_iter = 2.0 * (double)E.nnz + sweeps * (E.n + 1.0 * ee + 3.0 * ee);
        if (r0 <= o->tol) {
            rep->status = BGABP_CONVERGED;
        } else {
            for (int it = 1; it <= o->max_iter; ++it) {
                E.reset_ctrl();
                E.launch_residual(E.d_b, E.d_aux, E.d_r, nullptr, MODE_PLAIN);
                E.correction_sweeps_dev(E.d_r, *s, sweeps, E.d_e);
                k_axpy1<<<nblk(E.n), 256, 0, E.st>>>(E.d_aux, E.d_e, E.n);
                E.launch_residual(E.d_b, E.d_aux, nullptr, &E.d_ctrl->red[2], MODE_PLAIN);
                E.read_ctrl();
                const double r = bits2d(E.h_ctrl->red[2]);
                hist.push_back(r);
                rep->iterations = it;
                rep->flop_estimate += per_iter + 2.0 * (double)E.nnz;
                if (!std::isfinite(r) || r > o->divergence_factor * r0) {
                    rep->status = BGABP_DIVERGED;
                    d = "residual blowup";
                    break;
                }
                if (r <= o->tol) {
                    rep->status = BGABP_CONVERGED;
                    break;
                }
            }
        }
        if (x_out && E.n > 0)
            ck(cudaMemcpyAsync(x_out, E.d_aux, sizeof(double) * E.n, cudaMemcpyDeviceToHost, E.st), "D2H");
        ck(cudaStreamSynchronize(E.st), "sync");
        if (history) std::memcpy(history, hist.data(), sizeof(double) * hist.size());
        put_err(detail, dl, d);
        return BGABP_OK;
    })
}

}  // extern "C"
