// Geometric multigrid V-cycle with the GaBP smoother on the device (multigrid.hpp:17-103,
// multigrid.cpp:54-318).  Every level is a bgabp::Engine sharing one stream; a V-cycle is a
// host-driven sequence of kernel launches with no synchronisation inside the cycle.  Smoother
// breakdowns are recorded on the device (k_plain_check) and turned into the reference's
// "smoother breakdown on level k: ..." after the cycle.  The coarsest level is solved with a
// precomputed inverse (host partial-pivot LU at setup, device GEMV per cycle) in place of the
// reference's Eigen PartialPivLU; only that solve's rounding differs from the reference.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "engine.h"
#include "line.h"
#include "problems.h"

using namespace bgabp;

namespace {

enum { GabpSeq = 0, GabpRB = 1, GabpFC = 2, GabpFlood = 3, GabpLine = 4, Jacobi = 5, GsLex = 6, GsRB = 7, GsFC = 8 };
bool is_gabp(int s) { return s >= 0 && s <= 3; }
bool supported(int s) { return s >= 0 && s <= 8; }

struct MgLevel {
    std::unique_ptr<Engine> E;
    int nx = 0;
    bgabp_schedule sched{};
    bool frozen_ok = false;
    bool frozen_pending = false;  // precompute_lambda deferred to first use
    double *d_b = nullptr, *d_x = nullptr;  // this level's right-hand side and iterate (coarse levels)
    std::unique_ptr<LineEngine> line;        // GabpLine: grid-line region GaBP (multigrid.cpp:96-100)
};

// dense partial-pivot LU + explicit inverse of the coarsest operator (host, setup only)
std::vector<double> dense_inverse(Engine& E) {
    E.ensure_host();
    const int n = E.n;
    std::vector<double> a((size_t)n * n, 0.0), inv((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i)
        for (int p = E.ro[i]; p < E.ro[i + 1]; ++p) a[(size_t)i * n + E.ci[p]] = E.val[p];
    std::vector<int> piv(n);
    for (int k = 0; k < n; ++k) {
        int best = k;
        for (int i = k + 1; i < n; ++i)
            if (std::abs(a[(size_t)i * n + k]) > std::abs(a[(size_t)best * n + k])) best = i;
        piv[k] = best;
        if (best != k)
            for (int c = 0; c < n; ++c) std::swap(a[(size_t)k * n + c], a[(size_t)best * n + c]);
        const double d = a[(size_t)k * n + k];
        if (d == 0.0) continue;
        // rows are independent: the same operations per element as the serial loop
#pragma omp parallel for schedule(static) if (n - k > 64)
        for (int i = k + 1; i < n; ++i) {
            double& l = a[(size_t)i * n + k];
            l /= d;
            if (l != 0.0)
                for (int c = k + 1; c < n; ++c) a[(size_t)i * n + c] -= l * a[(size_t)k * n + c];
        }
    }
    // columns of the inverse, four at a time per thread: each column's operations and their
    // order are those of the one-column substitution (independent accumulations, more ILP)
    constexpr int B = 4;
#pragma omp parallel for schedule(dynamic, 2)
    for (int c0 = 0; c0 < n; c0 += B) {
        const int nb = std::min(B, n - c0);
        std::vector<double> y((size_t)n * B, 0.0);  // y[i * B + q]: column c0 + q
        for (int q = 0; q < nb; ++q) y[(size_t)(c0 + q) * B + q] = 1.0;
        for (int k = 0; k < n; ++k)
            if (piv[k] != k)
                for (int q = 0; q < B; ++q) std::swap(y[(size_t)k * B + q], y[(size_t)piv[k] * B + q]);
        for (int i = 0; i < n; ++i) {
            double acc[B];
            for (int q = 0; q < B; ++q) acc[q] = y[(size_t)i * B + q];
            const double* ai = a.data() + (size_t)i * n;
            for (int c = 0; c < i; ++c)
                for (int q = 0; q < B; ++q) acc[q] -= ai[c] * y[(size_t)c * B + q];
            for (int q = 0; q < B; ++q) y[(size_t)i * B + q] = acc[q];
        }
        for (int i = n - 1; i >= 0; --i) {
            double acc[B];
            for (int q = 0; q < B; ++q) acc[q] = y[(size_t)i * B + q];
            const double* ai = a.data() + (size_t)i * n;
            for (int c = i + 1; c < n; ++c)
                for (int q = 0; q < B; ++q) acc[q] -= ai[c] * y[(size_t)c * B + q];
            for (int q = 0; q < B; ++q) y[(size_t)i * B + q] = acc[q] / ai[i];
        }
        for (int i = 0; i < n; ++i)
            for (int q = 0; q < nb; ++q) inv[(size_t)i * n + c0 + q] = y[(size_t)i * B + q];
    }
    return inv;
}

// flop_table (analysis.cpp:135-154) for the smoother kinds a Hierarchy can carry: per-unknown
// cost of `sweeps` smoothing sweeps (SolveReport::flop_estimate of mg_solve, multigrid.cpp:288,302)
enum class FlopSmoother { Gabp, LineGabp, Gs };
double flop_table(bool five, FlopSmoother sm, int sweeps) {
    if (sweeps < 1) throw InvalidArg("flop_table: sweeps must be >= 1");
    const double M = sweeps;
    switch (sm) {
        case FlopSmoother::Gabp: return five ? 12.0 * M + 6.0 : 24.0 * M + 8.0;
        case FlopSmoother::LineGabp:
            if (!five)
                throw InvalidArg("flop_table: line regions do not cover the nine-point stencil's diagonal couplings");
            return sweeps == 1 ? 38.0 : 28.0 * M + 9.0;
        case FlopSmoother::Gs: return five ? 9.0 * M : 17.0 * M;
    }
    return 0.0;
}

// thrown by a checked smoothing call at the breakdown (the reference's runtime_error, which stops
// the cycle before the level's x += e, multigrid.cpp:183-186)
struct MgBreak {};

// reset every level's Ctrl the way the host template of Engine::reset_ctrl does; one block per level
__global__ void k_mg_clear(Ctrl* const* c, int nl) {
    if ((int)blockIdx.x >= nl) return;
    Ctrl* t = c[blockIdx.x];
    unsigned* w = reinterpret_cast<unsigned*>(t);
    for (int i = threadIdx.x; i < (int)(sizeof(Ctrl) / sizeof(unsigned)); i += blockDim.x) w[i] = 0u;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int q = 0; q < 4; ++q) t->epiv[q] = t->npiv[q] = kNone;
        t->opiv = kNone;
    }
}

// out[0] = the stop test's residual bits: *rres, or the max of the npart per-block values in
// rpart (k_residual_dia's rpart), or 0; out[1] = min over halted levels of
// (fail_seq << 32 | level), kNone if no level halted: the first failure in execution order.
// With rpart: kMgSummaryBlocks blocks of 1024 threads fold the partials into out[0] by atomicMax
// (the caller zeroes it first; one block alone is bound by a single SM's L2 bandwidth: 12-35 us
// for the 65k partials of a 4095^2 level); block 0 also scans the levels.  Otherwise one block.
constexpr int kMgSummaryBlocks = 16;
__global__ void __launch_bounds__(1024) k_mg_summary(Ctrl* const* c, int nl, const unsigned long long* rres,
                                                     const unsigned long long* rpart, int npart,
                                                     unsigned long long* out) {
    __shared__ unsigned long long part[32];
    unsigned long long m = 0ull;
    if (rpart) {
        // 16 independent loads in flight per thread (one dependent L2 round trip per element made
        // this 35 us for the 65k partials of a 4095^2 level)
        constexpr int U = 4;
        const int nthr = gridDim.x * blockDim.x;
        for (int i0 = blockIdx.x * blockDim.x + threadIdx.x; i0 < npart; i0 += U * nthr) {
            unsigned long long v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int i = i0 + u * nthr;
                v[u] = i < npart ? __ldcg(rpart + i) : 0ull;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) m = v[u] > m ? v[u] : m;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long other = __shfl_xor_sync(0xffffffffu, m, o);
            m = other > m ? other : m;
        }
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = m;
        __syncthreads();
    }
    if (blockIdx.x != 0) {  // the other blocks only fold their slice of the partials
        if (threadIdx.x == 0) {
            for (int k = 1; k < (int)(blockDim.x >> 5); ++k) m = part[k] > m ? part[k] : m;
            if (m != 0ull) atomicMax(&out[0], m);
        }
        return;
    }
    if (threadIdx.x >= 32) return;
    // the levels' halt words in parallel (lane k = level k, then levels k + 32, ...): one pair of
    // dependent loads instead of nl of them in a row
    unsigned long long best = kNone;
    for (int k = threadIdx.x; k < nl; k += 32) {
        const Ctrl* ck = c[k];
        if (ck->halt) {
            const unsigned long long key = ((unsigned long long)(unsigned)ck->fail_seq << 32) | (unsigned)k;
            best = key < best ? key : best;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
        best = other < best ? other : best;
    }
    if (threadIdx.x != 0) return;
    if (rpart)
        for (int k = 1; k < (int)(blockDim.x >> 5); ++k) m = part[k] > m ? part[k] : m;
    if (rpart) {
        if (m != 0ull) atomicMax(&out[0], m);  // out[0] was zeroed before the residual launch
    } else {
        out[0] = rres ? *rres : 0ull;
    }
    out[1] = best;
}

// a captured V-cycle (cycle(0, ...) plus the Ctrl reset) for one (spec, b, x, reuse) key
struct CycleGraph {
    int pre = 0, post = 0, frozen = 0;
    const double* b = nullptr;
    const double* x = nullptr;
    bool reuse = false;
    int seen = 0;
    cudaGraphExec_t exec = nullptr;
};

}  // namespace

struct bgmg {
    int smoother = 0;
    cudaStream_t st = nullptr;
    std::vector<MgLevel> levels;
    double* d_inv = nullptr;
    double* d_fine_b = nullptr;  // scratch for host-buffer calls
    double* d_fine_x = nullptr;
    std::vector<double> fine_rhs;  // named hierarchies: Hierarchy::fine_rhs
    Ctrl* h_ctrl = nullptr;
    int seq = 0;
    Ctrl** d_ctrls = nullptr;               // every level's d_ctrl, for k_mg_clear / k_mg_summary
    unsigned long long* d_sum = nullptr;    // k_mg_summary output
    unsigned long long* d_rpart = nullptr;  // per-block max |r| of the stop test's residual (DIA fine level)
    unsigned long long* h_sum = nullptr;    // pinned copy of it
    std::vector<CycleGraph> graphs;
    bool use_graphs = true;
    bool checked = false;       // smoothing calls synchronise and stop at a breakdown (MgBreak)
    int fine_nx = 0;            // fine grid and the population of its centre row / of A
    long long fine_center_nnz = 0, fine_nnz = 0;

    // Hierarchy::cycle_flops_per_unknown (multigrid.cpp:240-274): the fine stencil is classified
    // by its centre row (nine-point when it holds more than 5 entries)
    double cycle_flops_per_unknown(const bgmg_cycle& spec) const {
        const bool nine = fine_center_nnz > 5;
        auto analytic = [&](int sweeps) -> double {
            if (sweeps <= 0) return 0.0;
            if (is_gabp(smoother)) return flop_table(!nine, FlopSmoother::Gabp, sweeps);
            if (smoother == GabpLine && !nine) return flop_table(true, FlopSmoother::LineGabp, sweeps);
            if (smoother >= Jacobi && smoother <= GsFC) return flop_table(!nine, FlopSmoother::Gs, sweeps);
            const int n = levels[0].E->n;  // no closed form: multiply-adds per sweep
            return sweeps * 2.0 * (double)fine_nnz / n;
        };
        return analytic(spec.pre) + analytic(spec.post);
    }

    // checked mode: synchronise after a cold smoothing call and stop at its breakdown
    void check_breakdown(int k) {
        if (!checked) return;
        ck(cudaMemcpyAsync(h_ctrl, levels[k].E->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        if (h_ctrl->halt) throw MgBreak{};
    }

    ~bgmg() {
        if (st) cudaStreamSynchronize(st);
        for (auto& g : graphs)
            if (g.exec) cudaGraphExecDestroy(g.exec);
        if (d_ctrls) cudaFree(d_ctrls);
        if (d_sum) cudaFree(d_sum);
        if (d_rpart) cudaFree(d_rpart);
        if (h_sum) cudaFreeHost(h_sum);
        levels.clear();
        if (d_inv) cudaFree(d_inv);
        if (d_fine_b) cudaFree(d_fine_b);
        if (d_fine_x) cudaFree(d_fine_x);
        if (h_ctrl) cudaFreeHost(h_ctrl);
        if (st) cudaStreamDestroy(st);
    }

    Engine& E(int k) { return *levels[k].E; }
    int nl() const { return (int)levels.size(); }

    // whether smooth(k, ..., sweeps, frozen) runs the recorded red-black sweeps (rb_smooth_add)
    bool smooth_uses_rb(int k, int sweeps, bool frozen) {
        Engine& L = E(k);
        return sweeps > 0 && is_gabp(smoother) && !(frozen && levels[k].frozen_ok) &&
               L.rb_applicable(levels[k].sched) && L.rb_ready && L.rb_pre_sweeps >= sweeps;
    }

    // Hierarchy::smooth (multigrid.cpp:163-208)
    void smooth(int k, const double* b, double* x, int sweeps, bool frozen, bool have_r = false) {
        if (sweeps <= 0) return;
        Engine& L = E(k);
        if (L.n == 0) return;
        const unsigned g = nblk_host(L.n);
        ++seq;
        if (is_gabp(smoother)) {
            // the recorded red-black smoother reads r per colour: have the residual write it so
            const bool rb = smooth_uses_rb(k, sweeps, frozen);
            if (have_r && fine_r_compact != rb) have_r = false;
            if (!have_r) L.launch_residual(b, x, L.d_r, nullptr, MODE_PLAIN, 0, rb ? levels[k].sched.nx : 0);
            if (rb) {
                L.rb_smooth_add(L.d_r, sweeps, x, true);  // recorded lambda/sigma, x += e fused
                return;
            }
            if (frozen && levels[k].frozen_ok) {
                L.correction_sweeps_dev(L.d_r, levels[k].sched, sweeps, L.d_e);
            } else {
                std::string unused;
                L.cold_sweeps_dev(L.d_r, levels[k].sched, sweeps, L.d_e, unused, false, seq);
                check_breakdown(k);
            }
            k_axpy1<<<g, 256, 0, st>>>(x, L.d_e, L.n);
            return;
        }
        if (smoother == GabpLine) {  // multigrid.cpp:189-204: fresh block messages, sequential sweeps
            LineEngine& G = *levels[k].line;
            if (!have_r) L.launch_residual(b, x, L.d_r, nullptr, MODE_PLAIN);
            if (G.record(sweeps)) {  // recorded factors: mean-only sweeps, x += e in the last phase
                G.smooth_add(L.d_r, sweeps, x);
                return;
            }
            G.reset_state();
            ck(cudaMemsetAsync(G.d_fail, 0xff, sizeof(unsigned long long), st), "memset");
            for (int s = 0; s < sweeps; ++s) G.sweep(L.d_r, 0, L.d_e);
            k_line_check<<<1, 1, 0, st>>>(L.d_ctrl, G.d_fail, seq);
            check_breakdown(k);
            k_axpy1<<<g, 256, 0, st>>>(x, L.d_e, L.n);
            return;
        }
        // point relaxations in place (classic.cpp:99-146)
        k_plain_reset<<<1, 1, 0, st>>>(L.d_ctrl);
        if (smoother == Jacobi) {
            for (int s = 0; s < sweeps; ++s) {
                L.launch_jacobi(b, x, L.d_e);
                ck(cudaMemcpyAsync(x, L.d_e, sizeof(double) * L.n, cudaMemcpyDeviceToDevice, st), "copy");
            }
        } else if (smoother == GsRB && L.rb_applicable(levels[k].sched)) {  // colour-compact coefficients
            L.rb_build(levels[k].sched.nx, false);
            for (int s = 0; s < sweeps; ++s) L.launch_gs_rb(b, x);
        } else {
            const Levels& lv = L.levels_for(levels[k].sched);
            for (int s = 0; s < sweeps; ++s) L.launch_gs_levels(lv, b, x);
        }
        k_plain_check<<<1, 1, 0, st>>>(L.d_ctrl, seq, 5);
        check_breakdown(k);
    }

    // Hierarchy::cycle (multigrid.cpp:210-232)
    void cycle(int k, const bgmg_cycle& spec, const double* b, double* x) {
        Engine& L = E(k);
        if (k == nl() - 1) {  // direct solve overwrites x (multigrid.cpp:212-216)
            if (L.n > 0) k_gemv_rows<<<nblk_host((long long)L.n * 32), 256, 0, st>>>(d_inv, b, x, L.n);
            return;
        }
        // the stop test of the previous cycle left r = b - A x of this very x in d_r
        const bool reuse = k == 0 && fine_r_b == b && fine_r_x == x;
        if (k == 0) fine_r_b = fine_r_x = nullptr;
        smooth(k, b, x, spec.pre, spec.frozen != 0, reuse);
        MgLevel& C = levels[k + 1];
        L.launch_residual(b, x, L.d_r, nullptr, MODE_PLAIN);
        const int mc = (levels[k].nx - 1) / 2;
        if ((long long)mc * mc == C.E->n && C.E->n > 0) {  // the restriction also zeroes the coarse start vector
            k_restrict<<<nblk_host(C.E->n), 256, 0, st>>>(L.d_r, levels[k].nx, C.d_b, C.d_x);
        } else {
            k_restrict<<<nblk_host(C.E->n), 256, 0, st>>>(L.d_r, levels[k].nx, C.d_b);
            ck(cudaMemsetAsync(C.d_x, 0, sizeof(double) * std::max(C.E->n, 1), st), "memset");
        }
        cycle(k + 1, spec, C.d_b, C.d_x);
        k_prolong_add<<<dim3(nblk_host(C.nx + 1), levels[k].nx), 256, 0, st>>>(C.d_x, C.nx, x, 0);
        smooth(k, b, x, spec.post, spec.frozen != 0);
    }

    void clear_failures() {
        k_mg_clear<<<nl(), 128, 0, st>>>(d_ctrls, nl());
        seq = 0;
    }

    // first smoother failure of the last cycle, in execution order; "" if none (one summary read;
    // the per-level scan only when some level halted)
    std::string failure() {
        k_mg_summary<<<1, 32, 0, st>>>(d_ctrls, nl(), nullptr, nullptr, 0, d_sum);
        ck(cudaMemcpyAsync(h_sum, d_sum, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        return h_sum[1] == kNone ? std::string() : failure_detail();
    }

    std::string failure_detail() {
        int best_seq = 0x7fffffff, best = -1;
        std::string msg;
        for (int k = 0; k < nl(); ++k) {
            ck(cudaMemcpyAsync(h_ctrl, levels[k].E->d_ctrl, sizeof(Ctrl), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            if (h_ctrl->halt && h_ctrl->fail_seq < best_seq) {
                best_seq = h_ctrl->fail_seq;
                best = k;
                if (smoother == GabpLine) {
                    msg = levels[k].line->fail_message(h_ctrl->detail_key);
                } else {
                    const Levels* lv =
                        levels[k].sched.kind == BGABP_SCHED_FLOOD ? nullptr : &E(k).levels_for(levels[k].sched);
                    msg = E(k).decode_failure(*h_ctrl, lv ? &lv->order : nullptr);
                }
            }
        }
        if (best < 0) return "";
        if (is_gabp(smoother) || smoother == GabpLine)
            return "smoother breakdown on level " + std::to_string(best) + ": " + msg;
        return msg;  // relax() throws its own message (classic.cpp:27,43)
    }

    void ensure_frozen() {
        for (auto& lv : levels) {
            if (!lv.frozen_pending) continue;
            int cv = 0, its = 0;
            lv.E->precompute_lambda(lv.sched, 1e-10, 500, cv, its);  // multigrid.cpp:94-95
            lv.frozen_ok = cv != 0;
            lv.frozen_pending = false;
        }
    }

    // record the cold-start precisions the cycle's smoothing calls need (once per level)
    void prepare(const bgmg_cycle& spec) {
        if (spec.frozen) ensure_frozen();
        if (!is_gabp(smoother) || spec.frozen) return;
        const int sw = std::max(spec.pre, spec.post);
        if (sw <= 0) return;
        for (int k = 0; k + 1 < nl(); ++k) {
            Engine& L = E(k);
            if (!L.rb_applicable(levels[k].sched)) continue;
            L.rb_build(levels[k].sched.nx);
            L.rb_precompute(sw);
        }
    }

    // One V-cycle.  The launch sequence of a cycle depends only on (spec, b, x, reuse of the stop
    // test's residual): from the second cycle with a key on, the sequence is replayed from a CUDA
    // graph captured once (host launch overhead dominates the coarse levels).  Anything a first
    // call sets up (recorded factors, level orders, pipeline tables) exists by then; a capture
    // that fails for any reason turns graphs off and the cycle runs as plain launches.
    void v_cycle_dev(const bgmg_cycle& spec, const double* b, double* x) {
        prepare(spec);
        const bool reuse = fine_r_b == b && fine_r_x == x;
        CycleGraph* g = nullptr;
        if (use_graphs) {
            for (auto& c : graphs)
                if (c.pre == spec.pre && c.post == spec.post && c.frozen == spec.frozen && c.b == b && c.x == x &&
                    c.reuse == reuse)
                    g = &c;
            if (!g) {
                if (graphs.size() >= 8) {  // bounded: callers cycling through many buffers
                    if (graphs.front().exec) cudaGraphExecDestroy(graphs.front().exec);
                    graphs.erase(graphs.begin());
                }
                CycleGraph c;
                c.pre = spec.pre;
                c.post = spec.post;
                c.frozen = spec.frozen;
                c.b = b;
                c.x = x;
                c.reuse = reuse;
                graphs.push_back(c);
                g = &graphs.back();
            }
            if (!g->exec && ++g->seen >= 2) capture(*g, spec, b, x);
        }
        if (g && g->exec) {
            fine_r_b = fine_r_x = nullptr;
            seq = 0;
            ck(cudaGraphLaunch(g->exec, st), "graph launch");
            return;
        }
        clear_failures();
        cycle(0, spec, b, x);
        ck(cudaGetLastError(), "v-cycle");
    }

    // One V-cycle as plain launches that stops at the first smoother breakdown, leaving x where
    // the reference's exception leaves it (multigrid.cpp:234-238, 290-297): only the level-0
    // updates made before the breakdown.  Breakdowns are rare, so the fast path never pays for
    // this; the callers re-run a failed cycle in this mode from the same x.
    void v_cycle_checked(const bgmg_cycle& spec, const double* b, double* x) {
        prepare(spec);
        clear_failures();
        checked = true;
        try {
            cycle(0, spec, b, x);
        } catch (const MgBreak&) {
        }
        checked = false;
        fine_r_b = fine_r_x = nullptr;
        ck(cudaGetLastError(), "v-cycle");
    }

    void capture(CycleGraph& g, const bgmg_cycle& spec, const double* b, double* x) {
        const double *rb = fine_r_b, *rx = fine_r_x;
        cudaGraph_t graph = nullptr;
        bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
        if (ok) {
            try {
                clear_failures();
                cycle(0, spec, b, x);
            } catch (...) {
                ok = false;
            }
            ok = cudaStreamEndCapture(st, &graph) == cudaSuccess && ok && graph;
        }
        if (ok) ok = cudaGraphInstantiate(&g.exec, graph, 0) == cudaSuccess;
        if (graph) cudaGraphDestroy(graph);
        if (!ok) {
            g.exec = nullptr;
            use_graphs = false;
            cudaGetLastError();  // clear the capture error; the cycle runs uncaptured
        }
        fine_r_b = rb;  // cycle() consumed them during capture; the replay (or the plain cycle) needs them
        fine_r_x = rx;
    }

    // the stop test's residual r = b - A x also serves the next cycle's first smoothing call (same
    // x, same kernel): fine_r_for records which (b, x) it belongs to
    const double *fine_r_b = nullptr, *fine_r_x = nullptr;
    bool fine_r_compact = false;  // ... stored colour-compact (the next pre-smoothing is recorded red-black)

    // the stop test's residual, laid out for the pre-smoothing call of a following cycle.  On a
    // DIA fine level max |r| is left as one value per block in d_rpart (true is returned; the
    // summary kernel folds them), otherwise reduced into d_ctrl->red[2].
    bool stop_test_residual(const bgmg_cycle* spec, const double* b, const double* x) {
        Engine& L = E(0);
        fine_r_compact = spec && smooth_uses_rb(0, spec->pre, spec->frozen != 0);
        const bool parts = spec && L.layout == BGABP_LAYOUT_DIA && L.n > 0;
        if (parts && !d_rpart)
            ck(cudaMalloc(&d_rpart, sizeof(unsigned long long) * L.residual_blocks()), "malloc");
        if (parts) ck(cudaMemsetAsync(d_sum, 0, sizeof(unsigned long long), st), "memset");  // k_mg_summary's max
        if (!parts) ck(cudaMemsetAsync(&L.d_ctrl->red[2], 0, sizeof(unsigned long long), st), "memset");
        L.launch_residual(b, x, L.d_r, &L.d_ctrl->red[2], MODE_PLAIN, 0, fine_r_compact ? levels[0].sched.nx : 0,
                          parts ? d_rpart : nullptr);
        fine_r_b = b;
        fine_r_x = x;
        return parts;
    }

    double residual_inf(const double* b, const double* x) {
        Engine& L = E(0);
        if (L.n == 0) return 0.0;
        stop_test_residual(nullptr, b, x);
        unsigned long long r;
        ck(cudaMemcpyAsync(&r, &L.d_ctrl->red[2], sizeof(r), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        return bits2d(r);
    }

    double inf_norm_dev(const double* v, int n) {
        if (n == 0) return 0.0;
        Engine& L = E(0);
        ck(cudaMemsetAsync(&L.d_ctrl->red[3], 0, sizeof(unsigned long long), st), "memset");
        k_inf_norm<<<std::min<unsigned>(nblk_host(n), 1184), 256, 0, st>>>(v, n, &L.d_ctrl->red[3]);
        unsigned long long r;
        ck(cudaMemcpyAsync(&r, &L.d_ctrl->red[3], sizeof(r), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaStreamSynchronize(st), "sync");
        return bits2d(r);
    }

    // mg_solve (multigrid.cpp:276-318) on device vectors; history on the host.  A smoother
    // breakdown is detected after its cycle; the solve is then replayed (bit-identical up to that
    // cycle) with the failing cycle checked, so x is the reference's partly cycled x.
    void solve_dev(const bgmg_cycle& spec, const double* b, double* x, const bgmg_options& o, bgabp_report& rep,
                   std::vector<double>& hist, std::string& detail) {
        solve_loop(spec, b, x, o, rep, hist, detail, 0);
        if (rep.status == BGABP_DIVERGED && detail != "residual blowup") {
            bgabp_report r2{};
            std::vector<double> h2;
            std::string d2;
            solve_loop(spec, b, x, o, r2, h2, d2, rep.iterations);
        }
    }

    void solve_loop(const bgmg_cycle& spec, const double* b, double* x, const bgmg_options& o, bgabp_report& rep,
                    std::vector<double>& hist, std::string& detail, int checked_cycle) {
        struct ClearR {  // the saved residual is only valid inside this loop
            bgmg* h;
            ~ClearR() { h->fine_r_b = h->fine_r_x = nullptr; }
        } clear_r{this};
        fine_r_b = fine_r_x = nullptr;
        const int n = E(0).n;
        ck(cudaMemsetAsync(x, 0, sizeof(double) * std::max(n, 1), st), "memset");
        const double r0 = inf_norm_dev(b, n);
        hist.assign(1, r0);
        rep.status = BGABP_MAX_ITER;
        rep.iterations = 0;
        rep.flop_estimate = 0.0;
        detail.clear();
        if (r0 <= o.tol) {
            rep.status = BGABP_CONVERGED;
            return;
        }
        const double per_cycle = cycle_flops_per_unknown(spec) * n;
        for (int it = 1; it <= o.max_cycles; ++it) {
            if (it == checked_cycle)
                v_cycle_checked(spec, b, x);
            else
                v_cycle_dev(spec, b, x);
            // stop test and failure summary in one read
            Engine& L = E(0);
            const bool parts = stop_test_residual(&spec, b, x);
            k_mg_summary<<<parts ? kMgSummaryBlocks : 1, 1024, 0, st>>>(d_ctrls, nl(), &L.d_ctrl->red[2],
                                                                         parts ? d_rpart : nullptr,
                                                                         (int)L.residual_blocks(), d_sum);
            ck(cudaMemcpyAsync(h_sum, d_sum, 2 * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st), "D2H");
            ck(cudaStreamSynchronize(st), "sync");
            const double r = bits2d(h_sum[0]);
            std::string f = h_sum[1] == kNone ? std::string() : failure_detail();
            rep.iterations = it;
            if (!f.empty()) {
                rep.status = BGABP_DIVERGED;
                detail = f;
                return;
            }
            hist.push_back(r);
            rep.flop_estimate += per_cycle;
            if (!std::isfinite(r) || r > o.divergence_factor * r0) {
                rep.status = BGABP_DIVERGED;
                detail = "residual blowup";
                return;
            }
            if (r <= o.tol) {
                rep.status = BGABP_CONVERGED;
                return;
            }
        }
    }

    void ensure_fine_scratch() {
        const size_t vb = sizeof(double) * std::max(E(0).n, 1);
        if (!d_fine_b) ck(cudaMalloc(&d_fine_b, vb), "malloc");
        if (!d_fine_x) ck(cudaMalloc(&d_fine_x, vb), "malloc");
    }
};

static bgabp_schedule schedule_for(int sm, int nx) {  // multigrid.cpp:25-32
    bgabp_schedule s{};
    s.nx = s.ny = nx;
    switch (sm) {
        case GabpRB: case GsRB: s.kind = BGABP_SCHED_RED_BLACK_GRID; break;
        case GabpFC: case GsFC: s.kind = BGABP_SCHED_FOUR_COLOR_GRID; break;
        case GabpFlood: case Jacobi: s.kind = BGABP_SCHED_FLOOD; break;
        default: s.kind = BGABP_SCHED_SEQUENTIAL;
    }
    return s;
}

// Hierarchy ctor (multigrid.cpp:74-109) over caller-supplied levels
static void build_hierarchy(bgmg* h, int nlevels, const int* n, const int* const* ro, const int* const* ci,
                            const double* const* v, const int* nx, int smoother) {
    const bool timing = std::getenv("BGABP_TIMING") != nullptr;
    auto t_last = std::chrono::steady_clock::now();
    auto phase = [&](const char* what, int k) {
        if (!timing) return;
        ck(cudaStreamSynchronize(h->st), "sync");
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[mg] %-22s level %d %8.1f ms\n", what, k,
                     std::chrono::duration<double, std::milli>(now - t_last).count());
        t_last = now;
    };
    if (nlevels < 1) throw InvalidArg("Hierarchy: need 1 <= J2 and a coarsest exponent >= 1");
    if (!supported(smoother)) throw InvalidArg("Hierarchy: unsupported smoother " + std::to_string(smoother));
    h->smoother = smoother;
    if (n[0] > 0 && (long long)nx[0] * nx[0] == n[0]) {  // cycle_flops_per_unknown's centre row
        const int c = (nx[0] / 2) * nx[0] + nx[0] / 2;
        h->fine_nx = nx[0];
        h->fine_center_nnz = ro[0][c + 1] - ro[0][c];
        h->fine_nnz = ro[0][n[0]];
    }
    ck(cudaStreamCreateWithFlags(&h->st, cudaStreamNonBlocking), "stream");
    ck(cudaMallocHost((void**)&h->h_ctrl, sizeof(Ctrl)), "host ctrl");
    for (int k = 0; k < nlevels; ++k) {
        if (k + 1 < nlevels && nx[k + 1] != (nx[k] - 1) / 2)
            throw InvalidArg("Hierarchy: level sizes must halve ((nx-1)/2)");
        if ((long long)nx[k] * nx[k] != n[k]) throw InvalidArg("Hierarchy: level is not a square grid");
        MgLevel L;
        L.E = std::make_unique<Engine>();
        L.E->build(n[k], ro[k], ci[k], v[k], BGABP_LAYOUT_AUTO, h->st);
        L.nx = nx[k];
        L.sched = schedule_for(smoother, nx[k]);
        if (smoother == GabpLine) {  // RegionGabpEngine over grid_line_regions(nx, nx) per level
            L.line = std::make_unique<LineEngine>();
            L.line->build(n[k], ro[k], ci[k], v[k], nx[k], nx[k], h->st);
        }
        if (k > 0) {
            L.d_b = static_cast<double*>(L.E->dalloc(sizeof(double) * std::max(n[k], 1)));
            L.d_x = static_cast<double*>(L.E->dalloc(sizeof(double) * std::max(n[k], 1)));
        }
        h->levels.push_back(std::move(L));
        phase("engine build", k);
    }
    // BGABP_MG_NO_PROBE=1 (experiments only, tools/config5_coarse_rules.py): keep every level
    const bool probe = !(std::getenv("BGABP_MG_NO_PROBE") && std::atoi(std::getenv("BGABP_MG_NO_PROBE")) != 0);
    if (is_gabp(smoother)) {
        for (int k = 0; k < (int)h->levels.size(); ++k) {
            MgLevel& L = h->levels[k];
            if (probe && k > 0 && L.E->sweeps_expand(L.sched)) {  // multigrid.cpp:89-93
                h->levels.resize(k + 1);
                break;
            }
            phase("sweeps_expand probe", k);
            // multigrid.cpp:94-95 computes the frozen precisions here for every level it keeps
            // before a truncation; they are only read by frozen cycles and level_frozen_ok, so
            // they are computed on first use (bgmg::ensure_frozen) with the same values
            L.frozen_pending = true;
        }
    }
    std::vector<Ctrl*> ctrls;
    for (auto& L : h->levels) ctrls.push_back(L.E->d_ctrl);
    ck(cudaMalloc(&h->d_ctrls, sizeof(Ctrl*) * ctrls.size()), "malloc");
    ck(cudaMemcpyAsync(h->d_ctrls, ctrls.data(), sizeof(Ctrl*) * ctrls.size(), cudaMemcpyHostToDevice, h->st), "H2D");
    ck(cudaMalloc(&h->d_sum, 2 * sizeof(unsigned long long)), "malloc");
    ck(cudaMallocHost((void**)&h->h_sum, 2 * sizeof(unsigned long long)), "host sum");
    if (const char* e = std::getenv("BGABP_MG_GRAPH")) h->use_graphs = std::atoi(e) != 0;
    Engine& C = *h->levels.back().E;
    if (C.n > 20000)  // a dense n^2 inverse (and its LU) would not fit a sensible setup
        throw InvalidArg("Hierarchy: coarsest level has " + std::to_string(C.n) +
                         " unknowns, too many for the dense direct solve");
    std::vector<double> inv = dense_inverse(C);
    phase("coarse inverse", (int)h->levels.size() - 1);
    ck(cudaMalloc(&h->d_inv, sizeof(double) * std::max<size_t>(inv.size(), 1)), "malloc");
    if (!inv.empty())
        ck(cudaMemcpyAsync(h->d_inv, inv.data(), sizeof(double) * inv.size(), cudaMemcpyHostToDevice, h->st), "H2D");
    ck(cudaStreamSynchronize(h->st), "sync");
}

#define MG_GUARD(ERRBUF, ERRLEN, ...)       \
    try {                                   \
        __VA_ARGS__                         \
    } catch (const InvalidArg& ex) {        \
        put_err(ERRBUF, ERRLEN, ex.what()); \
        return BGABP_EINVAL;                \
    } catch (const CudaError& ex) {         \
        put_err(ERRBUF, ERRLEN, ex.what()); \
        return BGABP_ECUDA;                 \
    } catch (const std::exception& ex) {    \
        put_err(ERRBUF, ERRLEN, ex.what()); \
        return BGABP_ERUNTIME;              \
    }

extern "C" {

int bgmg_create(int nlevels, const int* n, const int* const* row_offsets, const int* const* col_indices,
                const double* const* values, const int* nx, int smoother, bgmg** out, char* err, size_t errlen) {
    *out = nullptr;
    auto h = std::make_unique<bgmg>();
    MG_GUARD(err, errlen, {
        build_hierarchy(h.get(), nlevels, n, row_offsets, col_indices, values, nx, smoother);
        *out = h.release();
        return BGABP_OK;
    })
}

int bgmg_create_named(const char* problem, int J1, int J2, int nparam, const char* const* keys, const double* vals,
                      int smoother, bgmg** out, char* err, size_t errlen) {
    *out = nullptr;
    auto h = std::make_unique<bgmg>();
    MG_GUARD(err, errlen, {
        if (J2 < 1 || J1 - J2 + 1 < 1) throw InvalidArg("Hierarchy: need 1 <= J2 and a coarsest exponent >= 1");
        std::vector<std::unique_ptr<bgabp_problem>> probs;
        std::vector<int> ns, nxs;
        std::vector<const int*> ros, cis;
        std::vector<const double*> vs;
        for (int J = J1; J >= J1 - J2 + 1; --J) {  // multigrid.cpp:79-83
            std::string e;
            probs.emplace_back(assemble_named(problem, J, nparam, keys, vals, e));
            if (!probs.back()) throw InvalidArg(e);
            const bgabp_problem& p = *probs.back();
            ns.push_back(p.n);
            nxs.push_back(p.nx);
            ros.push_back(p.ro.data());
            cis.push_back(p.ci.data());
            vs.push_back(p.val.data());
        }
        build_hierarchy(h.get(), (int)ns.size(), ns.data(), ros.data(), cis.data(), vs.data(), nxs.data(), smoother);
        h->fine_rhs = probs.front()->b;
        *out = h.release();
        return BGABP_OK;
    })
}

void bgmg_destroy(bgmg* h) { delete h; }
int bgmg_num_levels(const bgmg* h) { return (int)h->levels.size(); }
int bgmg_level_frozen_ok(const bgmg* h, int k) {
    try {
        const_cast<bgmg*>(h)->ensure_frozen();
    } catch (const std::exception&) {
        return -1;
    }
    return h->levels[k].frozen_ok ? 1 : 0;
}
int bgmg_level_n(const bgmg* h, int k) { return h->levels[k].E->n; }
int bgmg_level_nx(const bgmg* h, int k) { return h->levels[k].nx; }

int bgmg_cycle_flops_per_unknown(const bgmg* h, const bgmg_cycle* spec, double* out, char* err, size_t errlen) {
    MG_GUARD(err, errlen, {
        *out = h->cycle_flops_per_unknown(*spec);
        return BGABP_OK;
    })
}
void* bgmg_stream(bgmg* h) { return (void*)h->st; }

int bgmg_fine_rhs(const bgmg* h, double* b_out) {
    if (h->fine_rhs.empty()) return BGABP_EINVAL;
    std::memcpy(b_out, h->fine_rhs.data(), sizeof(double) * h->fine_rhs.size());
    return BGABP_OK;
}

int bgmg_vcycle(bgmg* h, const bgmg_cycle* spec, const double* b, double* x, char* err, size_t errlen) {
    MG_GUARD(err, errlen, {
        const int n = h->E(0).n;
        h->ensure_fine_scratch();
        host_to_device(h->d_fine_b, b, sizeof(double) * n, h->st);
        host_to_device(h->d_fine_x, x, sizeof(double) * n, h->st);
        h->fine_r_b = h->fine_r_x = nullptr;
        h->v_cycle_dev(*spec, h->d_fine_b, h->d_fine_x);
        std::string f = h->failure();
        if (!f.empty()) {  // replay from the caller's x, stopping where the reference's exception does
            host_to_device(h->d_fine_x, x, sizeof(double) * n, h->st);
            h->v_cycle_checked(*spec, h->d_fine_b, h->d_fine_x);
        }
        device_to_host(x, h->d_fine_x, sizeof(double) * n, h->st);
        ck(cudaStreamSynchronize(h->st), "sync");
        if (!f.empty()) {
            put_err(err, errlen, f);
            return BGABP_ERUNTIME;
        }
        return BGABP_OK;
    })
}

int bgmg_solve(bgmg* h, const bgmg_cycle* spec, const double* b, const bgmg_options* opt, bgabp_report* rep,
               double* x_out, double* history, char* detail, size_t dl) {
    MG_GUARD(detail, dl, {
        const int n = h->E(0).n;
        h->ensure_fine_scratch();
        host_to_device(h->d_fine_b, b, sizeof(double) * n, h->st);
        std::vector<double> hist;
        std::string d;
        h->solve_dev(*spec, h->d_fine_b, h->d_fine_x, *opt, *rep, hist, d);
        if (x_out) device_to_host(x_out, h->d_fine_x, sizeof(double) * n, h->st);
        ck(cudaStreamSynchronize(h->st), "sync");
        if (history) std::memcpy(history, hist.data(), sizeof(double) * hist.size());
        put_err(detail, dl, d);
        return BGABP_OK;
    })
}

int bgmg_solve_device(bgmg* h, const bgmg_cycle* spec, const double* b_dev, const bgmg_options* opt,
                      bgabp_report* rep, double* x_dev, double* history, char* detail, size_t dl) {
    MG_GUARD(detail, dl, {
        std::vector<double> hist;
        std::string d;
        h->solve_dev(*spec, b_dev, x_dev, *opt, *rep, hist, d);
        ck(cudaStreamSynchronize(h->st), "sync");
        if (history) std::memcpy(history, hist.data(), sizeof(double) * hist.size());
        put_err(detail, dl, d);
        return BGABP_OK;
    })
}

int bgmg_restrict(const double* fine, int mf, double* out) {
    try {
        const int mc = (mf - 1) / 2;
        if (mc <= 0) return BGABP_EINVAL;
        double *df, *dc;
        ck(cudaMalloc(&df, sizeof(double) * mf * mf), "malloc");
        ck(cudaMalloc(&dc, sizeof(double) * mc * mc), "malloc");
        ck(cudaMemcpy(df, fine, sizeof(double) * mf * mf, cudaMemcpyHostToDevice), "H2D");
        k_restrict<<<nblk_host((long long)mc * mc), 256>>>(df, mf, dc);
        ck(cudaMemcpy(out, dc, sizeof(double) * mc * mc, cudaMemcpyDeviceToHost), "D2H");
        cudaFree(df);
        cudaFree(dc);
        return BGABP_OK;
    } catch (const std::exception&) {
        return BGABP_ECUDA;
    }
}

int bgmg_prolong(const double* coarse, int mc, double* out) {
    try {
        const int mf = 2 * mc + 1;
        double *df, *dc;
        ck(cudaMalloc(&df, sizeof(double) * mf * mf), "malloc");
        ck(cudaMalloc(&dc, sizeof(double) * std::max(mc * mc, 1)), "malloc");
        if (mc > 0) ck(cudaMemcpy(dc, coarse, sizeof(double) * mc * mc, cudaMemcpyHostToDevice), "H2D");
        k_prolong_add<<<dim3(nblk_host(mc + 1), mf), 256>>>(dc, mc, df, 1);
        ck(cudaMemcpy(out, df, sizeof(double) * mf * mf, cudaMemcpyDeviceToHost), "D2H");
        cudaFree(df);
        cudaFree(dc);
        return BGABP_OK;
    } catch (const std::exception&) {
        return BGABP_ECUDA;
    }
}

}  // extern "C"
