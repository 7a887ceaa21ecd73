// Line GaBP engine (region_gabp.cpp:30-198 over grid_line_regions, region.cpp:208-221) and its
// C-ABI (include/gabp_b200.h, bglin_*).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "line.h"

namespace bgabp {

static inline unsigned lblk(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

LineEngine::~LineEngine() {
    if (st) cudaStreamSynchronize(st);
    for (void* p : allocs) cudaFree(p);
    if (h_ctrl) cudaFreeHost(h_ctrl);
    if (own_stream && st) cudaStreamDestroy(st);
}

void* LineEngine::dalloc(size_t bytes) {
    void* p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(bytes, 8)), "cudaMalloc");
    allocs.push_back(p);
    return p;
}

void LineEngine::build(int n_, const int* ro, const int* ci, const double* v, int nx_, int ny_, cudaStream_t shared) {
    if (n_ < 0 || nx_ <= 0 || ny_ <= 0) throw InvalidArg("line gabp: grid dimensions must be positive");
    n = n_;
    nx = nx_;
    ny = ny_;
    nnz = ro[n];
    const long long grid = (long long)nx * ny;
    // build_two_layer_region_graph checks, in its order (region.cpp:70-101): per large region
    // (rows, then columns) range and connectivity; then coverage of variables and of edges
    auto stored = [&](int i, int j) {
        if (i < 0 || i >= n || j < 0 || j >= n) return false;
        return std::binary_search(ci + ro[i], ci + ro[i + 1], j);
    };
    auto linked = [&](int i, int j) { return stored(i, j) || stored(j, i); };
    for (int L = 0; L < ny + nx; ++L) {
        const bool row = L < ny;
        const int len = row ? nx : ny;
        const long long first = row ? (long long)L * nx : (long long)(L - ny);
        const long long last = row ? first + nx - 1 : first + (long long)(ny - 1) * nx;
        if (last >= n) throw InvalidArg("large region " + std::to_string(L) + " index out of range");
        const int stride = row ? 1 : nx;
        for (int k = 0; k + 1 < len; ++k) {
            const int a = (int)(first + (long long)k * stride), b = a + stride;
            if (!linked(a, b))
                throw InvalidArg("large region " + std::to_string(L) + " induces a disconnected subgraph");
        }
    }
    if (grid < n) throw InvalidArg("variable " + std::to_string(grid) + " is covered by no large region");
    std::vector<double> diag(n, 0.0), w(n, 0.0), e(n, 0.0), s(n, 0.0), nn(n, 0.0);
    std::vector<uint32_t> mask(n, 0u);
    std::pair<int, int> uncovered{-1, -1};
    bool other = false;  // covered by a line but not a 5-point neighbour (unsupported here)
    for (int i = 0; i < n; ++i)
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            const int j = ci[p];
            if (j == i) {
                diag[i] = v[p];
                continue;
            }
            const bool same_row = i / nx == j / nx, same_col = i % nx == j % nx;
            if (same_row && j == i - 1) {
                w[i] = v[p];
                mask[i] |= 2u;
            } else if (same_row && j == i + 1) {
                e[i] = v[p];
                mask[i] |= 4u;
            } else if (j == i - nx) {
                s[i] = v[p];
                mask[i] |= 1u;
            } else if (j == i + nx) {
                nn[i] = v[p];
                mask[i] |= 8u;
            } else if (same_row || same_col) {
                other = true;
            } else {
                const std::pair<int, int> ed{std::min(i, j), std::max(i, j)};
                if (uncovered.first < 0 || ed < uncovered) uncovered = ed;
            }
        }
    if (uncovered.first >= 0)
        throw InvalidArg("edge (" + std::to_string(uncovered.first) + "," + std::to_string(uncovered.second) +
                         ") is covered by no large region");
    if (other) throw InvalidArg("line gabp: only 5-point couplings inside a grid line are supported on the device");
    if (shared) {
        st = shared;
    } else {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "stream");
        own_stream = true;
    }
    auto up = [&](const std::vector<double>& h) {
        double* d = static_cast<double*>(dalloc(sizeof(double) * std::max(n, 1)));
        if (n) ck(cudaMemcpyAsync(d, h.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
        return d;
    };
    P.nx = nx;
    P.ny = ny;
    P.n = n;
    P.diag = up(diag);
    P.w = up(w);
    P.e = up(e);
    P.s = up(s);
    P.nn = up(nn);
    uint32_t* dm = static_cast<uint32_t*>(dalloc(sizeof(uint32_t) * std::max(n, 1)));
    if (n) ck(cudaMemcpyAsync(dm, mask.data(), sizeof(uint32_t) * n, cudaMemcpyHostToDevice, st), "H2D");
    P.mask = dm;
    const size_t vb = sizeof(double) * std::max(n, 1);
    for (int k = 0; k < 2; ++k) {
        lr[k] = static_cast<double*>(dalloc(vb));
        mr[k] = static_cast<double*>(dalloc(vb));
        lc[k] = static_cast<double*>(dalloc(vb));
        mc[k] = static_cast<double*>(dalloc(vb));
    }
    d_fd = static_cast<double*>(dalloc(vb));
    d_fy = static_cast<double*>(dalloc(vb));
    d_x = static_cast<double*>(dalloc(vb));
    d_b = static_cast<double*>(dalloc(vb));
    d_ctrl = static_cast<LineCtrl*>(dalloc(sizeof(LineCtrl)));
    d_fail = &d_ctrl->fail;
    ck(cudaMallocHost((void**)&h_ctrl, sizeof(LineCtrl)), "cudaMallocHost");
    std::memset(h_ctrl, 0, sizeof(LineCtrl));
    h_ctrl->fail = kNone;
    ck(cudaMemcpyAsync(d_ctrl, h_ctrl, sizeof(LineCtrl), cudaMemcpyHostToDevice, st), "ctrl");
    reset_state();
    ck(cudaStreamSynchronize(st), "sync");
}

void LineEngine::reset_state() {
    const size_t vb = sizeof(double) * std::max(n, 1);
    for (int k = 0; k < 2; ++k) {
        ck(cudaMemsetAsync(lr[k], 0, vb, st), "memset");
        ck(cudaMemsetAsync(mr[k], 0, vb, st), "memset");
        ck(cudaMemsetAsync(lc[k], 0, vb, st), "memset");
        ck(cudaMemsetAsync(mc[k], 0, vb, st), "memset");
    }
    cur = 0;
}

void LineEngine::clear_fail() {
    const unsigned long long none = kNone;
    ck(cudaMemcpyAsync(d_fail, &none, sizeof none, cudaMemcpyHostToDevice, st), "fail");
    ck(cudaStreamSynchronize(st), "sync");
}

void LineEngine::sweep(const double* b, int mode, double* x, const int* done) {
    if (n == 0) return;
    const int c = cur, o = mode == 1 ? cur ^ 1 : cur;  // flood writes the other buffer
    k_line_full_rows<false><<<lblk(ny, 4), 128, 0, st>>>(P, b, lc[c], mc[c], lr[o], mr[o], d_fd, d_fy, d_fail, done,
                                                         LineRec{});
    k_line_full_cols<false><<<lblk(nx, kFCW), kFCT, 0, st>>>(P, b, mode == 1 ? lr[c] : lr[o],
                                                             mode == 1 ? mr[c] : mr[o], lc[o], mc[o], x, d_fd, d_fy,
                                                             d_fail, done, LineRec{});
    cur = o;
    ck(cudaGetLastError(), "line sweep");
}

bool LineEngine::record(int sweeps) {
    if (rec_failed) return false;
    if (rec_sweeps >= sweeps || n == 0) return true;
    const size_t vb = sizeof(double) * std::max(n, 1);
    auto one = [&]() {
        LineRec r;
        r.f = static_cast<double*>(dalloc(vb));
        r.rd = static_cast<double*>(dalloc(vb));
        r.W = static_cast<double*>(dalloc(vb));
        return r;
    };
    while ((int)rec_rows.size() < sweeps) {
        rec_rows.push_back(one());
        rec_cols.push_back(one());
    }
    ck(cudaMemsetAsync(d_b, 0, vb, st), "memset b");  // the factors do not depend on b
    reset_state();
    clear_fail();
    for (int s = 0; s < sweeps; ++s) {  // sequential mode: rows then columns, in place
        k_line_full_rows<true><<<lblk(ny, 4), 128, 0, st>>>(P, d_b, lc[0], mc[0], lr[0], mr[0], d_fd, d_fy, d_fail,
                                                            nullptr, rec_rows[s]);
        k_line_full_cols<true><<<lblk(nx, kFCW), kFCT, 0, st>>>(P, d_b, lr[0], mr[0], lc[0], mc[0], nullptr, d_fd,
                                                               d_fy, d_fail, nullptr, rec_cols[s]);
    }
    ck(cudaGetLastError(), "line record");
    if (read_fail() != kNone) {
        rec_failed = true;
        clear_fail();
        return false;
    }
    rec_sweeps = sweeps;
    return true;
}

void LineEngine::smooth_add(const double* r, int sweeps, double* x) {
    if (n == 0 || sweeps <= 0) return;
    ck(cudaMemsetAsync(mc[0], 0, sizeof(double) * n, st), "memset");  // cold start
    for (int s = 0; s < sweeps; ++s) {
        const bool last = s + 1 == sweeps;
        // parallel affine scans (k_line_mean_rows / _cols); k_line_mean_phase is the serial form
        k_line_mean_rows<false><<<lblk(ny, 4), 128, 0, st>>>(P, r, mc[0], mr[0], nullptr, d_fy, rec_rows[s].f,
                                                             rec_rows[s].rd, rec_rows[s].W);
        if (last)
            k_line_mean_cols<true><<<lblk(nx, kCW), kCT, 0, st>>>(P, r, mr[0], mc[0], x, d_fy, rec_cols[s].f,
                                                                       rec_cols[s].rd, rec_cols[s].W);
        else
            k_line_mean_cols<false><<<lblk(nx, kCW), kCT, 0, st>>>(P, r, mr[0], mc[0], nullptr, d_fy,
                                                                        rec_cols[s].f, rec_cols[s].rd, rec_cols[s].W);
    }
    ck(cudaGetLastError(), "line smooth");
}

unsigned long long LineEngine::read_fail() {
    unsigned long long f;
    ck(cudaMemcpyAsync(&f, d_fail, sizeof f, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    return f;
}

std::string LineEngine::fail_message(unsigned long long key) const {
    const int L = (int)(key >> 32), pos = (int)(key & 0xffffffffu);
    if (pos == 0) return "singular local system in region " + std::to_string(L);
    const int k = pos - 1;
    const int child = L < ny ? L * nx + k : k * nx + (L - ny);  // child ids are node ids for grid lines
    return "singular child covariance for region " + std::to_string(L) + " child " + std::to_string(child);
}

double LineEngine::sweep_flops() const {
    double t = 0.0;
    auto region = [](double N) { return N * (1.5 + 2.0 * 2.0) + 1.5 * N * N * N; };  // N children, |l| = 1, p = 2
    for (int L = 0; L < ny; ++L) t += region(nx);
    for (int L = 0; L < nx; ++L) t += region(ny);
    return t;
}

// reference edge order: row regions then column regions, each region's children in order
void LineEngine::set_state(const double* lam, const double* m) {
    std::vector<double> a(n), bm(n), c(n), cm(n);
    for (int v = 0; v < n; ++v) {
        a[v] = lam[v];
        bm[v] = m[v];
        const int ix = v % nx, iy = v / nx;
        c[v] = lam[n + (size_t)ix * ny + iy];
        cm[v] = m[n + (size_t)ix * ny + iy];
    }
    if (n) {
        ck(cudaMemcpyAsync(lr[cur], a.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(mr[cur], bm.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(lc[cur], c.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
        ck(cudaMemcpyAsync(mc[cur], cm.data(), sizeof(double) * n, cudaMemcpyHostToDevice, st), "H2D");
    }
    ck(cudaStreamSynchronize(st), "sync");
}

void LineEngine::get_state(double* lam, double* m) {
    std::vector<double> a(n), bm(n), c(n), cm(n);
    if (n) {
        ck(cudaMemcpyAsync(a.data(), lr[cur], sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(bm.data(), mr[cur], sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(c.data(), lc[cur], sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(cm.data(), mc[cur], sizeof(double) * n, cudaMemcpyDeviceToHost, st), "D2H");
    }
    ck(cudaStreamSynchronize(st), "sync");
    for (int v = 0; v < n; ++v) {
        lam[v] = a[v];
        m[v] = bm[v];
        const int ix = v % nx, iy = v / nx;
        lam[n + (size_t)ix * ny + iy] = c[v];
        m[n + (size_t)ix * ny + iy] = cm[v];
    }
}

}  // namespace bgabp

using namespace bgabp;

struct bglin_engine {
    LineEngine L;
};

#define LIN_GUARD(ERRBUF, ERRLEN, ...)       \
    try {                                    \
        __VA_ARGS__                          \
    } catch (const InvalidArg& ex) {         \
        put_err(ERRBUF, ERRLEN, ex.what());  \
        return BGABP_EINVAL;                 \
    } catch (const CudaError& ex) {          \
        put_err(ERRBUF, ERRLEN, ex.what());  \
        return BGABP_ECUDA;                  \
    } catch (const std::exception& ex) {     \
        put_err(ERRBUF, ERRLEN, ex.what());  \
        return BGABP_ERUNTIME;               \
    }

extern "C" {

int bglin_create(int n, const int* ro, const int* ci, const double* v, int nx, int ny, bglin_engine** out, char* err,
                 size_t errlen) {
    LIN_GUARD(err, errlen, {
        auto h = std::make_unique<bglin_engine>();
        h->L.build(n, ro, ci, v, nx, ny);
        *out = h.release();
        return BGABP_OK;
    })
}

void bglin_destroy(bglin_engine* h) { delete h; }

int bglin_num_edges(const bglin_engine* h) { return 2 * h->L.n; }

double bglin_sweep_flops(const bglin_engine* h) { return h->L.sweep_flops(); }

void* bglin_stream(bglin_engine* h) { return (void*)h->L.st; }

int bglin_reset_state(bglin_engine* h) {
    LIN_GUARD(nullptr, 0, {
        h->L.reset_state();
        ck(cudaStreamSynchronize(h->L.st), "sync");
        return BGABP_OK;
    })
}

int bglin_set_state(bglin_engine* h, const double* lam, const double* m) {
    LIN_GUARD(nullptr, 0, {
        h->L.set_state(lam, m);
        return BGABP_OK;
    })
}

int bglin_get_state(bglin_engine* h, double* lam, double* m) {
    LIN_GUARD(nullptr, 0, {
        h->L.get_state(lam, m);
        return BGABP_OK;
    })
}

// RegionGabpEngine::sweep (region_gabp.cpp:145-157) on host b / x
int bglin_sweep(bglin_engine* h, const double* b, int mode, double* x, char* err, size_t errlen) {
    LIN_GUARD(err, errlen, {
        LineEngine& L = h->L;
        if (mode != 0 && mode != 1) throw InvalidArg("line gabp: mode must be 0 (sequential) or 1 (flood)");
        if (L.n == 0) return BGABP_OK;
        const size_t vb = sizeof(double) * L.n;
        ck(cudaMemcpyAsync(L.d_b, b, vb, cudaMemcpyHostToDevice, L.st), "H2D b");
        ck(cudaMemcpyAsync(L.d_x, x, vb, cudaMemcpyHostToDevice, L.st), "H2D x");
        L.clear_fail();
        L.sweep(L.d_b, mode, L.d_x);
        ck(cudaMemcpyAsync(x, L.d_x, vb, cudaMemcpyDeviceToHost, L.st), "D2H x");
        const unsigned long long f = L.read_fail();
        if (f != kNone) {
            put_err(err, errlen, L.fail_message(f));
            return BGABP_EPIVOT;
        }
        return BGABP_OK;
    })
}

// RegionGabpEngine::solve (region_gabp.cpp:159-198): device-resident loop, host polls per chunk
int bglin_solve(bglin_engine* h, const double* b, const bglin_options* o, bgabp_report* rep, double* x_out,
                double* history, char* detail, size_t dl) {
    LIN_GUARD(detail, dl, {
        LineEngine& L = h->L;
        if (o->mode != 0 && o->mode != 1) throw InvalidArg("line gabp: mode must be 0 (sequential) or 1 (flood)");
        const int n = L.n;
        double r0 = 0.0;  // inf_norm (sparse.cpp): std::max skips NaN
        for (int i = 0; i < n; ++i) r0 = std::max(r0, std::abs(b[i]));
        rep->status = BGABP_MAX_ITER;
        rep->iterations = 0;
        rep->flop_estimate = 0.0;
        put_err(detail, dl, "");
        if (history) history[0] = r0;
        if (r0 <= o->tol || n == 0) {
            if (r0 <= o->tol) rep->status = BGABP_CONVERGED;
            if (x_out) std::fill(x_out, x_out + n, 0.0);
            return BGABP_OK;
        }
        if (L.hist_cap < (long long)o->max_iter + 2) {
            L.hist_cap = (long long)o->max_iter + 2;
            L.d_hist = static_cast<double*>(L.dalloc(sizeof(double) * L.hist_cap));
        }
        const size_t vb = sizeof(double) * n;
        ck(cudaMemcpyAsync(L.d_b, b, vb, cudaMemcpyHostToDevice, L.st), "H2D b");
        ck(cudaMemsetAsync(L.d_x, 0, vb, L.st), "memset x");
        L.reset_state();
        LineCtrl c{};
        c.step = 1;
        c.fail = kNone;
        c.r0 = r0;
        c.tol = o->tol;
        c.divergence = o->divergence_factor;
        c.max_iter = o->max_iter;
        c.mode = o->mode;
        c.status = BGABP_MAX_ITER;
        ck(cudaMemcpyAsync(L.d_ctrl, &c, sizeof c, cudaMemcpyHostToDevice, L.st), "ctrl");
        const int* done = &L.d_ctrl->done;
        int enq = 0, chunk = 16;
        while (enq < o->max_iter) {
            const int k = std::min(chunk, o->max_iter - enq);
            for (int i = 0; i < k; ++i) {
                L.sweep(L.d_b, o->mode, L.d_x, done);
                k_line_residual<<<lblk(n, 256), 256, 0, L.st>>>(L.P, L.d_b, L.d_x, nullptr, &L.d_ctrl->rmax, done);
                k_line_decide<<<1, 1, 0, L.st>>>(L.d_ctrl, L.d_hist, 0);
            }
            enq += k;
            chunk = std::min(chunk * 2, 256);
            ck(cudaMemcpyAsync(L.h_ctrl, L.d_ctrl, sizeof(LineCtrl), cudaMemcpyDeviceToHost, L.st), "D2H ctrl");
            ck(cudaStreamSynchronize(L.st), "sync");
            if (L.h_ctrl->done) break;
        }
        ck(cudaMemcpyAsync(L.h_ctrl, L.d_ctrl, sizeof(LineCtrl), cudaMemcpyDeviceToHost, L.st), "D2H ctrl");
        ck(cudaStreamSynchronize(L.st), "sync");
        const LineCtrl& hc = *L.h_ctrl;
        rep->status = hc.done ? hc.status : BGABP_MAX_ITER;
        rep->iterations = hc.done ? hc.iterations : o->max_iter;
        const bool sweep_failed = hc.done && hc.status == BGABP_DIVERGED && hc.detail_key != kNone - 1;
        const int good = rep->iterations - (sweep_failed ? 1 : 0);
        const double per = L.sweep_flops() + 2.0 * (double)L.nnz;
        for (int k = 0; k < good; ++k) rep->flop_estimate += per;
        if (hc.done && hc.status == BGABP_DIVERGED)
            put_err(detail, dl, sweep_failed ? L.fail_message(hc.detail_key) : std::string("residual blowup"));
        if (history && good > 0)
            ck(cudaMemcpyAsync(history + 1, L.d_hist + 1, sizeof(double) * good, cudaMemcpyDeviceToHost, L.st), "D2H");
        if (x_out) ck(cudaMemcpyAsync(x_out, L.d_x, vb, cudaMemcpyDeviceToHost, L.st), "D2H x");
        ck(cudaStreamSynchronize(L.st), "sync");
        return BGABP_OK;
    })
}

}  // extern "C"
