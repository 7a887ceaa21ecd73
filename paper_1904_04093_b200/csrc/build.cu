// Construction of the B200 GaBP engine (bgabp_create): host validation of the caller's CSR,
// device build of the DIA layout (build_kernels.cuh), host graphs on first use, union-CSR layout.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <omp.h>
#include <string>
#include <vector>

#include "engine.h"
#include "build_kernels.cuh"

namespace bgabp {

// ---------------------------------------------------------------------------------------------
// construction: validate the CSR on the host, then build the device layout.  DIA-eligible
// matrices (every config) are uploaded once and laid out by kernels (build_kernels.cuh); the
// host copies (transpose_pos, union neighbour lists) are derived on first use only, by the
// schedules that need them (greedy colourings, dependency levels) and the coarse LU.
// ---------------------------------------------------------------------------------------------
namespace {
struct Phase {
    bool on = getenv("BGABP_TIMING") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void operator()(const char* what) {
        if (!on) return;
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[build] %-28s %8.1f ms\n", what, std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};
}  // namespace

// sparse.hpp:10-27 canonical CSR and gabp.cpp:29-33, read in place (no copy).  Errors in the
// order the reference meets them: a bad row (range before order, first offending entry) before a
// structurally zero diagonal.  Also returns the sorted union offsets D u -D (capped at kMaxDia+1).
static void validate_csr(int n, const int* ro, const int* ci, std::vector<int>& offs) {
    if (ro[0] != 0) throw InvalidArg("gabp: row_offsets[0] must be 0");
    long long bad_mono = n;
#pragma omp parallel for schedule(static) reduction(min : bad_mono)
    for (int i = 0; i < n; ++i)
        if (ro[i + 1] < ro[i]) bad_mono = std::min<long long>(bad_mono, i);
    if (bad_mono < n) throw InvalidArg("gabp: row_offsets not monotone");
    long long bad_row = n, no_diag = n;
    const int T = std::max(1, omp_get_max_threads());
    std::vector<std::vector<int>> part(T);
#pragma omp parallel num_threads(T) reduction(min : bad_row, no_diag)
    {
        std::vector<int>& mine = part[omp_get_thread_num()];
#pragma omp for schedule(static)
        for (int i = 0; i < n; ++i) {
            bool diag = false;
            for (int p = ro[i]; p < ro[i + 1]; ++p) {
                const int j = ci[p];
                if (j < 0 || j >= n || (p > ro[i] && j <= ci[p - 1])) {
                    bad_row = std::min<long long>(bad_row, i);
                    break;
                }
                if (j == i) {
                    diag = true;
                } else if ((int)mine.size() <= kMaxDia &&
                           std::find(mine.begin(), mine.end(), j - i) == mine.end()) {
                    mine.push_back(j - i);
                }
            }
            if (!diag) no_diag = std::min<long long>(no_diag, i);
        }
    }
    if (bad_row < n) {
        const int i = (int)bad_row;
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            if (ci[p] < 0 || ci[p] >= n) throw InvalidArg("gabp: column index out of range");
            if (p > ro[i] && ci[p] <= ci[p - 1]) throw InvalidArg("gabp: CSR is not canonical (columns must increase)");
        }
    }
    if (no_diag < n) throw InvalidArg("gabp: matrix has a structurally zero diagonal entry");
    offs.clear();
    for (const auto& m : part)
        for (int d : m)
            for (int e : {d, -d})
                if ((int)offs.size() <= kMaxDia && std::find(offs.begin(), offs.end(), e) == offs.end())
                    offs.push_back(e);
    std::sort(offs.begin(), offs.end());
}

void Engine::build(int n_, const int* ro_, const int* ci_, const double* v_, int want_layout,
                   cudaStream_t shared_stream) {
    Phase phase;
    if (n_ < 0) throw InvalidArg("gabp: negative dimension");
    n = n_;
    std::vector<int> offs;
    validate_csr(n, ro_, ci_, offs);
    nnz = ro_[n];
    num_edges = nnz - n;
    const bool dia_ok = !offs.empty() && (int)offs.size() <= kMaxDia && offs.size() % 2 == 0;
    if (want_layout == BGABP_LAYOUT_DIA && !dia_ok)
        throw InvalidArg("gabp: DIA layout needs 1..8 symmetric neighbour offsets");
    layout = (want_layout == BGABP_LAYOUT_CSR || !dia_ok) ? BGABP_LAYOUT_CSR : BGABP_LAYOUT_DIA;
    phase("validate + offsets");

    ck(cudaGetDevice(&device), "device");
    if (shared_stream) {
        st = shared_stream;
        own_stream = false;
    } else {
        ck(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate");
    }
    ck(cudaMallocHost((void**)&h_ctrl, sizeof(Ctrl)), "cudaMallocHost");
    d_ctrl = static_cast<Ctrl*>(dalloc(sizeof(Ctrl)));

    const bool host_build = getenv("BGABP_HOST_BUILD") != nullptr;  // cross-check of the device build
    use_ucsr_solve = getenv("BGABP_UCSR_SOLVE") != nullptr;         // A/B: the union-CSR solve loop
    if (layout == BGABP_LAYOUT_DIA) {
        S = (int)offs.size();
        std::memset(&dia, 0, sizeof(dia));
        dia.n = n;
        dia.S = S;
        dia.j0 = 0;
        dia.j1 = n;
        dia.gofs = 0;
        dia.nneg = (int)(std::lower_bound(offs.begin(), offs.end(), 0) - offs.begin());
        for (int s = 0; s < S; ++s) dia.off[s] = offs[s];
        for (int s = 0; s < S; ++s) dia.rev[s] = (int)(std::find(offs.begin(), offs.end(), -offs[s]) - offs.begin());
        nslots = (long long)S * n;
        if (host_build) {
            host_graph(ro_, ci_, v_);
            phase("host graph");
            build_dia_host();
        } else {
            build_dia_device(ro_, ci_, v_);
        }
        phase("DIA layout");
    } else {
        host_graph(ro_, ci_, v_);
        phase("host graph");
        build_ucsr_host();
        phase("UCSR layout");
    }
    // the SELL solve layout (general sparsity) pads chunks: its slot count can exceed nslots
    msg_cap = std::max<long long>(std::max(nslots, sell_slots), 1);
    for (int k = 0; k < 2; ++k) {
        d_msg[k] = static_cast<double2*>(dalloc(sizeof(double2) * (size_t)msg_cap));
        ck(cudaMemsetAsync(d_msg[k], 0, sizeof(double2) * (size_t)msg_cap, st), "memset");
    }
    const size_t vb = sizeof(double) * (size_t)std::max(n, 1);
    d_b = static_cast<double*>(dalloc(vb));
    d_x = static_cast<double*>(dalloc(vb));
    d_r = static_cast<double*>(dalloc(vb));
    d_e = static_cast<double*>(dalloc(vb));
    d_aux = static_cast<double*>(dalloc(vb));
    d_spread = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long) * 8 * kSpread));
    cur = 0;
    ck(cudaStreamSynchronize(st), "setup sync");
    phase("buffers");
}

// the matrix in HBM (row offsets, columns, values) and the DIA arrays derived from it on the device
void Engine::build_dia_device(const int* ro_, const int* ci_, const double* v_) {
    Phase phase;
    auto sync_phase = [&](const char* what) {
        if (!phase.on) return;
        ck(cudaStreamSynchronize(st), "sync");
        phase(what);
    };
    d_ro = static_cast<int*>(dalloc(sizeof(int) * ((size_t)n + 1)));
    d_ci = static_cast<int*>(dalloc(sizeof(int) * (size_t)std::max<long long>(nnz, 1)));
    d_val = static_cast<double*>(dalloc(sizeof(double) * (size_t)std::max<long long>(nnz, 1)));
    sync_phase("  dia: csr allocations");
    upload_host(d_ro, ro_, sizeof(int) * ((size_t)n + 1));
    upload_host(d_ci, ci_, sizeof(int) * (size_t)nnz);
    upload_host(d_val, v_, sizeof(double) * (size_t)nnz);
    sync_phase("  dia: csr upload");
    uint32_t* mask = static_cast<uint32_t*>(dalloc(sizeof(uint32_t) * (size_t)std::max(n, 1)));
    double* c = static_cast<double*>(dalloc(sizeof(double) * (size_t)std::max<long long>(nslots, 1)));
    double* rowv = static_cast<double*>(dalloc(sizeof(double) * (size_t)std::max<long long>(nslots, 1)));
    double* diag = static_cast<double*>(dalloc(sizeof(double) * (size_t)std::max(n, 1)));
    ck(cudaMemsetAsync(mask, 0, sizeof(uint32_t) * (size_t)std::max(n, 1), st), "memset");
    ck(cudaMemsetAsync(c, 0, sizeof(double) * (size_t)std::max<long long>(nslots, 1), st), "memset");
    ck(cudaMemsetAsync(rowv, 0, sizeof(double) * (size_t)std::max<long long>(nslots, 1), st), "memset");
    sync_phase("  dia: layout allocations");
    DiaOffs o{};
    o.S = S;
    for (int s = 0; s < S; ++s) {
        o.off[s] = dia.off[s];
        o.rev[s] = dia.rev[s];
    }
    const unsigned g = std::min<unsigned>(nblk_host(n), 148u * 16u);
    if (n > 0) k_dia_fill<<<g, 256, 0, st>>>(n, d_ro, d_ci, d_val, o, mask, c, rowv, diag);
    // 5-point grid in x-fastest order: offsets {-nx, -1, +1, +nx}, no edge wrapping across rows
    int gx = 0;
    if (S == 4 && dia.off[1] == -1 && dia.off[2] == 1 && dia.off[3] == -dia.off[0] && dia.off[3] > 1 &&
        n % dia.off[3] == 0)
        gx = dia.off[3];
    DiaFacts* d_f = static_cast<DiaFacts*>(dalloc(sizeof(DiaFacts)));
    DiaFacts hf{};
    for (int s = 0; s < kMaxDia; ++s) hf.cmin[s] = ~0ull;
    hf.dmin = ~0ull;
    ck(cudaMemcpyAsync(d_f, &hf, sizeof hf, cudaMemcpyHostToDevice, st), "H2D");
    if (n > 0) k_dia_facts<<<g, 256, 0, st>>>(n, S, mask, c, rowv, diag, gx, d_f);
    ck(cudaGetLastError(), "dia build");
    ck(cudaMemcpyAsync(&hf, d_f, sizeof hf, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "dia build sync");
    phase("  dia: fill + facts kernels");
    symmetric = hf.asym == 0u;
    grid5 = gx > 0 && hf.wrap == 0u;
    grid5_full = grid5 && nnz == 5ll * n - 2ll * gx - 2ll * (n / gx);
    dia.full5nx = dia.full5ny = 0;
    if (grid5 && symmetric && nnz == 5ll * n - 2ll * gx - 2ll * (n / gx) &&  // every in-grid entry present
        !getenv("BGABP_NO_FULL5")) {                                          // (A/B knob)
        dia.full5nx = gx;
        dia.full5ny = n / gx;
    }
    grid5_nx = gx;
    dia.uniform = 0;
    if (symmetric && n > 0) {  // constant-coefficient stencil (one bit pattern per slot and diagonal)
        bool unif = hf.dmin == hf.dmax;
        for (int s = 0; s < S; ++s) {
            const bool any = hf.cmin[s] != ~0ull;
            if (any && hf.cmin[s] != hf.cmax[s]) unif = false;
            dia.cu[s] = any ? bits2d(hf.cmin[s]) : 0.0;
        }
        dia.uniform = unif ? 1 : 0;
        dia.du = bits2d(hf.dmin);
    }
    dia.mask = mask;
    dia.c = c;
    dia.diag = diag;
    if (symmetric) {
        dia.rowv = c;
        dfree(rowv);
    } else {
        dia.rowv = rowv;
    }
    dfree(d_f);
}

// host copies of the matrix and its message-graph structure: canonical CSR, transpose positions
// (sparse.cpp:70-74), bit-symmetry, union neighbour lists (row j and column j, sorted)
void Engine::host_graph(const int* ro_, const int* ci_, const double* v_) {
    ro.assign(ro_, ro_ + n + 1);
    ci.resize(nnz);
    val.resize(nnz);
#pragma omp parallel for schedule(static)
    for (long long c0 = 0; c0 < nnz; c0 += (1 << 20)) {  // parallel copies of the CSR arrays
        const long long c1 = std::min<long long>(nnz, c0 + (1 << 20));
        std::memcpy(ci.data() + c0, ci_ + c0, sizeof(int) * (size_t)(c1 - c0));
        std::memcpy(val.data() + c0, v_ + c0, sizeof(double) * (size_t)(c1 - c0));
    }
    tpos.assign(nnz, -1);
    int sym = 1;
#pragma omp parallel for schedule(static) reduction(min : sym)
    for (int i = 0; i < n; ++i)
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            tpos[p] = find_pos(ci[p], i);
            if (tpos[p] < 0 || std::memcmp(&val[tpos[p]], &val[p], sizeof(double)) != 0) sym = 0;
        }
    symmetric = sym != 0;
    // union lists: row part in parallel; entries whose transpose is absent (one-way couplings)
    // add the reverse neighbour, then each list is sorted
    std::vector<int> ucount(n + 1, 0);
    long long oneway = 0;
#pragma omp parallel for schedule(static) reduction(+ : oneway)
    for (int i = 0; i < n; ++i) {
        int c = 0;
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            if (ci[p] == i) continue;
            ++c;
            if (tpos[p] < 0) ++oneway;
        }
        ucount[i + 1] = c;
    }
    if (oneway) {
        for (int i = 0; i < n; ++i)
            for (int p = ro[i]; p < ro[i + 1]; ++p)
                if (ci[p] != i && tpos[p] < 0) ucount[ci[p] + 1]++;  // j has neighbour i only via j->i
    }
    uptr.assign(n + 1, 0);
    for (int i = 0; i < n; ++i) uptr[i + 1] = uptr[i] + ucount[i + 1];
    unbr.assign(uptr[n], 0);
    std::vector<int> fill(uptr.begin(), uptr.end() - 1);
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        int f = fill[i];
        for (int p = ro[i]; p < ro[i + 1]; ++p)
            if (ci[p] != i) unbr[f++] = ci[p];
        fill[i] = f;
    }
    if (oneway) {
        for (int i = 0; i < n; ++i)
            for (int p = ro[i]; p < ro[i + 1]; ++p)
                if (ci[p] != i && tpos[p] < 0) unbr[fill[ci[p]]++] = i;
#pragma omp parallel for schedule(static)
        for (int i = 0; i < n; ++i) std::sort(unbr.begin() + uptr[i], unbr.begin() + uptr[i + 1]);
    }
    host_ready = true;
}

// the host copies on first use, from the device-resident CSR
void Engine::ensure_host() {
    if (host_ready) return;
    std::vector<int> hro((size_t)n + 1), hci((size_t)nnz);
    std::vector<double> hval((size_t)nnz);
    ck(cudaMemcpyAsync(hro.data(), d_ro, sizeof(int) * hro.size(), cudaMemcpyDeviceToHost, st), "D2H");
    if (nnz) {
        ck(cudaMemcpyAsync(hci.data(), d_ci, sizeof(int) * hci.size(), cudaMemcpyDeviceToHost, st), "D2H");
        ck(cudaMemcpyAsync(hval.data(), d_val, sizeof(double) * hval.size(), cudaMemcpyDeviceToHost, st), "D2H");
    }
    ck(cudaStreamSynchronize(st), "sync");
    const bool sym = symmetric;
    host_graph(hro.data(), hci.data(), hval.data());
    symmetric = sym;  // same value, recomputed
}

long long Engine::find_pos(int r, int c) const {
    const int* lo = ci.data() + ro[r];
    const int* hi = ci.data() + ro[r + 1];
    const int* it = std::lower_bound(lo, hi, c);
    return (it != hi && *it == c) ? (long long)(it - ci.data()) : -1;
}

void Engine::ensure_csr2slot() {
    if (d_csr2slot || nnz == 0) return;
    if (layout == BGABP_LAYOUT_DIA && d_ro) {
        d_csr2slot = static_cast<long long*>(dalloc(sizeof(long long) * (size_t)nnz));
        DiaOffs o{};
        o.S = S;
        for (int s = 0; s < S; ++s) {
            o.off[s] = dia.off[s];
            o.rev[s] = dia.rev[s];
        }
        k_dia_csr2slot<<<std::min<unsigned>(nblk_host(n), 148u * 16u), 256, 0, st>>>(n, d_ro, d_ci, o, d_csr2slot);
        ck(cudaGetLastError(), "csr2slot");
        return;
    }
    d_csr2slot = upload(csr2slot);
}

// host build of the DIA arrays (BGABP_HOST_BUILD=1): the cross-check of build_dia_device
void Engine::build_dia_host() {
    std::vector<double> diag(n);
    for (int i = 0; i < n; ++i) diag[i] = val[find_pos(i, i)];
    csr2slot.assign(nnz, -1);
    auto slot_of = [&](int off) {  // <= 8 sorted offsets: a linear scan beats a map by far
        int s = 0;
        while (dia.off[s] != off) ++s;
        return s;
    };
    std::vector<uint32_t> mask(n, 0u);
    std::vector<double> c((size_t)nslots, 0.0), rowv;
    if (!symmetric) rowv.assign((size_t)nslots, 0.0);
    // per node i, everything it owns: in-edges j->i from row i (slot of j-i), out-edges i->k
    // from column i (the transpose partner of a row entry, or a union neighbour outside row i)
#pragma omp parallel for schedule(static)
    for (int i = 0; i < n; ++i) {
        uint32_t mk = 0u;
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            const int j = ci[p];
            if (j == i) continue;
            const int si = slot_of(j - i);
            mk |= 1u << si;
            if (!symmetric) rowv[(size_t)si * n + i] = val[p];
            csr2slot[p] = (long long)si * n + i;
            if (tpos[p] >= 0) {
                mk |= 1u << (16 + si);
                c[(size_t)si * n + i] = val[tpos[p]];
            }
        }
        for (long long u = uptr[i]; u < uptr[i + 1]; ++u) {
            const int k = unbr[u];
            if (find_pos(i, k) >= 0) continue;  // already handled through row i
            const int sk = slot_of(k - i);
            mk |= 1u << (16 + sk);
            c[(size_t)sk * n + i] = val[find_pos(k, i)];
        }
        mask[i] = mk;
    }
    if (S == 4 && dia.off[1] == -1 && dia.off[2] == 1 && dia.off[3] == -dia.off[0] && dia.off[3] > 1 &&
        n % dia.off[3] == 0) {
        const int gx = dia.off[3];
        bool clean = true;
        for (int i = 0; i < n && clean; i += gx)
            if ((mask[i] & (2u | (2u << 16))) || (mask[i + gx - 1] & (4u | (4u << 16)))) clean = false;
        grid5 = clean;
        grid5_nx = gx;
    }
    dia.uniform = 0;
    if (symmetric && n > 0) {
        bool unif = true;
        for (int s2 = 0; s2 < S && unif; ++s2) {
            int first = -1;  // first node with this out-edge: the reference value
            for (int i = 0; i < n; ++i)
                if (mask[i] & (1u << (16 + s2))) {
                    first = i;
                    break;
                }
            dia.cu[s2] = first >= 0 ? c[(size_t)s2 * n + first] : 0.0;
            if (first < 0) continue;
            for (int i = first; i < n && unif; ++i)
                if ((mask[i] & (1u << (16 + s2))) &&
                    std::memcmp(&c[(size_t)s2 * n + i], &c[(size_t)s2 * n + first], sizeof(double)) != 0)
                    unif = false;
        }
        for (int i = 1; i < n && unif; ++i)
            if (std::memcmp(&diag[i], &diag[0], sizeof(double)) != 0) unif = false;
        dia.uniform = unif ? 1 : 0;
        dia.du = diag[0];
    }
    dia.mask = upload(mask);
    dia.c = upload(c);
    dia.rowv = symmetric ? dia.c : upload(rowv);
    dia.diag = upload(diag);
}

// union-CSR layout for general sparsity (more than 8 neighbour offsets)
void Engine::build_ucsr_host() {
    S = 0;
    const long long U = uptr[n];
    nslots = U;
    std::vector<double> diag(n);
    for (int i = 0; i < n; ++i) diag[i] = val[find_pos(i, i)];
    csr2slot.assign(nnz, -1);
    std::vector<uint8_t> flg(U, 0);
    std::vector<double> uc(U, 0.0), urow(U, 0.0);
    std::vector<int> urev(U, -1), undiag(n, 0);
    auto slot = [&](int j, int k) -> long long {  // slot of neighbour k in j's sorted list
        auto b = unbr.begin() + uptr[j], e = unbr.begin() + uptr[j + 1];
        return (long long)(std::lower_bound(b, e, k) - unbr.begin());
    };
    for (int j = 0; j < n; ++j) {
        undiag[j] = (int)(std::lower_bound(unbr.begin() + uptr[j], unbr.begin() + uptr[j + 1], j) -
                          (unbr.begin() + uptr[j]));
        for (long long s = uptr[j]; s < uptr[j + 1]; ++s) urev[s] = (int)slot(unbr[s], j);
    }
    for (int i = 0; i < n; ++i)
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            const int j = ci[p];
            if (j == i) continue;
            const long long si = slot(i, j), sj = slot(j, i);
            flg[si] |= 1;
            flg[sj] |= 2;
            uc[sj] = val[p];
            urow[si] = val[p];
            csr2slot[p] = si;
        }
    std::memset(&csr, 0, sizeof(csr));
    csr.n = n;
    csr.uptr = upload(uptr);
    csr.unbr = upload(unbr);
    csr.uflg = upload(flg);
    csr.uc = upload(uc);
    csr.urev = upload(urev);
    csr.undiag = upload(undiag);
    csr.diag = upload(diag);
    csr.ro = upload(ro);
    csr.ci = upload(ci);
    csr.val = upload(val);
    d_ro = const_cast<int*>(csr.ro);
    d_ci = const_cast<int*>(csr.ci);
    d_val = const_cast<double*>(csr.val);
    build_sell(flg, uc, urow, urev, csr.diag);
}


}  // namespace bgabp
