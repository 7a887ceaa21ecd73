// Host side of the colour-compact red-black path (rb_kernels.cuh).
#include <algorithm>
#include <cstdlib>
#include <string>

#include "engine.h"

namespace bgabp {

// red_black_grid(nx, ny) on a DIA matrix whose neighbour offsets are exactly the 5-point stencil
// {-nx, -1, +1, +nx} (nx >= 2; odd nx: the colour is the index parity, even nx: one node of each
// colour per natural pair, rb_kernels.cuh)
bool Engine::rb_applicable(const bgabp_schedule& s) const {
    if (s.kind != BGABP_SCHED_RED_BLACK_GRID || layout != BGABP_LAYOUT_DIA || S != 4) return false;
    if (s.nx <= 1 || s.ny <= 0 || (long long)s.nx * s.ny != n) return false;
    return dia.off[0] == -s.nx && dia.off[1] == -1 && dia.off[2] == 1 && dia.off[3] == s.nx && dia.nneg == 2;
}

void Engine::rb_build(int nx, bool msgs) {
    if (rb_ready && rb_nx == nx) {
        if (msgs && !d_rbmsg) d_rbmsg = static_cast<double2*>(dalloc(sizeof(double2) * 4 * (size_t)std::max(n, 2)));
        return;
    }
    const int nR = (n + 1) / 2, nB = n / 2;
    rb.nx = nx;
    rb.nR = nR;
    rb.nB = nB;
    uint32_t* mR = static_cast<uint32_t*>(dalloc(sizeof(uint32_t) * std::max(nR, 1)));
    uint32_t* mB = static_cast<uint32_t*>(dalloc(sizeof(uint32_t) * std::max(nB, 1)));
    double* cR = static_cast<double*>(dalloc(sizeof(double) * 4 * std::max(nR, 1)));
    double* cB = static_cast<double*>(dalloc(sizeof(double) * 4 * std::max(nB, 1)));
    double *rR = nullptr, *rB = nullptr;
    if (!symmetric) {
        rR = static_cast<double*>(dalloc(sizeof(double) * 4 * std::max(nR, 1)));
        rB = static_cast<double*>(dalloc(sizeof(double) * 4 * std::max(nB, 1)));
    }
    double* dR = static_cast<double*>(dalloc(sizeof(double) * std::max(nR, 1)));
    double* dB = static_cast<double*>(dalloc(sizeof(double) * std::max(nB, 1)));
    k_rb_split<<<nblk_host(n), 256, 0, st>>>(n, nR, nx, dia.mask, dia.c, dia.rowv, dia.diag, mR, mB, cR, cB, rR, rB, dR,
                                             dB);
    ck(cudaGetLastError(), "rb split");
    rb.mask[0] = mR;
    rb.mask[1] = mB;
    rb.c[0] = cR;
    rb.c[1] = cB;
    rb.rowv[0] = symmetric ? cR : rR;
    rb.rowv[1] = symmetric ? cB : rB;
    rb.diag[0] = dR;
    rb.diag[1] = dB;
    rb.uniform = dia.uniform;
    for (int s = 0; s < 4; ++s) rb.cu[s] = dia.cu[s];
    rb.du = dia.du;
    if (msgs && !d_rbmsg) d_rbmsg = static_cast<double2*>(dalloc(sizeof(double2) * 4 * (size_t)std::max(n, 2)));
    rb_nx = nx;
    rb_ready = true;
}

// one red-black Gauss-Seidel pass (classic.cpp:16-30 in red_black_grid order) on the
// colour-compact coefficients: reds, then blacks, x in natural order, in place
void Engine::launch_gs_rb(const double* b, double* x) {
    if (n == 0) return;
    k_gs_rb_half<0><<<nblk_host(rb.nR), 256, 0, st>>>(rb, b, x, d_ctrl);
    if (rb.nB > 0) k_gs_rb_half<1><<<nblk_host(rb.nB), 256, 0, st>>>(rb, b, x, d_ctrl);
}

void Engine::launch_rb_sweep(const double* b, double* x, bool cold, bool delta, unsigned long long* dslot, int mode,
                             long long xstride) {
    if (n == 0) return;
    double2* mR = d_rbmsg;
    double2* mB = d_rbmsg + 4 * (size_t)rb.nR;
    const unsigned gr = nblk_host(rb.nR), gb = nblk_host(std::max(rb.nB, 1));
    if (rb.uniform && !delta) {  // constant stencil: no coefficient / diagonal loads
        if (cold)
            k_rb_half<0, true, false, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        else
            k_rb_half<0, false, false, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        if (rb.nB > 0) k_rb_half<1, false, false, true><<<gb, 256, 0, st>>>(rb, b, mB, mR, x, d_ctrl, dslot, mode, xstride);
        return;
    }
    if (delta) {
        if (cold)
            k_rb_half<0, true, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        else
            k_rb_half<0, false, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        if (rb.nB > 0) k_rb_half<1, false, true><<<gb, 256, 0, st>>>(rb, b, mB, mR, x, d_ctrl, dslot, mode, xstride);
    } else {
        if (cold)
            k_rb_half<0, true, false><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        else
            k_rb_half<0, false, false><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode, xstride);
        if (rb.nB > 0) k_rb_half<1, false, false><<<gb, 256, 0, st>>>(rb, b, mB, mR, x, d_ctrl, dslot, mode, xstride);
    }
}

// Record lambda^(s), sigma^(s) of a cold red-black start for s = 1..sweeps (rb_kernels.cuh).
// Returns false when the recursion breaks down within those sweeps (the caller then keeps the
// full sweep, which reports the breakdown exactly where the reference does).
bool Engine::rb_precompute(int sweeps) {
    if (rb_pre_failed) return false;
    if (rb_pre_sweeps >= sweeps) return true;
    const size_t nd = (size_t)std::max(n, 2);
    double* lam = static_cast<double*>(dalloc(sizeof(double) * 4 * nd));  // in-slot lambda, per colour
    for (int s = (int)rb_lamrec.size(); s < sweeps; ++s) {
        rb_lamrec.push_back(static_cast<double*>(dalloc(sizeof(double) * 4 * nd)));
        rb_sigrec.push_back(static_cast<double*>(dalloc(sizeof(double) * nd)));
    }
    reset_ctrl();
    const unsigned gr = nblk_host(rb.nR), gb = nblk_host(std::max(rb.nB, 1));
    double* lR = lam;
    double* lB = lam + 4 * (size_t)rb.nR;
    for (int s = 0; s < sweeps; ++s) {
        double* recR = rb_lamrec[s];
        double* recB = rb_lamrec[s] + 4 * (size_t)rb.nR;
        if (s == 0)
            k_rb_lambda_half<0, true><<<gr, 256, 0, st>>>(rb, lR, lB, recR, rb_sigrec[s], d_ctrl);
        else
            k_rb_lambda_half<0, false><<<gr, 256, 0, st>>>(rb, lR, lB, recR, rb_sigrec[s], d_ctrl);
        if (rb.nB > 0) k_rb_lambda_half<1, false><<<gb, 256, 0, st>>>(rb, lB, lR, recB, rb_sigrec[s] + rb.nR, d_ctrl);
    }
    ck(cudaGetLastError(), "rb precompute");
    read_ctrl();
    if (h_ctrl->opiv != kNone) {
        rb_pre_failed = true;
        return false;
    }
    rb_pre_sweeps = sweeps;
    return true;
}

// e from `sweeps` cold red-black mean-only sweeps on A e = r, then x += e (multigrid.cpp:180-188)
void Engine::rb_smooth_add(const double* r, int sweeps, double* x, bool r_compact) {
    if (n == 0 || sweeps <= 0) return;
    double* mR = reinterpret_cast<double*>(d_rbmsg);
    double* mB = mR + 4 * (size_t)rb.nR;
    const unsigned gr = nblk_host(rb.nR), gb = nblk_host(std::max(rb.nB, 1));
    const int rc = r_compact ? 1 : 0;  // r as launch_residual(..., rb_nx) wrote it
    // the last sweep's two phases in one launch (k_rb_mean_last_pair) on full grids
    static const bool pair_on = !(getenv("BGABP_RB_LAST_PAIR") && std::string(getenv("BGABP_RB_LAST_PAIR")) == "0");
    const bool full = pair_on && grid5_full && rb.nx >= 2 && rb.nB > 0;
    if (sweeps == 1 && full) {  // the whole call in one launch
        k_rb_mean_first_pair<true><<<gb, 256, 0, st>>>(rb, r, mR, rb_lamrec[0], rc, rb_sigrec[0], x);
        return;
    }
    int s0 = 0;
    if (sweeps >= 2 && rb.nB > 0) {  // sweep 1, both colours, one launch (k_rb_mean_first_pair)
        k_rb_mean_first_pair<false><<<gb, 256, 0, st>>>(rb, r, mR, rb_lamrec[0], rc, nullptr, nullptr);
        s0 = 1;
    }
    const bool last_pair = full && s0 == 1;
    for (int s = s0; s < sweeps; ++s) {
        if (last_pair && s + 1 == sweeps) {
            k_rb_mean_last_pair<<<gb, 256, 0, st>>>(rb, r, mR, rb_lamrec[s], rb_sigrec[s], x, rc);
            break;
        }
        const bool first = s == 0, last = s + 1 == sweeps;
        const double* recR = rb_lamrec[s];
        const double* recB = rb_lamrec[s] + 4 * (size_t)rb.nR;
        const double* sR = rb_sigrec[s];
        const double* sB = rb_sigrec[s] + rb.nR;
        if (first && last) k_rb_mean_half<0, true, true><<<gr, 256, 0, st>>>(rb, r, mR, mB, recR, sR, x, rc);
        else if (first) k_rb_mean_half<0, true, false><<<gr, 256, 0, st>>>(rb, r, mR, mB, recR, sR, x, rc);
        else if (last) k_rb_mean_half<0, false, true><<<gr, 256, 0, st>>>(rb, r, mR, mB, recR, sR, x, rc);
        else k_rb_mean_half<0, false, false><<<gr, 256, 0, st>>>(rb, r, mR, mB, recR, sR, x, rc);
        if (rb.nB > 0) {
            if (last) k_rb_mean_half<1, false, true><<<gb, 256, 0, st>>>(rb, r, mB, mR, recB, sB, x, rc);
            else k_rb_mean_half<1, false, false><<<gb, 256, 0, st>>>(rb, r, mB, mR, recB, sB, x, rc);
        }
    }
}

void Engine::rb_state(bool to_compact, double2* natural) {
    if (n == 0) return;
    if (to_compact)
        k_rb_convert<true><<<nblk_host(n), 256, 0, st>>>(n, rb.nR, rb.nx, natural, d_rbmsg);
    else
        k_rb_convert<false><<<nblk_host(n), 256, 0, st>>>(n, rb.nR, rb.nx, natural, d_rbmsg);
}

}  // namespace bgabp
