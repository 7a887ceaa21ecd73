// Host side of the colour-compact red-black path (rb_kernels.cuh).
#include <algorithm>

#include "engine.h"

namespace bgabp {

// red_black_grid(nx, ny) on a DIA matrix whose neighbour offsets are exactly the 5-point stencil
// {-nx, -1, +1, +nx} with nx odd: the colour is then the parity of the node index.
bool Engine::rb_applicable(const bgabp_schedule& s) const {
    if (s.kind != BGABP_SCHED_RED_BLACK_GRID || layout != BGABP_LAYOUT_DIA || S != 4) return false;
    if (s.nx <= 0 || s.ny <= 0 || (s.nx & 1) == 0 || (long long)s.nx * s.ny != n) return false;
    return dia.off[0] == -s.nx && dia.off[1] == -1 && dia.off[2] == 1 && dia.off[3] == s.nx && dia.nneg == 2;
}

void Engine::rb_build(int nx) {
    if (rb_ready && rb_nx == nx) return;
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
    k_rb_split<<<nblk_host(n), 256, 0, st>>>(n, nR, dia.mask, dia.c, dia.rowv, dia.diag, mR, mB, cR, cB, rR, rB, dR,
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
    if (!d_rbmsg) d_rbmsg = static_cast<double2*>(dalloc(sizeof(double2) * 4 * (size_t)std::max(n, 2)));
    rb_nx = nx;
    rb_ready = true;
}

void Engine::launch_rb_sweep(const double* b, double* x, bool cold, bool delta, unsigned long long* dslot, int mode) {
    if (n == 0) return;
    double2* mR = d_rbmsg;
    double2* mB = d_rbmsg + 4 * (size_t)rb.nR;
    const unsigned gr = nblk_host(rb.nR), gb = nblk_host(std::max(rb.nB, 1));
    if (delta) {
        if (cold)
            k_rb_half<0, true, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode);
        else
            k_rb_half<0, false, true><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode);
        if (rb.nB > 0) k_rb_half<1, false, true><<<gb, 256, 0, st>>>(rb, b, mB, mR, x, d_ctrl, dslot, mode);
    } else {
        if (cold)
            k_rb_half<0, true, false><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode);
        else
            k_rb_half<0, false, false><<<gr, 256, 0, st>>>(rb, b, mR, mB, x, d_ctrl, dslot, mode);
        if (rb.nB > 0) k_rb_half<1, false, false><<<gb, 256, 0, st>>>(rb, b, mB, mR, x, d_ctrl, dslot, mode);
    }
}

void Engine::rb_state(bool to_compact, double2* natural) {
    if (n == 0) return;
    if (to_compact)
        k_rb_convert<true><<<nblk_host(n), 256, 0, st>>>(n, rb.nR, natural, d_rbmsg);
    else
        k_rb_convert<false><<<nblk_host(n), 256, 0, st>>>(n, rb.nR, natural, d_rbmsg);
}

}  // namespace bgabp
