// SELL layout of the union message graph and the fused general-sparsity flood solve step
// (sell_kernels.cuh).  Built once per handle from the union-CSR lists (build.cu).
#include <algorithm>
#include <numeric>
#include <vector>

#include "engine.h"

namespace bgabp {

// flg / uc / urow / urev: the union-CSR slot arrays (build_ucsr_host): flags (bit 0 in-edge,
// bit 1 out-edge), A_kj, A_jk, and the union slot of j in k's list.
void Engine::build_sell(const std::vector<uint8_t>& flg, const std::vector<double>& uc, const std::vector<double>& urow,
                        const std::vector<int>& urev, const double* d_diag) {
    constexpr int kWindow = 1024;  // degree sort window (keeps chunk neighbourhoods local)
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
#pragma omp parallel for schedule(static)
    for (int w0 = 0; w0 < n; w0 += kWindow) {
        const int w1 = std::min(n, w0 + kWindow);
        std::stable_sort(perm.begin() + w0, perm.begin() + w1, [&](int a, int b) {
            return uptr[a + 1] - uptr[a] > uptr[b + 1] - uptr[b];
        });
    }
    const int C = (n + 31) / 32;
    std::vector<int> cnode((size_t)C * 32, -1), cwid(C, 0), chunk_of(n), lane_of(n);
    std::vector<long long> crow(C + 1, 0);
    for (int q = 0; q < n; ++q) {
        const int j = perm[q];
        cnode[q] = j;
        chunk_of[j] = q >> 5;
        lane_of[j] = q & 31;
        cwid[q >> 5] = std::max(cwid[q >> 5], uptr[j + 1] - uptr[j]);
    }
    for (int c = 0; c < C; ++c) crow[c + 1] = crow[c] + cwid[c];
    const long long slots = crow[C] * 32;
    if (slots > (long long)kSellSlot) throw InvalidArg("gabp: graph too large for the SELL solve layout");
    sell_slots = slots;
    auto pos = [&](int j, long long s) { return (crow[chunk_of[j]] + s) * 32 + lane_of[j]; };
    std::vector<unsigned> rev((size_t)std::max(slots, 1ll), 0u);
    std::vector<int> nbr((size_t)std::max(slots, 1ll), 0x7fffffff);
    std::vector<double> cout((size_t)std::max(slots, 1ll), 0.0), rowv(symmetric ? 0 : (size_t)std::max(slots, 1ll), 0.0);
#pragma omp parallel for schedule(dynamic, 4096)
    for (int j = 0; j < n; ++j)
        for (long long u = uptr[j]; u < uptr[j + 1]; ++u) {
            const long long p = pos(j, u - uptr[j]);
            const int k = unbr[u];
            unsigned f = 0;
            if (flg[u] & 1) f |= kSellIn;
            if (flg[u] & 2) f |= kSellOut | (unsigned)pos(k, urev[u] - uptr[k]);
            rev[p] = f;
            nbr[p] = k;
            cout[p] = uc[u];
            if (!symmetric) rowv[p] = urow[u];
        }
    std::vector<int> narrow, wide;  // chunk lists per bucket: <= 8 slot rows (register cached) / more
    for (int c = 0; c < C; ++c) (cwid[c] <= 8 ? narrow : wide).push_back(c);
    SellP P{};
    P.n = n;
    P.crow = upload(crow);
    P.cwid = upload(cwid);
    P.cnode = upload(cnode);
    P.rev = upload(rev);
    P.nbr = upload(nbr);
    P.cout = upload(cout);
    P.rowv = symmetric ? P.cout : upload(rowv);
    P.diag = d_diag;
    sell[0] = sell[1] = P;
    sell[0].chunks = upload(narrow);
    sell[0].nchunks = (int)narrow.size();
    sell[1].chunks = upload(wide);
    sell[1].nchunks = (int)wide.size();
    sell_ready = true;
}

// one fused solve step on the SELL layout: one launch per non-empty width bucket
void Engine::launch_sell_step(bool dl) {
    const bool damp = damping != 0.0;
    for (int q = 0; q < 2; ++q) {
        SellP P = sell[q];
        if (P.nchunks == 0) continue;
        P.damp = damping;
        P.undamp = 1.0 - damping;
        const unsigned g = nblk_host((long long)P.nchunks * 32);
        double2 *m0 = d_msg[0], *m1 = d_msg[1];
        double *x0 = d_xf, *x1 = d_xf + n;
#define SELL_LAUNCH(W_)                                                                                          \
    if (damp) {                                                                                                  \
        if (symmetric) {                                                                                         \
            if (dl) k_flood_solve_sell<W_, true, true, true><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
            else k_flood_solve_sell<W_, false, true, true><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
        } else {                                                                                                 \
            if (dl) k_flood_solve_sell<W_, true, false, true><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
            else k_flood_solve_sell<W_, false, false, true><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
        }                                                                                                        \
    } else if (symmetric) {                                                                                      \
        if (dl) k_flood_solve_sell<W_, true, true, false><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
        else k_flood_solve_sell<W_, false, true, false><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
    } else {                                                                                                     \
        if (dl) k_flood_solve_sell<W_, true, false, false><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
        else k_flood_solve_sell<W_, false, false, false><<<g, 256, 0, st>>>(P, solve_b, m0, m1, x0, x1, d_ctrl, d_spread); \
    }
        if (q == 0) {
            SELL_LAUNCH(8)
        } else {
            SELL_LAUNCH(0)
        }
#undef SELL_LAUNCH
    }
}

}  // namespace bgabp
