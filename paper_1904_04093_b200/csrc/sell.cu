// SELL layout of the union message graph and the fused general-sparsity flood solve step
// (sell_kernels.cuh).  Built once per handle from the union-CSR lists (build.cu).
#include <algorithm>
#include <cstdlib>
#include <string>
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
    // chunk lists per width bucket: <= 8, <= 16, <= 32 slot rows (shared-memory staged kernels)
    // and wider (register kernel, any width)
    std::vector<int> lists[kSellBuckets];
    for (int c = 0; c < C; ++c) lists[cwid[c] <= 8 ? 0 : cwid[c] <= 16 ? 1 : cwid[c] <= 32 ? 2 : 3].push_back(c);
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
    for (int q = 0; q < kSellBuckets; ++q) {
        sell[q] = P;
        sell[q].chunks = upload(lists[q]);
        sell[q].nchunks = (int)lists[q].size();
    }
    sell_tma_setup();
    if (const char* e = getenv("BGABP_SELL_KIND")) sell_reg = std::string(e) == "reg";
    // measured on the B200 (config 4 on SELL): one buffer and twice the warps 0.997 ms per step,
    // two buffers 1.610 ms (long-scoreboard bound at 12 warps/SM)
    sell_variant = 1;
    if (const char* e = getenv("BGABP_SELL_TMA")) sell_variant = std::atoi(e) == 0 ? 0 : 1;
    sell_ready = true;
}

// TMA-staged kernels: (max rows, warps per block, buffers) per bucket variant, and persistent grids
// (BGABP_SELL_TMA=v selects variant v of every bucket: 0 = double-buffered, 1 = one buffer with
// twice the warps per block)
#define SELL_TMA_VARIANTS(X) X(8, 4, 2) X(16, 2, 2) X(32, 1, 2) X(8, 8, 1) X(16, 4, 1) X(32, 2, 1)
template <int WMAX, int WPB, int NB>
static void sell_tma_attr(int& blocks_per_sm) {
    const size_t smem = sell_tma_smem<WMAX, WPB, NB>();
#define SET_ATTR(D_, S_, M_)                                                                                     \
    ck(cudaFuncSetAttribute(k_flood_solve_sell_tma<WMAX, WPB, NB, D_, S_, M_>,                                   \
                            cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),                             \
       "sell smem");
    SET_ATTR(false, false, false) SET_ATTR(true, false, false) SET_ATTR(false, true, false) SET_ATTR(true, true, false)
    SET_ATTR(false, false, true) SET_ATTR(true, false, true) SET_ATTR(false, true, true) SET_ATTR(true, true, true)
#undef SET_ATTR
    ck(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, k_flood_solve_sell_tma<WMAX, WPB, NB, false, true, false>,
                                                     32 * WPB, smem),
       "occupancy");
    blocks_per_sm = std::max(blocks_per_sm, 1);
}

void Engine::sell_tma_setup() {
    int sms = 148;
    ck(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    int q = 0;
#define SETUP(W_, P_, N_)                                                                                        \
    {                                                                                                            \
        int bps = 1;                                                                                             \
        sell_tma_attr<W_, P_, N_>(bps);                                                                          \
        sell_grid[q++] = sms * bps;                                                                              \
    }
    SELL_TMA_VARIANTS(SETUP)
#undef SETUP
}

template <int WMAX, int WPB, int NB>
static void launch_tma(const SellP& P, unsigned grid, bool dl, bool sym, bool damp, const double* b, double2* m0,
                       double2* m1, double* x0, double* x1, Ctrl* ctrl, unsigned long long* spread,
                       cudaStream_t st) {
    const unsigned g = std::min<unsigned>(grid, (unsigned)((P.nchunks + WPB - 1) / WPB));
    const size_t smem = sell_tma_smem<WMAX, WPB, NB>();
#define TMA_K(D_, S_, M_) \
    k_flood_solve_sell_tma<WMAX, WPB, NB, D_, S_, M_><<<g, 32 * WPB, smem, st>>>(P, b, m0, m1, x0, x1, ctrl, spread)
    if (damp) {
        if (sym) { if (dl) TMA_K(true, true, true); else TMA_K(false, true, true); }
        else { if (dl) TMA_K(true, false, true); else TMA_K(false, false, true); }
    } else {
        if (sym) { if (dl) TMA_K(true, true, false); else TMA_K(false, true, false); }
        else { if (dl) TMA_K(true, false, false); else TMA_K(false, false, false); }
    }
#undef TMA_K
}

// one fused solve step on the SELL layout: one launch per non-empty width bucket
void Engine::launch_sell_step(bool dl) {
    const bool damp = damping != 0.0;
    for (int q = 0; q < kSellBuckets; ++q) {
        SellP P = sell[q];
        if (P.nchunks == 0) continue;
        P.damp = damping;
        P.undamp = 1.0 - damping;
        const unsigned g = nblk_host((long long)P.nchunks * 32);
        double2 *m0 = d_msg[0], *m1 = d_msg[1];
        double *x0 = d_xf, *x1 = d_xf + n;
        // shared-memory staged (bulk async copies) for chunks of <= 8 slot rows; wider chunks run
        // the register kernel (a random 4M-node graph, chunks of 9-32 rows: 2.70 vs 2.89 ms per
        // step staged -- 16 KB of staging per warp leaves 12 warps per SM for its random gathers)
        if (!sell_reg && q < 1) {
#define TMA_L(W_, P_, N_, G_) \
    launch_tma<W_, P_, N_>(P, sell_grid[G_], dl, symmetric, damp, solve_b, m0, m1, x0, x1, d_ctrl, d_spread, st)
            if (sell_variant == 0) {
                if (q == 0) TMA_L(8, 4, 2, 0);
                else if (q == 1) TMA_L(16, 2, 2, 1);
                else TMA_L(32, 1, 2, 2);
            } else {
                if (q == 0) TMA_L(8, 8, 1, 3);
                else if (q == 1) TMA_L(16, 4, 1, 4);
                else TMA_L(32, 2, 1, 5);
            }
#undef TMA_L
            continue;
        }
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
