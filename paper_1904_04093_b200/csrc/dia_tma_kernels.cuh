// Fused DIA solve step with bulk-copy staging (the K1+K4 step of kernels.cuh, gabp.cpp:102-163 +
// 187-218): the node-major streams a step reads -- the S in-slot message arrays, the mask and b --
// are moved into shared memory by bulk asynchronous copies (cp.async.bulk, completion on an
// mbarrier) a tile ahead of their use, instead of per-thread loads that must be covered by
// resident warps.  Persistent warps: warp w of the grid walks tiles w, w + W, ... of kTmaTile
// consecutive nodes with two buffers, so one tile's copies are in flight while the previous one is
// evaluated.  The arithmetic per node is flood_solve_node's, in the same order: bit-identical.
// Everything else is as in k_flood_solve_dia: x(t-2) for the residual and (general coefficients)
// the coefficient columns through L1/L2, messages stored straight to the receivers' slots.
#pragma once

#include "kernels.cuh"
#include "sell_kernels.cuh"  // mbarrier / bulk-copy helpers

namespace bgabp {

constexpr int kTmaTile = 64;  // n must be a multiple of this (the largest tile below)

// one buffer of a warp tile of 32 * NPL nodes (NPL per lane): S message rows, mask, b
template <int S, int NPL>
__host__ __device__ constexpr unsigned dia_tma_buf_bytes() {
    return (unsigned)(32 * NPL * (S * 16 + 4 + 8));
}

template <int S, int NPL, int WPB>
__host__ __device__ constexpr size_t dia_tma_smem() {
    return (size_t)WPB * 2 * dia_tma_buf_bytes<S, NPL>() + (size_t)WPB * 2 * sizeof(unsigned long long);
}

// SYM / UNIF / DELTA as in k_flood_solve_dia (no sharding, peers or damping on this path).
// Requires n % kTmaTile == 0 (every tile full: the bulk copies stay 16-byte multiples).
template <int S, bool DELTA, bool SYM, bool UNIF, int WPB, int NPL = 2, int MINB = 2>
static __global__ void __launch_bounds__(32 * WPB, MINB) k_flood_solve_dia_tma(DiaP P, const double* __restrict__ b,
                                                                       double2* m0, double2* m1, double* x0,
                                                                       double* x1, Ctrl* ctrl,
                                                                       unsigned long long* spread) {
    extern __shared__ __align__(128) unsigned char smem[];
    if (ld_ctrl(&ctrl->done)) return;
    const int t = ld_ctrl(&ctrl->step);
    const double2* __restrict__ min = (t & 1) ? m0 : m1;
    double2* __restrict__ mout = (t & 1) ? m1 : m0;
    double* __restrict__ xw = ((t - 1) & 1) ? x1 : x0;        // x(t-1)
    const double* __restrict__ xr = ((t - 2) & 1) ? x1 : x0;  // x(t-2)
    const bool res = t >= 3;
    const int n = P.n;
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr unsigned kBuf = dia_tma_buf_bytes<S, NPL>();
    constexpr int T = 32 * NPL;  // nodes per tile
    unsigned char* wbase = smem + (size_t)wl * 2 * kBuf;
    unsigned long long* bars =
        reinterpret_cast<unsigned long long*>(smem + (size_t)WPB * 2 * kBuf) + 2 * wl;
    auto msg_of = [&](int buf) { return reinterpret_cast<double2*>(wbase + (size_t)buf * kBuf); };
    auto mask_of = [&](int buf) { return reinterpret_cast<uint32_t*>(msg_of(buf) + S * T); };
    auto b_of = [&](int buf) { return reinterpret_cast<double*>(mask_of(buf) + T); };
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    // (deriving the mask of a full 5-point grid from (row, column), as the one-thread-per-node
    // step does, measured 0.4 % slower here: the staged mask is nearly free)
    constexpr bool full5 = false;
    const int ntiles = n / T;
    const int stride = gridDim.x * WPB;
    auto issue = [&](int tile, int buf) {  // lane 0: the tile's streams into buffer `buf`
        const long long j0 = (long long)tile * T;
        mbar_arrive_tx(&bars[buf], full5 ? kBuf - T * 4u : kBuf);
#pragma unroll
        for (int s = 0; s < S; ++s)
            bulk_g2s(msg_of(buf) + s * T, min + (long long)s * n + j0, T * 16u, &bars[buf]);
        if (!full5) bulk_g2s(mask_of(buf), P.mask + j0, T * 4u, &bars[buf]);
        bulk_g2s(b_of(buf), b + j0, T * 8u, &bars[buf]);
    };
    double rabs = 0.0, dmax = 0.0;
    int tile = blockIdx.x * WPB + wl, buf = 0;
    unsigned phase[2] = {0u, 0u};
    if (tile < ntiles && lane == 0) issue(tile, 0);
    while (tile < ntiles) {
        const int nxt = tile + stride;
        if (nxt < ntiles && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of buf^1
            issue(nxt, buf ^ 1);
        }
        // the residual's x(t-2) gathers and (general coefficients) the coefficient columns do not
        // depend on the staged data: issue them before waiting (mask-independent, indices clamped)
        double xn[NPL][S], xjj[NPL], cc[NPL][S], dj[NPL];
#pragma unroll
        for (int h = 0; h < NPL; ++h) {
            const int j = tile * T + 32 * h + lane;
            xjj[h] = res ? __ldg(xr + j) : 0.0;
            dj[h] = UNIF ? P.du : __ldg(P.diag + j);
#pragma unroll
            for (int s = 0; s < S; ++s) {
                const int q = j + P.off[s];
                xn[h][s] = res ? __ldg(xr + (q < 0 ? 0 : (q >= n ? n - 1 : q))) : 0.0;
                cc[h][s] = UNIF ? P.cu[s]
                                : __ldg(SYM && s < P.nneg ? P.c + P.rev[s] * n + max(j + P.off[s], 0)
                                                          : P.c + s * n + j);
            }
        }
        mbar_wait(&bars[buf], phase[buf]);
        phase[buf] ^= 1u;
        const double2* sm = msg_of(buf);
        const uint32_t* smk = mask_of(buf);
        const double* sb = b_of(buf);
#pragma unroll
        for (int h = 0; h < NPL; ++h) {
            const int jl = 32 * h + lane;
            const int j = tile * T + jl;
            uint32_t mk;
            if (full5) {  // slots -nx, -1, +1, +nx; structurally symmetric
                const int row = j / P.full5nx, col = j - row * P.full5nx;
                const uint32_t e = (row > 0 ? 1u : 0u) | (col > 0 ? 2u : 0u) | (col < P.full5nx - 1 ? 4u : 0u) |
                                   (row < P.full5ny - 1 ? 8u : 0u);
                mk = e | (e << 16);
            } else {
                mk = smk[jl];
            }
            const double bj = sb[jl];
            double2 in[S];
            double c[S];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                in[s] = sm[s * T + jl];
                c[s] = (mk & (1u << (16 + s))) ? cc[h][s] : 0.0;
            }
            double sig = 0.0, acc = bj;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) sig = dadd(sig, dj[h]);
                if (mk & (1u << s)) {
                    acc = dadd(acc, in[s].y);
                    if (mk & (1u << (16 + s))) sig = dadd(sig, dmul(in[s].x, c[s]));
                }
            }
            if (P.nneg == S) sig = dadd(sig, dj[h]);
            if (t >= 2) {  // x-stage of sweep t-1
                xw[j] = ddiv(acc, sig);
                if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
            }
            if (res) {  // residual of x(t-2) in CSR order (sparse.cpp:108-114)
                double r = bj;
#pragma unroll
                for (int s = 0; s < S; ++s) {
                    if (s == P.nneg) r = dsub(r, dmul(dj[h], xjj[h]));
                    if (mk & (1u << s)) r = dsub(r, dmul(SYM ? c[s] : __ldg(P.rowv + s * n + j), xn[h][s]));
                }
                if (P.nneg == S) r = dsub(r, dmul(dj[h], xjj[h]));
                rabs = fmax(rabs, nan_skip_abs(r));
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (!(mk & (1u << (16 + s)))) continue;
                const double den = dsub(sig, dmul(in[s].x, c[s]));
                const int k = j + P.off[s];
                if (fabs(den) < kPivotFloor)
                    atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)k);
                const double nl = ddiv(-c[s], den);
                const double nm = dmul(nl, dsub(acc, in[s].y));
                double2* dst = mout + P.rev[s] * n + k;
                if (DELTA) {
                    const double2 o = min[P.rev[s] * n + k];
                    dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
                }
                *dst = make_double2(nl, nm);
            }
        }
        __syncwarp();  // every lane is done with `buf` before it is refilled
        buf ^= 1;
        tile = nxt;
    }
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
    if (DELTA) warp_max_spread(spread + (size_t)(4 + (t & 3)) * kSpread, dmax);
}

}  // namespace bgabp
