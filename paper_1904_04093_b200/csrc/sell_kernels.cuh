// Fused flood solve step for general sparsity (gabp.cpp:102-163 + 187-218 on matrices that are
// not a <= 8-offset stencil): the SELL layout of the union message graph.
//
// Layout (built on the host from the union-CSR lists, Engine::build_sell):
//   * nodes are grouped into chunks of 32 (one warp, one node per lane); inside windows of 1024
//     nodes they are stably sorted by degree first, so a chunk's lanes have similar degrees;
//   * chunk c holds cwid[c] slot rows; slot s of the node on lane l sits at (crow[c] + s) * 32 + l,
//     so a warp reading slot s of its 32 nodes touches 32 consecutive elements: every per-edge
//     array (messages, coefficients, indices) is read fully coalesced, the union-CSR layout's
//     per-thread strided reads are gone;
//   * a node's slots follow the sorted union of its row and column neighbours (CSR column
//     order), so the per-lane sums run in the reference's order and stay bit-identical;
//   * rev[p]: bit 31 = in-edge (A_jk structural: a message k -> j arrives in slot p and row j has
//     an entry), bit 30 = out-edge (A_kj structural: j sends to k), bits 0..29 = the slot of j in
//     k's list, where j's message to k is stored.  Padding slots are 0.
//   * the messages stay {lambda~, m} double2 per receiving slot (one 16-byte access per edge).
// Per edge one step reads 16 B of message, 8 B of coefficient (+8 B of row coefficient when A is
// not bit-symmetric), 8 B of index (rev + nbr), gathers x(t-2)_k for the residual (L2-resident
// for local graphs), and writes 16 B to the receiver's slot (the one scattered access).
#pragma once

#include "kernels.cuh"

namespace bgabp {

constexpr unsigned kSellIn = 1u << 31, kSellOut = 1u << 30, kSellSlot = (1u << 30) - 1;

// L2 cache policy "evict last" for operands a kernel reads twice, and read-only loads carrying it
__device__ __forceinline__ unsigned long long l2_evict_last_policy() {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    return pol;
}
__device__ __forceinline__ unsigned ldg_hint(const unsigned* p, unsigned long long pol) {
    unsigned v;
    asm("ld.global.nc.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ int ldg_hint(const int* p, unsigned long long pol) {
    int v;
    asm("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double ldg_hint(const double* p, unsigned long long pol) {
    double v;
    asm("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(v) : "l"(p), "l"(pol));
    return v;
}
__device__ __forceinline__ double2 ldg_hint(const double2* p, unsigned long long pol) {
    double2 v;
    asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(v.x), "=d"(v.y) : "l"(p), "l"(pol));
    return v;
}

struct SellP {
    int n;
    const int* chunks;      // chunk ids of the bucket this launch covers
    int nchunks;            // entries of `chunks`
    const long long* crow;  // [C] first slot row of chunk c
    const int* cwid;        // [C] slot rows of chunk c
    const int* cnode;       // [32 C] node on lane l of chunk c (-1: empty lane)
    const unsigned* rev;    // [slots] flags | target slot
    const int* nbr;         // [slots] neighbour k (0x7fffffff in padding)
    const double* cout;     // [slots] A_kj: the coefficient of j's message to k
    const double* rowv;     // [slots] A_jk: row j of A (the residual); == cout when A is symmetric
    const double* diag;     // [n]
    double damp, undamp;    // optional message damping (bgabp_set_damping)
};

// One warp = one chunk of 32 nodes.  W > 0: every chunk of the bucket has at most W slot rows
// and all per-slot operands stay in registers between the aggregation and the message stage;
// W == 0: any width, groups of 8 slots, the message stage re-reads its operands (L2 hits).
template <int W, bool DELTA, bool SYM, bool DAMP>
static __global__ void __launch_bounds__(256, 2) k_flood_solve_sell(SellP P, const double* __restrict__ b,
                                                                    double2* m0, double2* m1, double* x0,
                                                                    double* x1, Ctrl* ctrl,
                                                                    unsigned long long* spread) {
    if (ld_ctrl(&ctrl->done)) return;
    const int t = ld_ctrl(&ctrl->step);
    const double2* __restrict__ min = (t & 1) ? m0 : m1;
    double2* __restrict__ mout = (t & 1) ? m1 : m0;
    double* __restrict__ xw = ((t - 1) & 1) ? x1 : x0;        // x(t-1)
    const double* __restrict__ xr = ((t - 2) & 1) ? x1 : x0;  // x(t-2)
    const bool res = t >= 3;
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    double rabs = 0.0, dmax = 0.0;
    if (w < P.nchunks) {
        const int c = __ldg(P.chunks + w);
        const int wid = __ldg(P.cwid + c);
        const int j = __ldg(P.cnode + 32 * c + lane);
        const long long base = __ldg(P.crow + c) * 32 + lane;
        const int n = P.n;
        if (j >= 0) {
            const double dj = __ldg(P.diag + j), bj = __ldg(b + j);
            const double xj = res ? __ldg(xr + j) : 0.0;
            double sig = 0.0, acc = bj, r = bj;
            bool dsig = false, dres = false;
            // the diagonal enters both sums at its column position (before the first k > j)
            auto diag_before = [&](int k) {
                if (!dsig && k > j) {
                    sig = dadd(sig, dj);
                    dsig = true;
                }
                if (res && !dres && k > j) {
                    r = dsub(r, dmul(dj, xj));
                    dres = true;
                }
            };
            if constexpr (W > 0) {
                unsigned f[W];
                int kk[W];
                double2 v[W];
                double cs[W], rv[W], xk[W];
#pragma unroll
                for (int s = 0; s < W; ++s) {  // every load issued up front (padding slots are valid)
                    const bool on = s < wid;
                    const long long p = base + 32ll * s;
                    f[s] = on ? __ldg(P.rev + p) : 0u;
                    kk[s] = on ? __ldg(P.nbr + p) : 0x7fffffff;
                    v[s] = on ? __ldg(min + p) : make_double2(0.0, 0.0);
                    cs[s] = on ? __ldg(P.cout + p) : 0.0;
                    rv[s] = (!SYM && on) ? __ldg(P.rowv + p) : 0.0;
                }
#pragma unroll
                for (int s = 0; s < W; ++s) xk[s] = (res && (f[s] & kSellIn)) ? __ldg(xr + kk[s]) : 0.0;
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    if (s >= wid) break;
                    diag_before(kk[s]);
                    if (f[s] & kSellIn) {
                        acc = dadd(acc, v[s].y);
                        if (f[s] & kSellOut) sig = dadd(sig, dmul(v[s].x, cs[s]));
                        if (res) r = dsub(r, dmul(SYM ? cs[s] : rv[s], xk[s]));
                    }
                }
                diag_before(0x7fffffff);
                if (t >= 2) {  // x-stage of sweep t-1
                    xw[j] = ddiv(acc, sig);
                    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
                }
                if (res) rabs = nan_skip_abs(r);
#pragma unroll
                for (int s = 0; s < W; ++s) {
                    if (s >= wid) break;
                    if (!(f[s] & kSellOut)) continue;
                    const double2 vi = (f[s] & kSellIn) ? v[s] : make_double2(0.0, 0.0);
                    const double den = dsub(sig, dmul(vi.x, cs[s]));
                    if (fabs(den) < kPivotFloor)
                        atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)kk[s]);
                    double nl = ddiv(-cs[s], den);
                    double nm = dmul(nl, dsub(acc, vi.y));
                    const unsigned tgt = f[s] & kSellSlot;
                    if (DELTA || DAMP) {
                        const double2 o = min[tgt];
                        if (DAMP) {
                            const double2 q = damp_msg(nl, nm, o, P.damp, P.undamp);
                            nl = q.x;
                            nm = q.y;
                        }
                        if (DELTA) dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
                    }
                    mout[tgt] = make_double2(nl, nm);
                }
            } else {
                // any width: slots in groups of 8, every group's loads issued together; the
                // message stage reloads its operands (pass-1 loads carry an L2 evict-last policy,
                // so the reloads of a chunk normally hit L2)
                const unsigned long long pol = l2_evict_last_policy();
                for (int g0 = 0; g0 < wid; g0 += 8) {
                    unsigned f[8];
                    int kk[8];
                    double2 v[8];
                    double cs[8], rv[8], xk[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const bool on = g0 + q < wid;
                        const long long p = base + 32ll * (g0 + q);
                        f[q] = on ? ldg_hint(P.rev + p, pol) : 0u;
                        kk[q] = on ? ldg_hint(P.nbr + p, pol) : 0x7fffffff;
                        v[q] = on ? ldg_hint(min + p, pol) : make_double2(0.0, 0.0);
                        cs[q] = on ? ldg_hint(P.cout + p, pol) : 0.0;
                        rv[q] = (!SYM && on) ? __ldg(P.rowv + p) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) xk[q] = (res && (f[q] & kSellIn)) ? __ldg(xr + kk[q]) : 0.0;
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (g0 + q >= wid) break;
                        diag_before(kk[q]);
                        if (f[q] & kSellIn) {
                            acc = dadd(acc, v[q].y);
                            if (f[q] & kSellOut) sig = dadd(sig, dmul(v[q].x, cs[q]));
                            if (res) r = dsub(r, dmul(SYM ? cs[q] : rv[q], xk[q]));
                        }
                    }
                }
                diag_before(0x7fffffff);
                if (t >= 2) {
                    xw[j] = ddiv(acc, sig);
                    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
                }
                if (res) rabs = nan_skip_abs(r);
                for (int g0 = 0; g0 < wid; g0 += 8) {
                    unsigned f[8];
                    double2 v[8];
                    double cs[8];
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        const bool on = g0 + q < wid;
                        const long long p = base + 32ll * (g0 + q);
                        f[q] = on ? __ldg(P.rev + p) : 0u;
                        v[q] = on ? __ldg(min + p) : make_double2(0.0, 0.0);
                        cs[q] = on ? __ldg(P.cout + p) : 0.0;
                    }
#pragma unroll
                    for (int q = 0; q < 8; ++q) {
                        if (g0 + q >= wid) break;
                        if (!(f[q] & kSellOut)) continue;
                        const double2 vi = (f[q] & kSellIn) ? v[q] : make_double2(0.0, 0.0);
                        const double den = dsub(sig, dmul(vi.x, cs[q]));
                        if (fabs(den) < kPivotFloor)
                            atomicMin(&ctrl->epiv[t & 3],
                                      ((unsigned long long)j << 32) | (unsigned)__ldg(P.nbr + base + 32ll * (g0 + q)));
                        double nl = ddiv(-cs[q], den);
                        double nm = dmul(nl, dsub(acc, vi.y));
                        const unsigned tgt = f[q] & kSellSlot;
                        if (DELTA || DAMP) {
                            const double2 o = min[tgt];
                            if (DAMP) {
                                const double2 w2 = damp_msg(nl, nm, o, P.damp, P.undamp);
                                nl = w2.x;
                                nm = w2.y;
                            }
                            if (DELTA)
                                dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
                        }
                        mout[tgt] = make_double2(nl, nm);
                    }
                }
            }
        }
        (void)n;
    }
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
    if (DELTA) warp_max_spread(spread + (size_t)(4 + (t & 3)) * kSpread, dmax);
}

}  // namespace bgabp

namespace bgabp {

// ---- TMA-staged SELL step ---------------------------------------------------------------------
// The same step with the chunk's slot rows moved into shared memory by bulk asynchronous copies
// (cp.async.bulk, completion on an mbarrier) instead of per-lane loads held in registers: each
// warp walks its chunks (stride = all warps of the grid) with NB buffers: two = the copies of
// chunk i+1 in flight while chunk i is evaluated from shared memory; one = more warps per SM.  A chunk's rows of rev, nbr,
// messages and coefficients are contiguous in HBM (crow[c]*32 ... (crow[c]+wid)*32), so each is
// one bulk copy; registers no longer limit the bytes in flight (the register-cached kernel ran
// at 16 warps/SM, long-scoreboard bound).  Per slot row: rev 128 B + nbr 128 B + messages 512 B +
// coefficients 256 B = 1 KB of shared memory per buffer and row.
constexpr int kSellRowBytes = 32 * (4 + 4 + 16 + 8);

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_tx(unsigned long long* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, unsigned long long* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

template <int WMAX, int WPB, int NB, bool DELTA, bool SYM, bool DAMP>
static __global__ void __launch_bounds__(32 * WPB) k_flood_solve_sell_tma(SellP P, const double* __restrict__ b,
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
    const int wl = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // per warp: [2 buffers][rev | nbr | msg | cout] rows, then two mbarriers at the block's end
    unsigned char* wbase = smem + (size_t)wl * NB * WMAX * kSellRowBytes;
    unsigned long long* bars = reinterpret_cast<unsigned long long*>(smem + (size_t)WPB * NB * WMAX * kSellRowBytes) + 2 * wl;
    auto rev_of = [&](int buf) { return reinterpret_cast<unsigned*>(wbase + (size_t)buf * WMAX * kSellRowBytes); };
    auto nbr_of = [&](int buf) { return reinterpret_cast<int*>(rev_of(buf) + 32 * WMAX); };
    auto msg_of = [&](int buf) { return reinterpret_cast<double2*>(nbr_of(buf) + 32 * WMAX); };
    auto cs_of = [&](int buf) { return reinterpret_cast<double*>(msg_of(buf) + 32 * WMAX); };
    if (lane == 0) {
        mbar_init(&bars[0], 1);
        mbar_init(&bars[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    const int stride = gridDim.x * WPB;
    auto issue = [&](int idx, int buf) {  // lane 0: the chunk's rows into buffer `buf`
        const int c = __ldg(P.chunks + idx);
        const int wid = __ldg(P.cwid + c);
        const long long r0 = __ldg(P.crow + c) * 32;
        const unsigned rows = (unsigned)wid;
        mbar_arrive_tx(&bars[buf], rows * kSellRowBytes);
        if (rows) {
            bulk_g2s(rev_of(buf), P.rev + r0, rows * 128u, &bars[buf]);
            bulk_g2s(nbr_of(buf), P.nbr + r0, rows * 128u, &bars[buf]);
            bulk_g2s(msg_of(buf), min + r0, rows * 512u, &bars[buf]);
            bulk_g2s(cs_of(buf), P.cout + r0, rows * 256u, &bars[buf]);
        }
    };
    double rabs = 0.0, dmax = 0.0;
    int idx = blockIdx.x * WPB + wl, buf = 0;
    unsigned phase[2] = {0u, 0u};
    if (idx < P.nchunks && lane == 0) issue(idx, 0);
    while (idx < P.nchunks) {
        const int nxt = idx + stride;
        if (NB == 2 && nxt < P.nchunks && lane == 0) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // earlier generic reads of buf^1
            issue(nxt, buf ^ 1);
        }
        const int c = __ldg(P.chunks + idx);
        const int wid = __ldg(P.cwid + c);
        const int j = __ldg(P.cnode + 32 * c + lane);
        const long long base = __ldg(P.crow + c) * 32 + lane;
        mbar_wait(&bars[buf], phase[buf]);
        phase[buf] ^= 1u;
        const unsigned* sr = rev_of(buf);
        const int* sn = nbr_of(buf);
        const double2* sm = msg_of(buf);
        const double* sc = cs_of(buf);
        if (j >= 0) {
            const double dj = __ldg(P.diag + j), bj = __ldg(b + j);
            const double xj = res ? __ldg(xr + j) : 0.0;
            double sig = 0.0, acc = bj, r = bj;
            bool dsig = false, dres = false;
            for (int g0 = 0; g0 < wid; g0 += 8) {
                double xk[8], rv[8];
#pragma unroll
                for (int q = 0; q < 8; ++q) {  // the residual's gathers, issued together
                    const int s = g0 + q;
                    const bool in = s < wid && (sr[32 * s + lane] & kSellIn);
                    xk[q] = (res && in) ? __ldg(xr + sn[32 * s + lane]) : 0.0;
                    rv[q] = (!SYM && res && in) ? __ldg(P.rowv + base + 32ll * s) : 0.0;
                }
#pragma unroll
                for (int q = 0; q < 8; ++q) {
                    const int s = g0 + q;
                    if (s >= wid) break;
                    const unsigned f = sr[32 * s + lane];
                    const int k = sn[32 * s + lane];
                    if (k > j) {
                        if (!dsig) {
                            sig = dadd(sig, dj);
                            dsig = true;
                        }
                        if (res && !dres) {
                            r = dsub(r, dmul(dj, xj));
                            dres = true;
                        }
                    }
                    if (f & kSellIn) {
                        const double2 v = sm[32 * s + lane];
                        const double cs = sc[32 * s + lane];
                        acc = dadd(acc, v.y);
                        if (f & kSellOut) sig = dadd(sig, dmul(v.x, cs));
                        if (res) r = dsub(r, dmul(SYM ? cs : rv[q], xk[q]));
                    }
                }
            }
            if (!dsig) sig = dadd(sig, dj);
            if (res && !dres) r = dsub(r, dmul(dj, xj));
            if (t >= 2) {  // x-stage of sweep t-1
                xw[j] = ddiv(acc, sig);
                if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
            }
            if (res) rabs = fmax(rabs, nan_skip_abs(r));
            for (int s = 0; s < wid; ++s) {
                const unsigned f = sr[32 * s + lane];
                if (!(f & kSellOut)) continue;
                const double cs = sc[32 * s + lane];
                const double2 vi = (f & kSellIn) ? sm[32 * s + lane] : make_double2(0.0, 0.0);
                const double den = dsub(sig, dmul(vi.x, cs));
                if (fabs(den) < kPivotFloor)
                    atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)sn[32 * s + lane]);
                double nl = ddiv(-cs, den);
                double nm = dmul(nl, dsub(acc, vi.y));
                const unsigned tgt = f & kSellSlot;
                if (DELTA || DAMP) {
                    const double2 o = min[tgt];
                    if (DAMP) {
                        const double2 w2 = damp_msg(nl, nm, o, P.damp, P.undamp);
                        nl = w2.x;
                        nm = w2.y;
                    }
                    if (DELTA) dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
                }
                mout[tgt] = make_double2(nl, nm);
            }
        }
        __syncwarp();  // every lane is done with `buf` before it is refilled
        if (NB == 1 && nxt < P.nchunks && lane == 0) {  // one buffer: refill it now
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue(nxt, 0);
        }
        if (NB == 2) buf ^= 1;
        idx = nxt;
    }
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
    if (DELTA) warp_max_spread(spread + (size_t)(4 + (t & 3)) * kSpread, dmax);
}

template <int WMAX, int WPB, int NB>
constexpr size_t sell_tma_smem() {
    return (size_t)WPB * NB * WMAX * kSellRowBytes + (size_t)WPB * 2 * sizeof(unsigned long long);
}

}  // namespace bgabp
