// Two flood solve iterations per launch on 5-point grids (temporal blocking, 2.5-D streaming).
//
// The fused solve step (kernels.cuh, k_flood_solve_dia) moves every message twice per sweep: the
// messages of sweep t-1 are read from HBM and those of sweep t written back.  Sweep t+1 at node j
// only needs sweep t's messages into j, which its neighbours compute from THEIR incoming
// messages of sweep t-1 -- so a block that owns a W x H tile of nodes can read the sweep-(t-1)
// messages of the tile plus a two-node halo, compute sweep t for that extended region on chip,
// and emit only sweep t+1's messages: one read and one write of the message state per TWO sweeps.
//
// Layout: thread c of a block owns grid column x = x0 - 2 + c (TPB = W + 4 columns) and walks
// the rows y0 - 2 .. y0 + H + 1.  At row step ya it
//   A. runs sweep t on node (x, ya): aggregation (= the x-stage x(t-1)), outgoing messages of
//      sweep t.  North-going messages stay in the thread's registers (they are consumed by the
//      same column one and two rows later), east/west-going ones go through shared memory;
//   B. runs sweep t+1 on node (x, ya - 1) from sweep t's messages: x(t), and for tile nodes the
//      outgoing messages of sweep t+1 (to HBM);
//   C. evaluates ||b - A x(t-1)|| on row ya - 1 and ||b - A x(t)|| on row ya - 2 (both need the
//      neighbours' x, which the extended region provides).
// Every node's arithmetic is the reference's (gabp.cpp:108-160, sparse.cpp:104-115) in the same
// order as k_flood_solve_dia, so the iterates are bit-identical.  Pivots and residual maxima are
// reported only by a node's owner tile.  Sweep t+1's messages go to the OTHER message buffer than
// the one read (halo reads of neighbouring tiles must still see sweep t-1), and x(k) lives in
// slot k % 4 of the x ring: the decision for iteration t-2 (taken after this launch) may still
// need x(t-2) and x(t-3) while this launch already wrote x(t-1) and x(t).
#pragma once

#include "kernels.cuh"

namespace bgabp {

constexpr int kXRing2 = 4;

// per-node operands of one grid node (UNIF: coefficients are kernel parameters)
template <bool UNIF, bool SYM>
struct Node5 {
    uint32_t mk;
    double bj, dj;
    double cc[UNIF ? 1 : 4];
    double rv[(UNIF || SYM) ? 1 : 4];
};

template <bool UNIF, bool SYM>
__device__ __forceinline__ void load_node5(const DiaP& P, const double* __restrict__ b, int n, int j,
                                           Node5<UNIF, SYM>& d) {
    d.mk = __ldg(P.mask + j);
    d.bj = __ldg(b + j);
    d.dj = UNIF ? P.du : __ldg(P.diag + j);
    if (!UNIF) {
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            // symmetric A: the negative-offset coefficients from the partner's positive slot
            // (same bits; the line is the neighbour's), as k_flood_solve_dia
            const double v = __ldg(SYM && s < 2 ? P.c + (size_t)P.rev[s] * n + max(j + P.off[s], 0)
                                                : P.c + (size_t)s * n + j);
            d.cc[s] = (d.mk & (1u << (16 + s))) ? v : 0.0;
            if (!SYM) d.rv[s] = __ldg(P.rowv + (size_t)s * n + j);
        }
    }
}

template <bool UNIF, bool SYM>
__device__ __forceinline__ double cc5(const DiaP& P, const Node5<UNIF, SYM>& d, int s) {
    if (UNIF) return (d.mk & (1u << (16 + s))) ? P.cu[s] : 0.0;
    return d.cc[s];
}
template <bool UNIF, bool SYM>
__device__ __forceinline__ double rv5(const DiaP& P, const Node5<UNIF, SYM>& d, int s) {
    if (UNIF || SYM) return cc5<UNIF, SYM>(P, d, s);
    return d.rv[s];
}

// aggregation of node d from its incoming messages in[4] (masked): sigma and the mean sum
// (gabp.cpp:108-119, diagonal at its CSR position between the negative and positive offsets)
template <bool UNIF, bool SYM>
__device__ __forceinline__ void aggregate5(const DiaP& P, const Node5<UNIF, SYM>& d, const double2 (&in)[4],
                                           double& sig, double& acc) {
    sig = 0.0;
    acc = d.bj;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (s == 2) sig = dadd(sig, d.dj);
        if (d.mk & (1u << s)) {
            acc = dadd(acc, in[s].y);
            if (d.mk & (1u << (16 + s))) sig = dadd(sig, dmul(in[s].x, cc5<UNIF, SYM>(P, d, s)));
        }
    }
}

// residual row b_j - sum_k A_jk x_k in CSR order (sparse.cpp:108-114); xn = (south, west, east, north)
template <bool UNIF, bool SYM>
__device__ __forceinline__ double residual5(const DiaP& P, const Node5<UNIF, SYM>& d, double xj, double xs, double xw,
                                            double xe, double xnn) {
    const double xn[4] = {xs, xw, xe, xnn};
    double r = d.bj;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (s == 2) r = dsub(r, dmul(d.dj, xj));
        if (d.mk & (1u << s)) r = dsub(r, dmul(rv5<UNIF, SYM>(P, d, s), xn[s]));
    }
    return r;
}

__device__ __forceinline__ void warp_max_spread2(unsigned long long* slots, double v, unsigned wid) {
    unsigned long long bits = __double_as_longlong(v);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        unsigned long long other = __shfl_xor_sync(0xffffffffu, bits, o);
        bits = other > bits ? other : bits;
    }
    if ((threadIdx.x & 31) == 0 && bits != 0ull) atomicMax(slots + (wid & (kSpread - 1)), bits);
}

// cp.async (LDGSTS): global -> shared without registers; each thread stages only its own column,
// so the staging needs no barrier (wait_group orders a thread's own copies)
__device__ __forceinline__ void cpa16(void* sm, const void* g) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(g));
}
__device__ __forceinline__ void cpa8(void* sm, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(g));
}
__device__ __forceinline__ void cpa4(void* sm, const void* g) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(sm)), "l"(g));
}
__device__ __forceinline__ void cpa_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cpa_wait() {
    asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

// per-row staging of one column's operands (ST rows in flight)
template <int TPB, int ST>
struct Stage5Base {
    double2 msg[ST][4][TPB];
    double bv[ST][TPB];
    uint32_t mk[ST][TPB];
};
template <bool UNIF, bool SYM, int TPB, int ST>
struct Stage5 : Stage5Base<TPB, ST> {  // variable coefficients, nonsymmetric
    double cf[ST][4][TPB];
    double dg[ST][TPB];
    double rw[ST][4][TPB];
};
template <int TPB, int ST>
struct Stage5<false, true, TPB, ST> : Stage5Base<TPB, ST> {  // variable coefficients, symmetric
    double cf[ST][4][TPB];
    double dg[ST][TPB];
};
template <bool SYM, int TPB, int ST>
struct Stage5<true, SYM, TPB, ST> : Stage5Base<TPB, ST> {};  // constant stencil: nothing else

template <bool UNIF, bool SYM, int TPB, int ST>
__device__ __forceinline__ void stage5_issue(Stage5<UNIF, SYM, TPB, ST>& S, int st, int c, const DiaP& P,
                                             const double* __restrict__ b, const double2* __restrict__ mi, int n,
                                             int j) {
#pragma unroll
    for (int s = 0; s < 4; ++s) cpa16(&S.msg[st][s][c], mi + (size_t)s * n + j);
    cpa8(&S.bv[st][c], b + j);
    cpa4(&S.mk[st][c], P.mask + j);
    if constexpr (!UNIF) {
        cpa8(&S.dg[st][c], P.diag + j);
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            cpa8(&S.cf[st][s][c], SYM && s < 2 ? P.c + (size_t)P.rev[s] * n + max(j + P.off[s], 0)
                                               : P.c + (size_t)s * n + j);
            if constexpr (!SYM) cpa8(&S.rw[st][s][c], P.rowv + (size_t)s * n + j);
        }
    }
}

template <bool UNIF, bool SYM, int TPB, int ST>
__device__ __forceinline__ void stage5_node(const Stage5<UNIF, SYM, TPB, ST>& S, int st, int c, const DiaP& P,
                                            Node5<UNIF, SYM>& d) {
    d.mk = S.mk[st][c];
    d.bj = S.bv[st][c];
    if constexpr (UNIF) {
        d.dj = P.du;
    } else {
        d.dj = S.dg[st][c];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            const double v = S.cf[st][s][c];
            d.cc[s] = (d.mk & (1u << (16 + s))) ? v : 0.0;
            if constexpr (!SYM) d.rv[s] = S.rw[st][s][c];
        }
    }
}

// ---- full-mask fast path: every in- and out-edge of the node exists (interior of a 5-point grid);
// the same operations in the same order as aggregate5 / residual5 / the edge loop, minus the mask
// logic (warp-uniform: taken only when every active lane of the warp qualifies)
constexpr uint32_t kFull5 = 0x000F000Fu;

// sigma, mean sum, x = acc / sigma (when want_x) and the four outgoing messages; den[] for pivots
__device__ __forceinline__ void node_full5(const double (&cf)[4], double dj, double bj, const double2 (&in)[4],
                                           bool want_x, double& sig, double& acc, double& xq, double (&den)[4],
                                           double2 (&g)[4]) {
    sig = dadd(0.0, dmul(in[0].x, cf[0]));
    acc = dadd(bj, in[0].y);
    acc = dadd(acc, in[1].y);
    sig = dadd(sig, dmul(in[1].x, cf[1]));
    sig = dadd(sig, dj);
    acc = dadd(acc, in[2].y);
    sig = dadd(sig, dmul(in[2].x, cf[2]));
    acc = dadd(acc, in[3].y);
    sig = dadd(sig, dmul(in[3].x, cf[3]));
    bool ok, o;
    xq = ddiv_fast(acc, sig, ok);
    ok = ok || !want_x;
    double q[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        den[s] = dsub(sig, dmul(in[s].x, cf[s]));
        q[s] = ddiv_fast(-cf[s], den[s], o);
        ok = ok && o;
    }
    if (!ok) {  // operands outside the fast path's range: the library division, same bits
        if (want_x) xq = ddiv(acc, sig);
#pragma unroll
        for (int s = 0; s < 4; ++s) q[s] = ddiv(-cf[s], den[s]);
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) g[s] = make_double2(q[s], dmul(q[s], dsub(acc, in[s].y)));
}

__device__ __forceinline__ double residual_full5(const double (&rv)[4], double dj, double bj, double xj, double xs,
                                                 double xw, double xe, double xn) {
    double r = dsub(bj, dmul(rv[0], xs));
    r = dsub(r, dmul(rv[1], xw));
    r = dsub(r, dmul(dj, xj));
    r = dsub(r, dmul(rv[2], xe));
    return dsub(r, dmul(rv[3], xn));
}

template <bool UNIF, bool SYM>
__device__ __forceinline__ void coef_full5(const Node5<UNIF, SYM>& d, const double (&cu)[4], double (&cf)[4],
                                           double (&rv)[4]) {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if constexpr (UNIF) {
            cf[s] = cu[s];
            rv[s] = cu[s];
        } else {
            cf[s] = d.cc[s];
            if constexpr (SYM) rv[s] = d.cc[s];
            else rv[s] = d.rv[s];
        }
    }
}

// One launch = solve iterations t and t+1 (t odd).  Messages of sweep 2m live in buffer m & 1.
// Row step ya (one barrier, at its end) does A on row ya, B on row ya - 2, the x(t-1) residual on
// row ya - 2 and the x(t) residual on row ya - 4: everything but A reads values produced at least
// two row steps earlier, so the division chains of A and B are independent within a step.

template <bool UNIF, bool SYM, int TPB, int ST>
struct Flood2 {
    // launch constants
    const DiaP& P;
    const double* __restrict__ b;
    const double2* __restrict__ mi;
    double2* __restrict__ mout;
    double* __restrict__ xa_out;
    double* __restrict__ xb_out;
    Ctrl* ctrl;
    Stage5<UNIF, SYM, TPB, ST>& SG;
    double2 (*sE)[TPB];
    double2 (*sW)[TPB];
    double (*sXA)[TPB];
    double (*sXB)[TPB];
    int n, nx, ny, t, c, x, y0, H, ylo, yhi;
    bool have_xa, colv, col1, coli;
    double cu[4];
    // per-column row queues
    Node5<UNIF, SYM> d0, d1, d2, d3, d4;
    double2 nq1, nq2, nq3, sq1;
    double xa1, xa2, xa3, xb1, xb2, xb3;
    double ra, rb;
    int sa, it;

    __device__ __forceinline__ void issue(int yy, int st) {
        if (colv && yy >= 0 && yy < ny) stage5_issue<UNIF, SYM, TPB, ST>(SG, st, c, P, b, mi, n, yy * nx + x);
        cpa_commit();
    }

    // STEADY: interior block, rows where every phase is active -- the range tests are compile-time
    template <bool STEADY>
    __device__ __forceinline__ void step(int ya) {
        const double2 z2 = make_double2(0.0, 0.0);
        const int r = it & 3, r2 = (it - 2) & 3;
        {
            const int yy = ya + ST - 1, sq = sa == 0 ? ST - 1 : sa - 1;
            if (yy <= y0 + H + 1) {
                if (STEADY) stage5_issue<UNIF, SYM, TPB, ST>(SG, sq, c, P, b, mi, n, yy * nx + x);
                else if (colv && yy >= 0 && yy < ny) stage5_issue<UNIF, SYM, TPB, ST>(SG, sq, c, P, b, mi, n, yy * nx + x);
            }
            cpa_commit();
            cpa_wait<ST - 1>();
        }
        // ---- A: sweep t on node (x, ya) ------------------------------------------------------
        double2 gS = z2, gW = z2, gE = z2, gN = z2;
        double xA = 0.0;
        const bool va = STEADY || (colv && ya >= 0 && ya < ny && ya <= y0 + H + 1);
        const bool fullA = __all_sync(0xffffffffu, !va || SG.mk[sa][c] == kFull5);
        if (va) {
            const int j = ya * nx + x;
            stage5_node<UNIF, SYM, TPB, ST>(SG, sa, c, P, d0);
            const bool own = STEADY ? coli : (coli && ya >= ylo && ya < yhi);
            double2 in[4];
#pragma unroll
            for (int s = 0; s < 4; ++s) in[s] = SG.msg[sa][s][c];
            double sig, acc, den[4];
            double2 g[4];
            if (fullA) {
                double cf[4], rv[4];
                coef_full5<UNIF, SYM>(d0, cu, cf, rv);
                node_full5(cf, d0.dj, d0.bj, in, have_xa, sig, acc, xA, den, g);
                const bool piv = fabs(den[0]) < kPivotFloor || fabs(den[1]) < kPivotFloor ||
                                 fabs(den[2]) < kPivotFloor || fabs(den[3]) < kPivotFloor;
                if (own && piv) {
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if (fabs(den[s]) < kPivotFloor)
                            atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                }
            } else {
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (!(d0.mk & (1u << s))) in[s] = z2;
                aggregate5<UNIF, SYM>(P, d0, in, sig, acc);
                double q[5];
                bool ok = true, o;
                q[4] = ddiv_fast(acc, sig, o);
                ok = ok && (o || !have_xa);
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    const double cs = cc5<UNIF, SYM>(P, d0, s);
                    den[s] = dsub(sig, dmul(in[s].x, cs));
                    q[s] = ddiv_fast(-cs, den[s], o);
                    ok = ok && (o || !(d0.mk & (1u << (16 + s))));
                }
                if (!ok) {
                    if (have_xa) q[4] = ddiv(acc, sig);
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if (d0.mk & (1u << (16 + s))) q[s] = ddiv(-cc5<UNIF, SYM>(P, d0, s), den[s]);
                }
                xA = q[4];
#pragma unroll
                for (int s = 0; s < 4; ++s) {
                    g[s] = z2;
                    if (!(d0.mk & (1u << (16 + s)))) continue;
                    if (own && fabs(den[s]) < kPivotFloor)
                        atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                    g[s] = make_double2(q[s], dmul(q[s], dsub(acc, in[s].y)));
                }
            }
            if (!have_xa) xA = 0.0;
            if (have_xa && own) {
                xa_out[j] = xA;
                if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
            }
            gS = g[0];
            gW = g[1];
            gE = g[2];
            gN = g[3];
        } else {
            d0.mk = 0u;
            d0.bj = 0.0;
        }
        sE[r][c] = gE;
        sW[r][c] = gW;
        sXA[r][c] = xA;
        // ---- B: sweep t+1 on node (x, yb), yb = ya - 2, from sweep t's messages ---------------
        const int yb = ya - 2;
        double xB = 0.0;
        const bool vb = STEADY ? col1 : (col1 && yb >= 0 && yb < ny && yb >= y0 - 1 && yb <= y0 + H);
        const bool fullB = __all_sync(0xffffffffu, !vb || d2.mk == kFull5);
        const bool ownB = STEADY ? coli : (coli && yb >= ylo && yb < yhi);
        if (vb) {
            const int j = yb * nx + x;
            double2 in[4];
            in[0] = nq3;                // from (x, yb - 1), north-going
            in[1] = sE[r2][c - 1];      // from (x - 1, yb)
            in[2] = sW[r2][c + 1];      // from (x + 1, yb)
            in[3] = sq1;                // from (x, yb + 1), south-going
            if (fullB) {
                double cf[4], rv[4], sig, acc, den[4];
                double2 g[4];
                coef_full5<UNIF, SYM>(d2, cu, cf, rv);
                node_full5(cf, d2.dj, d2.bj, in, true, sig, acc, xB, den, g);
                if (ownB) {
                    xb_out[j] = xB;
                    // 5-point DIA: slots (-nx, -1, +1, +nx), rev = (3, 2, 1, 0)
                    mout[(size_t)3 * n + j - nx] = g[0];
                    mout[(size_t)2 * n + j - 1] = g[1];
                    mout[(size_t)1 * n + j + 1] = g[2];
                    mout[j + nx] = g[3];
                    const bool piv = fabs(sig) < kPivotFloor || fabs(den[0]) < kPivotFloor ||
                                     fabs(den[1]) < kPivotFloor || fabs(den[2]) < kPivotFloor ||
                                     fabs(den[3]) < kPivotFloor;
                    if (piv) {
                        if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[t & 3], (unsigned long long)j);
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            if (fabs(den[s]) < kPivotFloor)
                                atomicMin(&ctrl->epiv[(t + 1) & 3],
                                          ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                    }
                }
            } else {
#pragma unroll
                for (int s = 0; s < 4; ++s)
                    if (!(d2.mk & (1u << s))) in[s] = z2;
                double sig, acc;
                aggregate5<UNIF, SYM>(P, d2, in, sig, acc);
                bool ok, o;
                xB = ddiv_fast(acc, sig, ok);
                if (ownB) {
                    double q[4], den[4];
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        const double cs = cc5<UNIF, SYM>(P, d2, s);
                        den[s] = dsub(sig, dmul(in[s].x, cs));
                        q[s] = ddiv_fast(-cs, den[s], o);
                        ok = ok && (o || !(d2.mk & (1u << (16 + s))));
                    }
                    if (!ok) {
                        xB = ddiv(acc, sig);
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            if (d2.mk & (1u << (16 + s))) q[s] = ddiv(-cc5<UNIF, SYM>(P, d2, s), den[s]);
                    }
                    xb_out[j] = xB;
                    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[t & 3], (unsigned long long)j);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if (!(d2.mk & (1u << (16 + s)))) continue;
                        const int k = j + P.off[s];
                        if (fabs(den[s]) < kPivotFloor)
                            atomicMin(&ctrl->epiv[(t + 1) & 3], ((unsigned long long)j << 32) | (unsigned)k);
                        mout[(size_t)P.rev[s] * n + k] = make_double2(q[s], dmul(q[s], dsub(acc, in[s].y)));
                    }
                } else if (!ok) {
                    xB = ddiv(acc, sig);
                }
            }
        }
        sXB[r][c] = xB;
        // ---- C: residuals of x(t-1) on row ya - 2 and of x(t) on row ya - 4 ----------------------
        if (have_xa && ownB) {
            const double xw = sXA[r2][c - 1], xe = sXA[r2][c + 1];
            double rr;
            if (d2.mk == kFull5) {
                double cf[4], rv[4];
                coef_full5<UNIF, SYM>(d2, cu, cf, rv);
                rr = residual_full5(rv, d2.dj, d2.bj, xa2, xa3, xw, xe, xa1);
            } else {
                rr = residual5<UNIF, SYM>(P, d2, xa2, xa3, xw, xe, xa1);
            }
            ra = fmax(ra, nan_skip_abs(rr));
        }
        const int yc = ya - 4;
        if (STEADY ? coli : (coli && yc >= ylo && yc < yhi)) {
            Node5<UNIF, SYM> dc;
            if constexpr (UNIF) {
                dc = d4;
            } else {
                load_node5<UNIF, SYM>(P, b, n, yc * nx + x, dc);
            }
            const double xw = sXB[r2][c - 1], xe = sXB[r2][c + 1];
            double rr;
            if (dc.mk == kFull5) {
                double cf[4], rv[4];
                coef_full5<UNIF, SYM>(dc, cu, cf, rv);
                rr = residual_full5(rv, dc.dj, dc.bj, xb2, xb3, xw, xe, xb1);
            } else {
                rr = residual5<UNIF, SYM>(P, dc, xb2, xb3, xw, xe, xb1);
            }
            rb = fmax(rb, nan_skip_abs(rr));
        }
        advance(gN, gS, xA, xB);
    }

    // shift the per-column row queues, then the step's barrier
    __device__ __forceinline__ void advance(double2 gN, double2 gS, double xA, double xB) {
        if constexpr (UNIF) {
            d4 = d3;
            d3 = d2;
        }
        d2 = d1;
        d1 = d0;
        nq3 = nq2;
        nq2 = nq1;
        nq1 = gN;
        sq1 = gS;
        xa3 = xa2;
        xa2 = xa1;
        xa1 = xA;
        xb3 = xb2;
        xb2 = xb1;
        xb1 = xB;
        sa = sa == ST - 1 ? 0 : sa + 1;
        ++it;
        __syncthreads();
    }
};

template <bool UNIF, bool SYM, int TPB, int MINB, int ST>
static __global__ void __launch_bounds__(TPB, MINB)
    k_flood2_grid5(DiaP P, int nx, int ny, int H, const double* __restrict__ b, double2* m0, double2* m1,
                   double* xring, Ctrl* ctrl, unsigned long long* spread) {
    constexpr int W = TPB - 4;
    if (ld_ctrl(&ctrl->done)) return;
    __shared__ double2 sE[4][TPB], sW[4][TPB];  // east- / west-going messages of sweep t, per row
    __shared__ double sXA[4][TPB], sXB[4][TPB];  // x(t-1) of row ya, x(t) of row ya - 2
    extern __shared__ __align__(16) unsigned char dsm[];
    const int t = ld_ctrl(&ctrl->step);
    const int n = P.n;
    const int x0 = blockIdx.x * W, y0 = blockIdx.y * H;
    Flood2<UNIF, SYM, TPB, ST> F{P,
                                 b,
                                 (((t - 1) >> 1) & 1) ? m1 : m0,  // sweep t-1
                                 (((t + 1) >> 1) & 1) ? m1 : m0,  // sweep t+1
                                 xring + (size_t)((t - 1) & (kXRing2 - 1)) * n,
                                 xring + (size_t)(t & (kXRing2 - 1)) * n,
                                 ctrl,
                                 *reinterpret_cast<Stage5<UNIF, SYM, TPB, ST>*>(dsm),
                                 sE,
                                 sW,
                                 sXA,
                                 sXB};
    F.n = n;
    F.nx = nx;
    F.ny = ny;
    F.t = t;
    F.c = threadIdx.x;
    F.x = x0 - 2 + F.c;
    F.y0 = y0;
    F.H = H;
    F.ylo = y0;
    F.yhi = min(y0 + H, ny);
    F.have_xa = t >= 2;  // x(t-1) is the x-stage of a sweep
    F.colv = F.x >= 0 && F.x < nx;
    F.col1 = F.colv && F.c >= 1 && F.c <= W + 2;
    F.coli = F.colv && F.c >= 2 && F.c < W + 2;
#pragma unroll
    for (int s = 0; s < 4; ++s) F.cu[s] = UNIF ? P.cu[s] : 0.0;
    F.d1.mk = F.d2.mk = F.d3.mk = F.d4.mk = 0u;
    F.d1.bj = F.d2.bj = F.d3.bj = F.d4.bj = 0.0;
    F.nq1 = F.nq2 = F.nq3 = F.sq1 = make_double2(0.0, 0.0);
    F.xa1 = F.xa2 = F.xa3 = F.xb1 = F.xb2 = F.xb3 = 0.0;
    F.ra = F.rb = 0.0;
    F.sa = 0;
    F.it = 0;
#pragma unroll
    for (int q = 0; q < ST - 1; ++q) F.issue(y0 - 2 + q, q);  // row ya + ST - 1 is issued at step ya
    const bool interior = x0 - 2 >= 0 && x0 + W + 1 < nx && y0 - 2 >= 0 && y0 + H + 1 < ny && H >= 2;
    if (interior) {
        for (int ya = y0 - 2; ya < y0 + 4; ++ya) F.template step<false>(ya);
        for (int ya = y0 + 4; ya <= y0 + H + 1; ++ya) F.template step<true>(ya);
        for (int ya = y0 + H + 2; ya <= y0 + H + 3; ++ya) F.template step<false>(ya);
    } else {
        for (int ya = y0 - 2; ya <= y0 + H + 3; ++ya) F.template step<false>(ya);
    }
    cpa_wait<0>();
    const unsigned wid = ((blockIdx.y * gridDim.x + blockIdx.x) * TPB + threadIdx.x) >> 5;
    if (F.have_xa) warp_max_spread2(spread + (size_t)((t - 1) & 3) * kSpread, F.ra, wid);
    warp_max_spread2(spread + (size_t)(t & 3) * kSpread, F.rb, wid);
}

}  // namespace bgabp

namespace bgabp {

// ---------------------------------------------------------------------------------------------
// Banded variant: the block (128 columns x R rows of threads) walks its tile R rows at a time in
// three fully parallel passes per band -- A (sweep t, rows ya), B (sweep t+1, rows ya - 2) and the
// x(t) residual (rows ya - 4) -- with the sweep-t messages and both x rings in shared memory
// (8-row rings, two barriers per band).  Each thread owns one node per pass: no per-thread row
// queues, so the register budget stays small and many more warps are resident than in the
// column-walking kernel above.  Same arithmetic, same ownership rules, bit-identical.
// ---------------------------------------------------------------------------------------------
template <bool UNIF, bool SYM, int R>
struct Band5Smem {
    double2 msg[8][4][128];  // outgoing sweep-t messages (S, W, E, N) of each ring row
    double xa[8][128];       // x(t-1)
    double xb[8][128];       // x(t)
};

template <bool UNIF, bool SYM, int R, int MINB>
static __global__ void __launch_bounds__(128 * R, MINB)
    k_flood2b_grid5(DiaP P, int nx, int ny, int H, const double* __restrict__ b, double2* m0, double2* m1,
                    double* xring, Ctrl* ctrl, unsigned long long* spread) {
    constexpr int TX = 128, W = TX - 4;
    if (ld_ctrl(&ctrl->done)) return;
    extern __shared__ __align__(16) unsigned char dsm[];
    Band5Smem<UNIF, SYM, R>& S = *reinterpret_cast<Band5Smem<UNIF, SYM, R>*>(dsm);
    const int t = ld_ctrl(&ctrl->step);
    const int n = P.n;
    const double2* __restrict__ mi = (((t - 1) >> 1) & 1) ? m1 : m0;  // sweep t-1
    double2* __restrict__ mout = (((t + 1) >> 1) & 1) ? m1 : m0;       // sweep t+1
    double* __restrict__ xa_out = xring + (size_t)((t - 1) & (kXRing2 - 1)) * n;
    double* __restrict__ xb_out = xring + (size_t)(t & (kXRing2 - 1)) * n;
    const bool have_xa = t >= 2;
    const int c = threadIdx.x, r = threadIdx.y;
    const int x0 = blockIdx.x * W, y0 = blockIdx.y * H;
    const int x = x0 - 2 + c;
    const bool colv = x >= 0 && x < nx;
    const bool col1 = colv && c >= 1 && c <= W + 2;
    const bool coli = colv && c >= 2 && c < W + 2;
    const int ylo = y0, yhi = min(y0 + H, ny);
    const int yfirst = y0 - 2;  // ring slot of row y: (y - yfirst) & 7
    double cu[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) cu[s] = UNIF ? P.cu[s] : 0.0;
    const double2 z2 = make_double2(0.0, 0.0);
    double ra = 0.0, rb = 0.0;

    // A-pass operands of the next band, prefetched into registers one band ahead
    auto load_a = [&](int ya, Node5<UNIF, SYM>& d, double2 (&in)[4]) {
        if (colv && ya >= 0 && ya < ny && ya <= y0 + H + 1) {
            const int j = ya * nx + x;
            load_node5<UNIF, SYM>(P, b, n, j, d);
#pragma unroll
            for (int s = 0; s < 4; ++s) in[s] = __ldg(mi + (size_t)s * n + j);
        } else {
            d.mk = 0u;
        }
    };
    Node5<UNIF, SYM> dn;
    double2 inn[4];
    load_a(yfirst + r, dn, inn);
    for (int ybase = yfirst; ybase <= y0 + H + 3; ybase += R) {
        const int ya = ybase + r;
        Node5<UNIF, SYM> da = dn;
        double2 ina[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) ina[s] = inn[s];
        load_a(ya + R, dn, inn);  // in flight during this band's three passes
        const int sa = (ya - yfirst) & 7;
        // ---- A: sweep t on node (x, ya) ------------------------------------------------------
        {
            double2 g[4] = {z2, z2, z2, z2};
            double xA = 0.0;
            const bool va = colv && ya >= 0 && ya < ny && ya <= y0 + H + 1;
            if (va) {
                const int j = ya * nx + x;
                const bool own = coli && ya >= ylo && ya < yhi;
                double sig, acc, den[4];
                if (da.mk == kFull5) {
                    double cf[4], rv[4];
                    coef_full5<UNIF, SYM>(da, cu, cf, rv);
                    node_full5(cf, da.dj, da.bj, ina, have_xa, sig, acc, xA, den, g);
                    if (own) {
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            if (fabs(den[s]) < kPivotFloor)
                                atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                    }
                } else {
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if (!(da.mk & (1u << s))) ina[s] = z2;
                    aggregate5<UNIF, SYM>(P, da, ina, sig, acc);
                    if (have_xa) xA = ddiv(acc, sig);
#pragma unroll
                    for (int s = 0; s < 4; ++s) {
                        if (!(da.mk & (1u << (16 + s)))) continue;
                        const double cs = cc5<UNIF, SYM>(P, da, s);
                        den[s] = dsub(sig, dmul(ina[s].x, cs));
                        if (own && fabs(den[s]) < kPivotFloor)
                            atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                        const double q = ddiv(-cs, den[s]);
                        g[s] = make_double2(q, dmul(q, dsub(acc, ina[s].y)));
                    }
                }
                if (!have_xa) xA = 0.0;
                if (have_xa && own) {
                    xa_out[j] = xA;
                    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
                }
            }
#pragma unroll
            for (int s = 0; s < 4; ++s) S.msg[sa][s][c] = g[s];
            S.xa[sa][c] = xA;
        }
        __syncthreads();
        // ---- B: sweep t+1 on node (x, yb), yb = ya - 2; x(t-1) residual there ----------------------
        const int yb = ya - 2;
        {
            const bool vb = col1 && yb >= 0 && yb < ny && yb >= y0 - 1 && yb <= y0 + H;
            const int sb = (yb - yfirst) & 7, sbm = (yb - 1 - yfirst) & 7, sbp = (yb + 1 - yfirst) & 7;
            double xB = 0.0;
            if (vb) {
                const int j = yb * nx + x;
                const bool own = coli && yb >= ylo && yb < yhi;
                Node5<UNIF, SYM> d;
                load_node5<UNIF, SYM>(P, b, n, j, d);
                double2 in[4];
                in[0] = S.msg[sbm][3][c];      // north-going from (x, yb - 1)
                in[1] = S.msg[sb][2][c - 1];   // east-going from (x - 1, yb)
                in[2] = S.msg[sb][1][c + 1];   // west-going from (x + 1, yb)
                in[3] = S.msg[sbp][0][c];      // south-going from (x, yb + 1)
                double sig, acc, den[4];
                double2 g[4];
                double cf[4], rv[4];
                const bool full = d.mk == kFull5;
                if (full) {
                    coef_full5<UNIF, SYM>(d, cu, cf, rv);
                    node_full5(cf, d.dj, d.bj, in, true, sig, acc, xB, den, g);
                } else {
#pragma unroll
                    for (int s = 0; s < 4; ++s)
                        if (!(d.mk & (1u << s))) in[s] = z2;
                    aggregate5<UNIF, SYM>(P, d, in, sig, acc);
                    xB = ddiv(acc, sig);
                }
                if (own) {
                    xb_out[j] = xB;
                    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[t & 3], (unsigned long long)j);
                    if (full) {
                        mout[(size_t)3 * n + j - nx] = g[0];
                        mout[(size_t)2 * n + j - 1] = g[1];
                        mout[(size_t)1 * n + j + 1] = g[2];
                        mout[j + nx] = g[3];
#pragma unroll
                        for (int s = 0; s < 4; ++s)
                            if (fabs(den[s]) < kPivotFloor)
                                atomicMin(&ctrl->epiv[(t + 1) & 3],
                                          ((unsigned long long)j << 32) | (unsigned)(j + P.off[s]));
                    } else {
#pragma unroll
                        for (int s = 0; s < 4; ++s) {
                            if (!(d.mk & (1u << (16 + s)))) continue;
                            const double cs = cc5<UNIF, SYM>(P, d, s);
                            const double dn2 = dsub(sig, dmul(in[s].x, cs));
                            const int k = j + P.off[s];
                            if (fabs(dn2) < kPivotFloor)
                                atomicMin(&ctrl->epiv[(t + 1) & 3], ((unsigned long long)j << 32) | (unsigned)k);
                            const double q = ddiv(-cs, dn2);
                            mout[(size_t)P.rev[s] * n + k] = make_double2(q, dmul(q, dsub(acc, in[s].y)));
                        }
                    }
                    if (have_xa) {  // residual of x(t-1) at (x, yb)
                        const double rr =
                            full ? residual_full5(rv, d.dj, d.bj, S.xa[sb][c], S.xa[sbm][c], S.xa[sb][c - 1],
                                                  S.xa[sb][c + 1], S.xa[sbp][c])
                                 : residual5<UNIF, SYM>(P, d, S.xa[sb][c], S.xa[sbm][c], S.xa[sb][c - 1],
                                                        S.xa[sb][c + 1], S.xa[sbp][c]);
                        ra = fmax(ra, nan_skip_abs(rr));
                    }
                }
            }
            S.xb[sb][c] = xB;
        }
        __syncthreads();
        // ---- C: residual of x(t) at (x, yc), yc = ya - 4 ------------------------------------------
        const int yc = ya - 4;
        if (coli && yc >= ylo && yc < yhi) {
            const int sc = (yc - yfirst) & 7, scm = (yc - 1 - yfirst) & 7, scp = (yc + 1 - yfirst) & 7;
            Node5<UNIF, SYM> d;
            load_node5<UNIF, SYM>(P, b, n, yc * nx + x, d);
            double rr;
            if (d.mk == kFull5) {
                double cf[4], rv[4];
                coef_full5<UNIF, SYM>(d, cu, cf, rv);
                rr = residual_full5(rv, d.dj, d.bj, S.xb[sc][c], S.xb[scm][c], S.xb[sc][c - 1], S.xb[sc][c + 1],
                                    S.xb[scp][c]);
            } else {
                rr = residual5<UNIF, SYM>(P, d, S.xb[sc][c], S.xb[scm][c], S.xb[sc][c - 1], S.xb[sc][c + 1],
                                          S.xb[scp][c]);
            }
            rb = fmax(rb, nan_skip_abs(rr));
        }
    }
    const unsigned tid = threadIdx.y * 128 + threadIdx.x;
    const unsigned wid = ((blockIdx.y * gridDim.x + blockIdx.x) * (128 * R) + tid) >> 5;
    if (have_xa) warp_max_spread2(spread + (size_t)((t - 1) & 3) * kSpread, ra, wid);
    warp_max_spread2(spread + (size_t)(t & 3) * kSpread, rb, wid);
}

}  // namespace bgabp
