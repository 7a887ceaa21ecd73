// Colour-compact red-black GaBP sweep for 5-point grids, SURVEY.md §2.2 K2 specialised.
//
// With nx odd (every multigrid level: 2^J - 1 points per axis) the red-black colour (ix+iy) mod 2
// equals the parity of the natural index g, so red node q is g = 2q and black node q is g = 2q+1.
// With nx even each natural pair (2q, 2q+1) holds one node of each colour, which one depending on
// the row.  Either way node g has compact index g >> 1 in its colour, so a neighbour g + off
// sits at (g + off) >> 1 in the other colour's numbering.
// Messages and coefficients are stored per colour, slot-major ([4][n_colour]), so the red phase
// and the black phase each read and write fully coalesced lines instead of every other element
// of the natural-order arrays (the generic level kernel wastes half of every 32-byte sector).
// Arithmetic is the reference's in-place visit (gabp.cpp:49-100) in natural CSR column order
// (S, W, diagonal, E, N); the colour-grouped order of red_black_grid (schedule.cpp:78-83) visits
// reds by ascending g, then blacks, so a node's pivot position is q (red) or n_red + q (black).
#pragma once

#include "kernels.cuh"

namespace bgabp {

struct RbP {
    int nx, nR, nB;
    const uint32_t* mask[2];  // [colour] DIA mask bits of the natural slots (-nx, -1, +1, +nx)
    const double* c[2];       // [colour][4][n_c] A_{k,j} of the node's outgoing message per slot
    const double* rowv[2];    // [colour][4][n_c] A_{j,k} (residual / GS), == c if symmetric
    const double* diag[2];    // [colour][n_c]
    int uniform;              // constant stencil (DiaP::uniform): cu / du replace c / diag
    double cu[4], du;
};

// Even nx: natural pair (2q, 2q+1) lies in one row and holds one red and one black node, so the
// compact index of natural node g is g >> 1 for both colours and for both parities of nx; which
// element of the pair has colour C depends on the row when nx is even.
__device__ __forceinline__ int rb_nat(const RbP& P, int q, int colour) {
    return 2 * q + ((P.nx & 1) ? colour : ((colour + (2 * q) / P.nx) & 1));
}
__host__ __device__ __forceinline__ int rb_colour(int g, int nx) { return (nx & 1) ? (g & 1) : ((g + g / nx) & 1); }

__device__ __forceinline__ int rb_other(int g, int s, int nx) {
    // compact index (in the other colour) of neighbour slot s of natural node g
    const int off = s == 0 ? -nx : s == 1 ? -1 : s == 2 ? 1 : nx;
    return (g + off) >> 1;
}

// One colour phase of a red-black sweep.  COLD: first sweep of a cold start on the red phase
// (every in-message is still zero, so none is read and no buffer has to be cleared).
template <int COLOUR, bool COLD, bool DELTA, bool UNIF = false>
static __global__ void __launch_bounds__(256) k_rb_half(RbP P, const double* __restrict__ b, double2* mine,
                                                       double2* other, double* __restrict__ x, Ctrl* ctrl,
                                                       unsigned long long* dslot, int mode, long long xstride = 0) {
    if (mode == MODE_SOLVE && ld_ctrl(&ctrl->done)) return;
    if (block_sees_failure(ctrl)) return;
    if (mode == MODE_SOLVE && xstride && (ld_ctrl(&ctrl->step) & 1)) x += xstride;  // x(t) in ring slot t & 1
    const int nc = COLOUR == 0 ? P.nR : P.nB, no = COLOUR == 0 ? P.nB : P.nR;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    double dmax = 0.0;
    if (q < nc) {
        const int g = rb_nat(P, q, COLOUR);
        const uint32_t mk = P.mask[COLOUR][q];
        const double dj = UNIF ? P.du : P.diag[COLOUR][q];
        double sig = 0.0, acc = b[g];
        double2 in[4];
        double cc[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            in[s] = make_double2(0.0, 0.0);
            cc[s] = 0.0;
            if (!COLD && (mk & (1u << s))) in[s] = mine[s * nc + q];
            if (mk & (1u << (16 + s))) cc[s] = UNIF ? P.cu[s] : __ldg(P.c[COLOUR] + s * nc + q);
        }
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (s == 2) sig = dadd(sig, dj);
            if (mk & (1u << s)) {
                acc = dadd(acc, in[s].y);
                if (mk & (1u << (16 + s))) sig = dadd(sig, dmul(in[s].x, cc[s]));
            }
        }
        const unsigned long long pk = (unsigned long long)(COLOUR == 0 ? q : P.nR + q) << 32;
        if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->opiv, pk);
        x[g] = ddiv(acc, sig);
        const int off[4] = {-P.nx, -1, 1, P.nx};
#pragma unroll
        for (int s = 0; s < 4; ++s) {
            if (!(mk & (1u << (16 + s)))) continue;
            const double den = dsub(sig, dmul(in[s].x, cc[s]));
            if (fabs(den) < kPivotFloor) atomicMin(&ctrl->opiv, pk | (unsigned)(g + off[s] + 1));
            const double nl = ddiv(-cc[s], den);
            const double nm = dmul(nl, dsub(acc, in[s].y));
            double2* dst = other + (3 - s) * no + rb_other(g, s, P.nx);
            if (DELTA) {
                const double2 o = *dst;
                dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
            }
            *dst = make_double2(nl, nm);
        }
    }
    if (DELTA) warp_max_commit(dslot, dmax);
}

// One colour of a red-black Gauss-Seidel pass (classic.cpp:16-30, gs_pass in red_black_grid
// order): x_g = (b_g - sum_{k != g} A_gk x_k) / A_gg with the row in CSR column order.  Row
// coefficients and the diagonal come from the colour-compact copies (coalesced); x stays in
// natural order, where a warp's 32 nodes and their 64 horizontal neighbours share the same
// 512 bytes.  Zero diagonal: the visit position (reds first, ascending) into opiv, like the level
// kernel.
template <int COLOUR>
static __global__ void __launch_bounds__(256) k_gs_rb_half(RbP P, const double* __restrict__ b, double* x,
                                                          Ctrl* ctrl) {
    if (ctrl->opiv != kNone) return;
    const int nc = COLOUR == 0 ? P.nR : P.nB, n = P.nR + P.nB;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nc) return;
    const int g = rb_nat(P, q, COLOUR);
    const uint32_t mk = P.mask[COLOUR][q];
    const int off[4] = {-P.nx, -1, 1, P.nx};
    double cv[4], xv[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // every load up front; the mask selects the terms
        const int k = g + off[s];
        cv[s] = __ldg(P.rowv[COLOUR] + s * nc + q);
        xv[s] = x[k < 0 ? 0 : (k >= n ? n - 1 : k)];
    }
    const double d = __ldg(P.diag[COLOUR] + q);
    double acc = b[g];
#pragma unroll
    for (int s = 0; s < 4; ++s)
        if (mk & (1u << s)) acc = dsub(acc, dmul(cv[s], xv[s]));
    if (d == 0.0) atomicMin(&ctrl->opiv, (unsigned long long)(COLOUR == 0 ? q : P.nR + q) << 32);
    x[g] = ddiv(acc, d);
}

// colour-split copies of the DIA arrays (natural slots -nx, -1, +1, +nx)
static __global__ void k_rb_split(int n, int nR, int nx, const uint32_t* __restrict__ mask, const double* __restrict__ c,
                                  const double* __restrict__ rowv, const double* __restrict__ diag, uint32_t* mR,
                                  uint32_t* mB, double* cR, double* cB, double* rR, double* rB, double* dR, double* dB) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const int q = g >> 1, nB = n - nR;
    const bool red = rb_colour(g, nx) == 0;
    (red ? mR : mB)[q] = mask[g];
    (red ? dR : dB)[q] = diag[g];
    for (int s = 0; s < 4; ++s) {
        (red ? cR : cB)[s * (red ? nR : nB) + q] = c[(size_t)s * n + g];
        if (rR) (red ? rR : rB)[s * (red ? nR : nB) + q] = rowv[(size_t)s * n + g];
    }
}

// ---------------------------------------------------------------------------------------------
// Cold smoothing with precomputed precisions ("optimisations that preserve bitwise
// results"): Hierarchy::smooth restarts the messages at zero on every call (multigrid.cpp:180),
// and the lambda recursion never reads the means, so lambda^(s) and sigma^(s) of sweep s of a
// cold start depend on A alone.  They are recorded once per level (k_rb_lambda_half) and every
// smoothing sweep then moves only the means: per edge 8 B in, 8 B lambda, 8 B out instead of
// 16 + 8 + 16, with the values the reference computes bit for bit.
// ---------------------------------------------------------------------------------------------

// one colour phase of a cold lambda-only red-black sweep; records sigma of every visited node
// (the x-stage divisor) and the lambda of every outgoing message, source-major
template <int COLOUR, bool COLD>
static __global__ void __launch_bounds__(256) k_rb_lambda_half(RbP P, double* lam_mine, double* lam_other,
                                                              double* __restrict__ lam_rec,
                                                              double* __restrict__ sig_rec, Ctrl* ctrl) {
    const int nc = COLOUR == 0 ? P.nR : P.nB, no = COLOUR == 0 ? P.nB : P.nR;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nc) return;
    const int g = rb_nat(P, q, COLOUR);
    const uint32_t mk = P.mask[COLOUR][q];
    double sig = 0.0, in[4], cc[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        in[s] = (!COLD && (mk & (1u << s))) ? lam_mine[s * nc + q] : 0.0;
        cc[s] = (mk & (1u << (16 + s))) ? __ldg(P.c[COLOUR] + s * nc + q) : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (s == 2) sig = dadd(sig, P.diag[COLOUR][q]);
        if ((mk & (1u << s)) && (mk & (1u << (16 + s)))) sig = dadd(sig, dmul(in[s], cc[s]));
    }
    sig_rec[q] = sig;
    const unsigned long long pk = (unsigned long long)(COLOUR == 0 ? q : P.nR + q) << 32;
    if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->opiv, pk);
    const int off[4] = {-P.nx, -1, 1, P.nx};
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        double nl = 0.0;
        if (mk & (1u << (16 + s))) {
            const double den = dsub(sig, dmul(in[s], cc[s]));
            if (fabs(den) < kPivotFloor) atomicMin(&ctrl->opiv, pk | (unsigned)(g + off[s] + 1));
            nl = ddiv(-cc[s], den);
            lam_other[(3 - s) * no + rb_other(g, s, P.nx)] = nl;
        }
        lam_rec[s * nc + q] = nl;
    }
}

// one colour phase of a cold mean-only red-black sweep with the recorded lambda/sigma of this
// sweep.  FIRST: the red phase of sweep 1 (no message read).  LAST: the last sweep of the call,
// which folds Hierarchy::smooth's x += e (multigrid.cpp:188) into the visit; earlier sweeps
// write no e at all (every visit overwrites it, only the last value is ever used).
template <int COLOUR, bool FIRST, bool LAST>
static __global__ void __launch_bounds__(256) k_rb_mean_half(RbP P, const double* __restrict__ r, double* m_mine,
                                                            double* m_other, const double* __restrict__ lam_rec,
                                                            const double* __restrict__ sig_rec, double* __restrict__ x,
                                                            int r_compact) {
    const int nc = COLOUR == 0 ? P.nR : P.nB, no = COLOUR == 0 ? P.nB : P.nR;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nc) return;
    const int g = rb_nat(P, q, COLOUR);
    const uint32_t mk = P.mask[COLOUR][q];
    // all loads issued before the mask is known (slot arrays are full size; the mask still
    // selects every term): predicated loads wait for the mask's DRAM round trip first
    // r_compact: r is stored per colour (k_residual_dia rb_nx), this colour's half contiguous
    // The black phase of the last sweep sends nothing: the call ends there and its messages are
    // never read (every smoothing call starts cold), so neither the recorded lambda of that
    // visit is loaded nor the four messages stored (64 of the phase's 150 B per node).
    constexpr bool SEND = !(LAST && COLOUR == 1);
    double acc = r[r_compact ? (COLOUR ? P.nR : 0) + q : g], in[4], lam[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        in[s] = FIRST ? 0.0 : m_mine[s * nc + q];
        lam[s] = SEND ? __ldg(lam_rec + s * nc + q) : 0.0;
    }
    const double sg = LAST ? __ldg(sig_rec + q) : 1.0;
    const double xg = LAST ? x[g] : 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (!(mk & (1u << s))) in[s] = 0.0;
        else acc = dadd(acc, in[s]);  // (adding a zero would turn acc = -0 into +0)
    }
    if (LAST) x[g] = dadd(xg, ddiv(acc, sg));
    if (SEND) {
#pragma unroll
        for (int s = 0; s < 4; ++s)
            if (mk & (1u << (16 + s))) m_other[(3 - s) * no + rb_other(g, s, P.nx)] = dmul(lam[s], dsub(acc, in[s]));
    }
}

// The first sweep's red and black phases in one launch over the black nodes.  After a cold start
// a red node's first messages depend on nothing but its own r (acc = r, every in-message zero),
// so each black node forms its four in-messages itself from the neighbours' r and recorded
// lambda (the same operations the red phase performs: r + 0 per in-slot, (acc - 0) * lambda) and
// goes on as the black phase does.  The red phase's message stores and the black phase's
// message loads (64 B per red-black pair) never reach memory; every recorded lambda entry of
// the reds is still read exactly once, by the node it points to.  Sweeps >= 2 only (with one
// sweep the red nodes' x += e needs its own visit).
// ONLY: a one-sweep call (V(1,1)) on a full grid: this pair is also the last one, so the black node
// sends nothing and the x += e of itself and of the red neighbour it owns (k_rb_mean_last_pair's
// rule) happen here; sig_rec / x are used only then.
template <bool ONLY>
static __global__ void __launch_bounds__(256) k_rb_mean_first_pair(RbP P, const double* __restrict__ r,
                                                                  double* m_red, const double* __restrict__ lam_rec,
                                                                  int r_compact, const double* __restrict__ sig_rec,
                                                                  double* __restrict__ x) {
    const int nR = P.nR, nB = P.nB;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nB) return;
    const int g = rb_nat(P, q, 1);
    const uint32_t mk = P.mask[1][q];
    const double* __restrict__ lamR = lam_rec;                    // [4][nR]
    const double* __restrict__ lamB = lam_rec + 4 * (size_t)nR;   // [4][nB]
    const int off[4] = {-P.nx, -1, 1, P.nx};
    double acc = r[r_compact ? nR + q : g], in[4], lam[4];
    int kq[4];
    uint32_t mkk[4];
    double rk[4], lk[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {  // every load first, independent of the masks (indices clamped)
        const int k = g + off[s];
        const int kc = k < 0 ? 0 : (k > 2 * nR - 2 ? 2 * nR - 2 : k);  // clamped into the reds' natural range
        kq[s] = kc >> 1;
        rk[s] = r[r_compact ? kq[s] : rb_nat(P, kq[s], 0)];
        mkk[s] = __ldg(P.mask[0] + kq[s]);
        lk[s] = __ldg(lamR + (size_t)(3 - s) * nR + kq[s]);
        lam[s] = ONLY ? 0.0 : __ldg(lamB + (size_t)s * nB + q);
    }
    double sk[4], xk[4];
    const double sg = ONLY ? __ldg(sig_rec + nR + q) : 1.0, xg = ONLY ? x[g] : 0.0;
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const bool ew = ONLY && (s == 1 || s == 2);  // only an eastern / western neighbour can own k
        sk[s] = ew ? __ldg(sig_rec + kq[s]) : 1.0;
        xk[s] = ew ? x[rb_nat(P, kq[s], 0)] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        // the red neighbour's visit (k_rb_mean_half<0, FIRST>): acc = r (+ 0 per in-slot), message
        // = lambda * (acc - 0)
        double ak = rk[s];
        if (mkk[s] & 0xfu) ak = dadd(ak, 0.0);
        in[s] = dmul(lk[s], dsub(ak, 0.0));
        if (ONLY && (s == 1 || s == 2) && (mk & (1u << s)) && (s == 1 || !(mkk[s] & (1u << 2))))
            x[rb_nat(P, kq[s], 0)] = dadd(xk[s], ddiv(ak, sk[s]));
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (!(mk & (1u << s))) in[s] = 0.0;
        else acc = dadd(acc, in[s]);
    }
    if (ONLY) {
        x[g] = dadd(xg, ddiv(acc, sg));
        return;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s)
        if (mk & (1u << (16 + s))) m_red[(3 - s) * nR + rb_other(g, s, P.nx)] = dmul(lam[s], dsub(acc, in[s]));
}

// The last sweep's red and black phases in one launch over the black nodes (sweeps >= 2, grids
// with every in-grid neighbour present).  The last black visit needs from each red neighbour k
// only k's message to it, lambda * (acc_k - in_k), and acc_k is r_k plus k's four in-messages --
// which are in memory (the previous black phase put them there) and shared by k's four black
// neighbours through L1 / L2.  So each black node rebuilds its neighbours' accumulators (the red
// visit's own operations in its own order), takes its four in-messages from them and finishes;
// the red node's x += e is done by exactly one of its neighbours (the eastern one, else the
// western: the pair is adjacent in x).  The red phase's message stores and this phase's message
// loads, and the half-used sectors of two strided passes over x, never reach DRAM: 136 instead
// of 232 B per red-black pair.
static __global__ void __launch_bounds__(256) k_rb_mean_last_pair(RbP P, const double* __restrict__ r,
                                                                 const double* __restrict__ m_red,
                                                                 const double* __restrict__ lam_rec,
                                                                 const double* __restrict__ sig_rec,
                                                                 double* __restrict__ x, int r_compact) {
    const int nR = P.nR, nB = P.nB;
    const int q = blockIdx.x * blockDim.x + threadIdx.x;
    if (q >= nB) return;
    const int g = rb_nat(P, q, 1);
    const uint32_t mk = P.mask[1][q];
    const int off[4] = {-P.nx, -1, 1, P.nx};
    double acc = r[r_compact ? nR + q : g];
    const double sg = __ldg(sig_rec + nR + q), xg = x[g];
    double in[4];
    // every load first (independent of the masks, indices clamped), then the arithmetic: the
    // kernel is a gather of ~36 values per node, so what counts is how many are in flight
    int kn[4];
    uint32_t mkk[4];
    double ak[4], lk[4], ik[4][4], sk[4], xk[4];
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        const int k = g + off[s];
        const int kc = k < 0 ? 0 : (k > 2 * nR - 2 ? 2 * nR - 2 : k);
        const int kq = kc >> 1;
        kn[s] = rb_nat(P, kq, 0);
        mkk[s] = __ldg(P.mask[0] + kq);
        ak[s] = r[r_compact ? kq : kn[s]];
        lk[s] = __ldg(lam_rec + (size_t)(3 - s) * nR + kq);
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) ik[s][s2] = m_red[(size_t)s2 * nR + kq];
        const bool ew = s == 1 || s == 2;  // only an eastern / western neighbour can own k
        sk[s] = ew ? __ldg(sig_rec + kq) : 1.0;
        xk[s] = ew ? x[kn[s]] : 0.0;
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
#pragma unroll
        for (int s2 = 0; s2 < 4; ++s2) {  // k's visit (k_rb_mean_half<0, false, true>)
            if (!(mkk[s] & (1u << s2))) ik[s][s2] = 0.0;
            else ak[s] = dadd(ak[s], ik[s][s2]);
        }
        in[s] = dmul(lk[s], dsub(ak[s], ik[s][3 - s]));
        // k's x += e: by its eastern neighbour (k's slot 2, reached from here as s = 1), else the western
        if ((s == 1 || s == 2) && (mk & (1u << s)) && (s == 1 || !(mkk[s] & (1u << 2))))
            x[kn[s]] = dadd(xk[s], ddiv(ak[s], sk[s]));
    }
#pragma unroll
    for (int s = 0; s < 4; ++s) {
        if (!(mk & (1u << s))) in[s] = 0.0;
        else acc = dadd(acc, in[s]);
    }
    x[g] = dadd(xg, ddiv(acc, sg));
}

// message state natural DIA [4][n] <-> colour-compact ([4][nR] reds, then [4][nB] blacks)
template <bool TO_COMPACT>
static __global__ void k_rb_convert(int n, int nR, int nx, double2* nat, double2* cmp) {
    const int g = blockIdx.x * blockDim.x + threadIdx.x;
    if (g >= n) return;
    const int q = g >> 1, nB = n - nR;
    const bool red = rb_colour(g, nx) == 0;
    double2* base = red ? cmp : cmp + 4 * (size_t)nR;
    const int nc = red ? nR : nB;
    for (int s = 0; s < 4; ++s) {
        if (TO_COMPACT)
            base[s * nc + q] = nat[(size_t)s * n + g];
        else
            nat[(size_t)s * n + g] = base[s * nc + q];
    }
}

}  // namespace bgabp
