// Line GaBP on a 5-point grid: the two-layer region GaBP of region_gabp.cpp:64-157 with the grid
// lines of region.cpp:208-221 as large regions (rows first, then columns) and the single grid
// nodes as children (parent sets {row, column}, counting number -1).
//
// A line is a tridiagonal local system T (diagonal A_vv + Lambda_other, right-hand side
// b_v + m_other, where "other" is the node's message from its crossing line).  The reference
// factors T densely (Eigen FullPivLU), solves it, inverts it and inverts each 1x1 child block of
// the inverse.  Here each thread owns one line and runs the O(N) equivalent:
//   forward   d_k = a_k - (l_k / d_{k-1}) u_{k-1},  y_k = b0_k - (l_k / d_{k-1}) y_{k-1}
//   backward  x_k = (y_k - u_k x_{k+1}) / d_k,      g_k = a_k - u_k (l_{k+1} / g_{k+1})
//   child precision  W_k = 1 / (T^-1)_kk = d_k + g_k - a_k
//   outgoing message Lambda_k = W_k - A_vv - Lambda_other,  m_k = W_k x_k - b_v - m_other
// (l_k = T(k,k-1), u_k = T(k,k+1)).  The result equals the reference's to rounding (it is not
// the same sequence of operations), so parity is a tolerance, not bits.
//
// Rows phase: thread per row, columns phase: thread per column (coalesced across the warp).
// Sequential mode runs rows then columns on the freshest messages (rows read column messages and
// write row messages, so all rows are independent, and likewise the columns); flood mode reads
// both from the previous sweep.  x is the column phase's solution (the reference's later regions
// overwrite earlier ones).
#pragma once

#include "kernels.cuh"

namespace bgabp {

struct LineP {
    int nx, ny, n;
    const double* diag;  // A_vv
    const double* w;     // A_{v,v-1} (same row), 0 when absent
    const double* e;     // A_{v,v+1}
    const double* s;     // A_{v,v-nx}
    const double* nn;    // A_{v,v+nx}
    const uint32_t* mask;  // bits 0..3: A_{v,v-nx}, A_{v,v-1}, A_{v,v+1}, A_{v,v+nx} stored
};

// failure key: (region << 32) | 0 for a singular local system, | (1 + child position) for a
// singular child block; atomicMin gives the reference's first failure in region order
// REC: also record, per node, the right-hand-side independent factors of this phase -- the forward
// multiplier f_k, 1/d_k and the child precision W_k -- for the mean-only phases below
struct LineRec {
    double *f, *rd, *W;  // [n] each, natural node order
};

template <bool ROW, bool REC = false>
static __global__ void __launch_bounds__(32) k_line_phase(LineP P, const double* __restrict__ b,
                                                         const double* __restrict__ lam_o,
                                                         const double* __restrict__ m_o, double* __restrict__ lam_n,
                                                         double* __restrict__ m_n, double* __restrict__ x,
                                                         double* __restrict__ fd, double* __restrict__ fy,
                                                         unsigned long long* fail, const int* done, LineRec rec = {}) {
    if (done && *(volatile const int*)done) return;
    // a region already failed (rows of this sweep, or an earlier sweep of a smoothing call): the
    // reference stopped there
    if (*(volatile unsigned long long*)fail != kNone) return;
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int nlines = ROW ? P.ny : P.nx, N = ROW ? P.nx : P.ny;
    if (line >= nlines) return;
    const int stride = ROW ? 1 : P.nx;
    const int base = ROW ? line * P.nx : line;
    const double* lo = ROW ? P.w : P.s;   // T(k, k-1)
    const double* up = ROW ? P.e : P.nn;  // T(k, k+1)
    const unsigned long long region = (unsigned long long)(ROW ? line : P.ny + line);
    // Loads do not depend on the recurrences: each chunk of kLC steps issues all of its loads
    // first, so one memory latency is paid per chunk instead of per step (one warp holds 32
    // lines and there are only nx + ny lines, so other warps cannot hide it).
    constexpr int kLC = 8;
    bool singular = false;
    double dprev = 0.0, yprev = 0.0, uprev = 0.0;
    for (int k0 = 0; k0 < N; k0 += kLC) {
        double av[kLC], bv[kLC], lv[kLC], uv[kLC];
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int k = k0 + q;
            const int v = base + (k < N ? k : N - 1) * stride;
            av[q] = dadd(__ldg(P.diag + v), lam_o[v]);
            bv[q] = dadd(__ldg(b + v), m_o[v]);
            lv[q] = __ldg(lo + v);
            uv[q] = __ldg(up + v);
        }
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int k = k0 + q;
            if (k >= N) break;
            const int v = base + k * stride;
            double d, y;
            if (k == 0) {
                d = av[q];
                y = bv[q];
                if (REC) rec.f[v] = 0.0;
            } else {
                const double f = ddiv(lv[q], dprev);
                d = dsub(av[q], dmul(f, uprev));
                y = dsub(bv[q], dmul(f, yprev));
                if (REC) rec.f[v] = f;
            }
            if (d == 0.0 || !isfinite(d)) singular = true;
            if (REC) rec.rd[v] = ddiv(1.0, d);
            fd[v] = d;
            fy[v] = y;
            dprev = d;
            yprev = y;
            uprev = uv[q];
        }
    }
    if (singular) {
        atomicMin(fail, region << 32);
        return;
    }
    double xnext = 0.0, gnext = 0.0, lnext = 0.0;
    unsigned long long bad = kNone;
    for (int k1 = N - 1; k1 >= 0; k1 -= kLC) {
        double lo_v[kLC], mo_v[kLC], dv[kLC], bb[kLC], dd[kLC], yy[kLC], uu[kLC], ll[kLC];
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int k = k1 - q;
            const int v = base + (k >= 0 ? k : 0) * stride;
            lo_v[q] = lam_o[v];
            mo_v[q] = m_o[v];
            dv[q] = __ldg(P.diag + v);
            bb[q] = __ldg(b + v);
            dd[q] = fd[v];
            yy[q] = fy[v];
            uu[q] = __ldg(up + v);
            ll[q] = __ldg(lo + v);
        }
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int k = k1 - q;
            if (k < 0) break;
            const int v = base + k * stride;
            const double a = dadd(dv[q], lo_v[q]);
            double xk, g;
            if (k == N - 1) {
                xk = ddiv(yy[q], dd[q]);
                g = a;
            } else {
                xk = ddiv(dsub(yy[q], dmul(uu[q], xnext)), dd[q]);
                g = dsub(a, dmul(uu[q], ddiv(lnext, gnext)));
            }
            const double W = dsub(dadd(dd[q], g), a);
            if (W == 0.0 || !isfinite(W)) bad = (region << 32) | (unsigned long long)(1 + k);
            if (REC) rec.W[v] = W;
            lam_n[v] = dsub(dsub(W, dv[q]), lo_v[q]);
            m_n[v] = dsub(dsub(dmul(W, xk), bb[q]), mo_v[q]);
            if (x) x[v] = xk;
            xnext = xk;
            gnext = g;
            lnext = ll[q];
        }
    }
    if (bad != kNone) atomicMin(fail, bad);
}

// Mean-only phase with the recorded factors of a cold start (multigrid smoothing: every call
// restarts the block messages at zero, multigrid.cpp:195, and the precision recursion never reads
// the means, so f, 1/d and W of sweep s depend on A alone).  The forward and backward recurrences
// are then one multiply-add each: y_k = b0_k - f_k y_{k-1}, x_k = (y_k - u_k x_{k+1}) / d_k (as a
// product with the recorded reciprocal, so the smoother's x agrees with the full line solve to
// rounding), m_k = W_k x_k - b_k - m_other_k.  ADDX: the call's last column phase adds x into the
// iterate (Hierarchy::smooth's x += e) instead of writing e.
template <bool ROW, bool ADDX>
static __global__ void __launch_bounds__(32) k_line_mean_phase(LineP P, const double* __restrict__ b,
                                                              const double* __restrict__ m_o,
                                                              double* __restrict__ m_n, double* __restrict__ x,
                                                              double* __restrict__ fy, const double* __restrict__ f,
                                                              const double* __restrict__ rd,
                                                              const double* __restrict__ W) {
    const int line = blockIdx.x * blockDim.x + threadIdx.x;
    const int nlines = ROW ? P.ny : P.nx, N = ROW ? P.nx : P.ny;
    if (line >= nlines) return;
    const int stride = ROW ? 1 : P.nx;
    const int base = ROW ? line * P.nx : line;
    const double* up = ROW ? P.e : P.nn;
    constexpr int kLC = 16;
    double yprev = 0.0;
    for (int k0 = 0; k0 < N; k0 += kLC) {
        double bv[kLC], fv[kLC];
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int v = base + min(k0 + q, N - 1) * stride;
            bv[q] = dadd(__ldg(b + v), m_o[v]);
            fv[q] = __ldg(f + v);
        }
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            if (k0 + q >= N) break;
            yprev = dsub(bv[q], dmul(fv[q], yprev));
            fy[base + (k0 + q) * stride] = yprev;
        }
    }
    double xnext = 0.0;
    for (int k1 = N - 1; k1 >= 0; k1 -= kLC) {
        double yy[kLC], uu[kLC], rr[kLC], ww[kLC], bb[kLC], mo[kLC], xo[ADDX ? kLC : 1];
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int v = base + max(k1 - q, 0) * stride;
            yy[q] = fy[v];
            uu[q] = __ldg(up + v);
            rr[q] = __ldg(rd + v);
            ww[q] = __ldg(W + v);
            bb[q] = __ldg(b + v);
            mo[q] = m_o[v];
            if (ADDX) xo[ADDX ? q : 0] = x[v];  // the iterate, read with the chunk (not per step)
        }
#pragma unroll
        for (int q = 0; q < kLC; ++q) {
            const int k = k1 - q;
            if (k < 0) break;
            const int v = base + k * stride;
            const double xk = dmul(k == N - 1 ? yy[q] : dsub(yy[q], dmul(uu[q], xnext)), rr[q]);
            m_n[v] = dsub(dsub(dmul(ww[q], xk), bb[q]), mo[q]);
            if (x) x[v] = ADDX ? dadd(xo[ADDX ? q : 0], xk) : xk;
            xnext = xk;
        }
    }
}

// ---- parallel-scan versions of the mean-only phases ------------------------------------------
// The two recurrences are affine: forward y_k = -f_k y_{k-1} + c_k, backward
// x_k = q_k x_{k+1} + p_k with q_k = -u_k / d_k, p_k = y_k / d_k.  Composing the affine maps with a
// scan runs a line in O(N / P + log P) dependent steps instead of N (the association differs from
// the sequential loop, so x agrees with it to rounding; each node is still evaluated by the serial
// formula from its segment's carry-in).
//  Rows: one warp per row; a lane owns kLV consecutive nodes of a 32·kLV tile, composes their maps
//  serially, the warp scans the 32 lane maps with shuffles, a carry runs between tiles.
//  Columns: a block owns kCW adjacent columns (kCW threads read 8·kCW contiguous bytes of a row:
//  whole sectors) and splits each column into kSeg segments; the segment maps are scanned in
//  shared memory.
struct Aff {
    double a, b;  // v -> a v + b
};
__device__ __forceinline__ Aff aff_then(Aff first, Aff second) {  // second(first(v))
    return {dmul(second.a, first.a), dadd(dmul(second.a, first.b), second.b)};
}
__device__ __forceinline__ double aff_apply(Aff m, double v) { return dadd(dmul(m.a, v), m.b); }
// exclusive scan of the lane maps in lane order
__device__ __forceinline__ Aff warp_scan_aff_excl(Aff m) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        Aff p;
        p.a = __shfl_up_sync(0xffffffffu, m.a, o);
        p.b = __shfl_up_sync(0xffffffffu, m.b, o);
        if (lane >= o) m = aff_then(p, m);
    }
    Aff e;
    e.a = __shfl_up_sync(0xffffffffu, m.a, 1);
    e.b = __shfl_up_sync(0xffffffffu, m.b, 1);
    return lane == 0 ? Aff{1.0, 0.0} : e;
}

constexpr int kLV = 4;  // nodes per lane per row tile

template <bool ADDX>
static __global__ void __launch_bounds__(128) k_line_mean_rows(LineP P, const double* __restrict__ b,
                                                              const double* __restrict__ m_o, double* __restrict__ m_n,
                                                              double* __restrict__ x, double* __restrict__ fy,
                                                              const double* __restrict__ f,
                                                              const double* __restrict__ rd,
                                                              const double* __restrict__ W) {
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= P.ny) return;  // warp-uniform
    const int N = P.nx, base = row * P.nx;
    double carry = 0.0;
    for (int t0 = 0; t0 < N; t0 += 32 * kLV) {
        const int k0 = t0 + lane * kLV;
        double fk[kLV], ck[kLV];
        Aff m{1.0, 0.0};
#pragma unroll
        for (int j = 0; j < kLV; ++j) {
            const int k = k0 + j;
            fk[j] = 0.0;
            ck[j] = 0.0;
            if (k < N) {
                fk[j] = -__ldg(f + base + k);
                ck[j] = dadd(__ldg(b + base + k), m_o[base + k]);
                m = aff_then(m, Aff{fk[j], ck[j]});
            }
        }
        double y = aff_apply(warp_scan_aff_excl(m), carry);
#pragma unroll
        for (int j = 0; j < kLV; ++j)
            if (k0 + j < N) {
                y = dadd(dmul(fk[j], y), ck[j]);
                fy[base + k0 + j] = y;
            }
        carry = __shfl_sync(0xffffffffu, y, 31);
    }
    carry = 0.0;
    for (int t0 = 0; t0 < N; t0 += 32 * kLV) {  // from the end of the row: lane 0 owns the highest k
        const int k0 = N - 1 - (t0 + lane * kLV);
        double qk[kLV], pk[kLV];
        Aff m{1.0, 0.0};
#pragma unroll
        for (int j = 0; j < kLV; ++j) {
            const int k = k0 - j;
            qk[j] = 0.0;
            pk[j] = 0.0;
            if (k >= 0) {
                const double r = __ldg(rd + base + k);
                qk[j] = -dmul(__ldg(P.e + base + k), r);
                pk[j] = dmul(fy[base + k], r);
                m = aff_then(m, Aff{qk[j], pk[j]});
            }
        }
        double xk = aff_apply(warp_scan_aff_excl(m), carry);
#pragma unroll
        for (int j = 0; j < kLV; ++j) {
            const int k = k0 - j;
            if (k >= 0) {
                const int v = base + k;
                xk = dadd(dmul(qk[j], xk), pk[j]);
                m_n[v] = dsub(dsub(dmul(__ldg(W + v), xk), __ldg(b + v)), m_o[v]);
                if (x) x[v] = ADDX ? dadd(x[v], xk) : xk;
            }
        }
        carry = __shfl_sync(0xffffffffu, xk, 31);
    }
}

constexpr int kCW = 8;                // columns per block
constexpr int kCT = 1024;             // threads per block
constexpr int kSeg = kCT / kCW;       // segments per column

// inclusive scan over the kSeg segment maps of each column; REV: segment order kSeg-1 .. 0
template <bool REV>
__device__ __forceinline__ Aff seg_scan_excl(Aff m, int sgm, int c, Aff (*sh)[kCW]) {
    for (int o = 1; o < kSeg; o <<= 1) {
        sh[sgm][c] = m;
        __syncthreads();
        const int src = REV ? sgm + o : sgm - o;
        if (REV ? src < kSeg : src >= 0) m = aff_then(sh[src][c], m);
        __syncthreads();
    }
    sh[sgm][c] = m;
    __syncthreads();
    const int src = REV ? sgm + 1 : sgm - 1;
    const Aff e = (REV ? src < kSeg : src >= 0) ? sh[src][c] : Aff{1.0, 0.0};
    __syncthreads();
    return e;
}

template <bool ADDX>
static __global__ void __launch_bounds__(kCT) k_line_mean_cols(LineP P, const double* __restrict__ b,
                                                              const double* __restrict__ m_o, double* __restrict__ m_n,
                                                              double* __restrict__ x, double* __restrict__ fy,
                                                              const double* __restrict__ f,
                                                              const double* __restrict__ rd,
                                                              const double* __restrict__ W) {
    __shared__ Aff sh[kSeg][kCW];
    const int c = threadIdx.x % kCW, sgm = threadIdx.x / kCW;
    const int col = blockIdx.x * kCW + c;
    const bool ok = col < P.nx;
    const int nx = P.nx, N = P.ny, L = (N + kSeg - 1) / kSeg;
    const int k0 = min(N, sgm * L), k1 = min(N, k0 + L);
    Aff m{1.0, 0.0};
    if (ok)
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
            const int v = k * nx + col;
            m = aff_then(m, Aff{-__ldg(f + v), dadd(__ldg(b + v), m_o[v])});
        }
    double y = aff_apply(seg_scan_excl<false>(m, sgm, c, sh), 0.0);
    // the forward evaluation also builds the segment's backward map x_{k0} = C(x_{k1}), composed
    // from k0 upward (C <- C o N_k), so fy is not re-read for it
    m = Aff{1.0, 0.0};
    if (ok)
#pragma unroll 4
        for (int k = k0; k < k1; ++k) {
            const int v = k * nx + col;
            y = dadd(dmul(-__ldg(f + v), y), dadd(__ldg(b + v), m_o[v]));
            fy[v] = y;
            const double r = __ldg(rd + v);
            m = aff_then(Aff{-dmul(__ldg(P.nn + v), r), dmul(y, r)}, m);
        }
    double xn = aff_apply(seg_scan_excl<true>(m, sgm, c, sh), 0.0);
    if (ok)
#pragma unroll 4
        for (int k = k1 - 1; k >= k0; --k) {
            const int v = k * nx + col;
            const double r = __ldg(rd + v);
            const double xk = dadd(dmul(-dmul(__ldg(P.nn + v), r), xn), dmul(fy[v], r));
            m_n[v] = dsub(dsub(dmul(__ldg(W + v), xk), __ldg(b + v)), m_o[v]);
            if (x) x[v] = ADDX ? dadd(x[v], xk) : xk;
            xn = xk;
        }
}

// ---- parallel-scan versions of the full phases (precisions and means) -------------------------
// Forward: with d_{k-1} = p / q and y_{k-1} = Z / q the pair of recurrences
//   d_k = a_k - c_k / d_{k-1} (c_k = l_k u_{k-1}),  y_k = bv_k - (l_k / d_{k-1}) y_{k-1}
// is linear in the state (p, q, Z):  p' = a p - c q,  q' = p,  Z' = bv p - l Z, i.e. a 3x3 block
// lower-triangular matrix [[a, -c, 0], [1, 0, 0], [bv, 0, -l]]; products keep that shape.
// Backward: g_k = a_k - c'_k / g_{k+1} (c'_k = u_k l_{k+1}) is the 2x2 Moebius map
// [[a, -c'], [1, 0]] on (P, Q), and x_k = (-u_k / d_k) x_{k+1} + y_k / d_k is affine.
// Maps are composed and scanned exactly like the mean phases, with every product rescaled by a
// power of two (exact; the state is projective) so long lines cannot overflow.  Each node is
// still evaluated by the serial formula from its lane's / segment's carry-in, so d, y, x, g and
// the messages agree with the sequential recurrences to rounding; lines of up to kLV (rows) or
// kMinSeg (columns) nodes are evaluated entirely serially, i.e. with identical operations.
struct FwdM {
    double a00, a01, a10, a11, b0, b1, l;  // [[a00 a01 0] [a10 a11 0] [b0 b1 l]]
};
struct BwdM {
    double g00, g01, g10, g11;  // Moebius map of g on (P, Q)
    double xa, xb;              // x -> xa x + xb
};
__device__ __forceinline__ FwdM fwd_identity() { return {1.0, 0.0, 0.0, 1.0, 0.0, 0.0, 1.0}; }
__device__ __forceinline__ BwdM bwd_identity() { return {1.0, 0.0, 0.0, 1.0, 1.0, 0.0}; }
__device__ __forceinline__ double pow2_scale_for(double m) {  // 2^-e with m ~ 2^e (1 if m is 0 / inf / nan)
    if (!(m > 0.0) || !isfinite(m)) return 1.0;
    return ldexp(1.0, -ilogb(m));
}
// second o first (apply first, then second); NORM: rescaled by a power of two (the lane and
// segment loops compose a few raw products between rescales)
template <bool NORM = true>
__device__ __forceinline__ FwdM fwd_then(const FwdM& F, const FwdM& G) {
    FwdM r;
    r.a00 = G.a00 * F.a00 + G.a01 * F.a10;
    r.a01 = G.a00 * F.a01 + G.a01 * F.a11;
    r.a10 = G.a10 * F.a00 + G.a11 * F.a10;
    r.a11 = G.a10 * F.a01 + G.a11 * F.a11;
    r.b0 = G.b0 * F.a00 + G.b1 * F.a10 + G.l * F.b0;
    r.b1 = G.b0 * F.a01 + G.b1 * F.a11 + G.l * F.b1;
    r.l = G.l * F.l;
    if (!NORM) return r;
    const double m = fmax(fmax(fmax(fabs(r.a00), fabs(r.a01)), fmax(fabs(r.a10), fabs(r.a11))),
                          fmax(fmax(fabs(r.b0), fabs(r.b1)), fabs(r.l)));
    const double sc = pow2_scale_for(m);
    r.a00 *= sc; r.a01 *= sc; r.a10 *= sc; r.a11 *= sc; r.b0 *= sc; r.b1 *= sc; r.l *= sc;
    return r;
}
template <bool NORM = true>
__device__ __forceinline__ BwdM bwd_then(const BwdM& F, const BwdM& G) {
    BwdM r;
    r.g00 = G.g00 * F.g00 + G.g01 * F.g10;
    r.g01 = G.g00 * F.g01 + G.g01 * F.g11;
    r.g10 = G.g10 * F.g00 + G.g11 * F.g10;
    r.g11 = G.g10 * F.g01 + G.g11 * F.g11;
    r.xa = G.xa * F.xa;
    r.xb = G.xa * F.xb + G.xb;
    if (!NORM) return r;
    const double sc = pow2_scale_for(fmax(fmax(fabs(r.g00), fabs(r.g01)), fmax(fabs(r.g10), fabs(r.g11))));
    r.g00 *= sc; r.g01 *= sc; r.g10 *= sc; r.g11 *= sc;
    return r;
}
// the state (dprev, yprev) reached from state s = (p, q, Z) through M
__device__ __forceinline__ void fwd_apply(const FwdM& M, double p, double q, double Z, double& d, double& y) {
    const double p2 = M.a00 * p + M.a01 * q, q2 = M.a10 * p + M.a11 * q, Z2 = M.b0 * p + M.b1 * q + M.l * Z;
    d = p2 / q2;
    y = Z2 / q2;
}
__device__ __forceinline__ void bwd_apply(const BwdM& M, double P, double Q, double x, double& g, double& xo) {
    g = (M.g00 * P + M.g01 * Q) / (M.g10 * P + M.g11 * Q);
    xo = M.xa * x + M.xb;
}
template <class T>
__device__ __forceinline__ T shfl_up_struct(const T& v, int o) {
    T r;
    const double* s = reinterpret_cast<const double*>(&v);
    double* d = reinterpret_cast<double*>(&r);
#pragma unroll
    for (int i = 0; i < (int)(sizeof(T) / sizeof(double)); ++i) d[i] = __shfl_up_sync(0xffffffffu, s[i], o);
    return r;
}
template <class T, class Then>
__device__ __forceinline__ T warp_scan_excl_gen(T m, T ident, Then then) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const T p = shfl_up_struct(m, o);
        if (lane >= o) m = then(p, m);
    }
    const T e = shfl_up_struct(m, 1);
    return lane == 0 ? ident : e;
}

constexpr int kFLV = 4;  // nodes per lane per row tile (full phase)

// rows phase, one warp per row (the serial k_line_phase<true, REC> reorganised as scans)
template <bool REC>
static __global__ void __launch_bounds__(128) k_line_full_rows(LineP P, const double* __restrict__ b,
                                                              const double* __restrict__ lam_o,
                                                              const double* __restrict__ m_o,
                                                              double* __restrict__ lam_n, double* __restrict__ m_n,
                                                              double* __restrict__ fd, double* __restrict__ fy,
                                                              unsigned long long* fail, const int* done,
                                                              LineRec rec) {
    if (done && *(volatile const int*)done) return;
    if (*(volatile unsigned long long*)fail != kNone) return;
    const int row = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (row >= P.ny) return;  // warp-uniform
    const int N = P.nx, base = row * P.nx;
    const unsigned long long region = (unsigned long long)row;
    bool singular = false;
    // forward: carry state (p, q, Z); (1, 0, 0) before node 0
    double cp = 1.0, cq = 0.0, cZ = 0.0;
    for (int t0 = 0; t0 < N; t0 += 32 * kFLV) {
        const int k0 = t0 + lane * kFLV;
        double av[kFLV], bv[kFLV], lv[kFLV], uv[kFLV];  // uv[j] = u_{k-1}
        FwdM M = fwd_identity();
#pragma unroll
        for (int j = 0; j < kFLV; ++j) {
            const int k = k0 + j, v = base + min(k, N - 1);
            av[j] = dadd(__ldg(P.diag + v), lam_o[v]);
            bv[j] = dadd(__ldg(b + v), m_o[v]);
            lv[j] = __ldg(P.w + v);
            uv[j] = (k >= 1 && k < N) ? __ldg(P.e + v - 1) : 0.0;
            if (k < N) M = fwd_then<false>(M, FwdM{av[j], -(lv[j] * uv[j]), 1.0, 0.0, bv[j], 0.0, -lv[j]});
        }
        M = fwd_then(M, fwd_identity());  // rescale once per lane
        const FwdM E = warp_scan_excl_gen(M, fwd_identity(), [](const FwdM& f, const FwdM& g) { return fwd_then<true>(f, g); });
        double dprev, yprev;
        fwd_apply(E, cp, cq, cZ, dprev, yprev);
#pragma unroll
        for (int j = 0; j < kFLV; ++j) {
            const int k = k0 + j;
            if (k >= N) break;
            const int v = base + k;
            double d, y;
            if (k == 0) {
                d = av[j];
                y = bv[j];
                if (REC) rec.f[v] = 0.0;
            } else {
                const double f = ddiv(lv[j], dprev);
                d = dsub(av[j], dmul(f, uv[j]));
                y = dsub(bv[j], dmul(f, yprev));
                if (REC) rec.f[v] = f;
            }
            if (d == 0.0 || !isfinite(d)) singular = true;
            if (REC) rec.rd[v] = ddiv(1.0, d);
            fd[v] = d;
            fy[v] = y;
            dprev = d;
            yprev = y;
        }
        cp = __shfl_sync(0xffffffffu, dprev, 31);
        cq = 1.0;
        cZ = __shfl_sync(0xffffffffu, yprev, 31);
    }
    if (__any_sync(0xffffffffu, singular)) {
        if (lane == 0) atomicMin(fail, region << 32);
        return;
    }
    // backward from the end of the row: lane 0 owns the highest k; carry (P, Q) = (1, 0), x = 0
    double gP = 1.0, gQ = 0.0, cx = 0.0;
    unsigned long long bad = kNone;
    for (int t0 = 0; t0 < N; t0 += 32 * kFLV) {
        const int k0 = N - 1 - (t0 + lane * kFLV);
        double av[kFLV], dv[kFLV], yv[kFLV], uv[kFLV], ln[kFLV], dg[kFLV], lo[kFLV], bb[kFLV], mo[kFLV];
        BwdM M = bwd_identity();
#pragma unroll
        for (int j = 0; j < kFLV; ++j) {
            const int k = k0 - j, v = base + max(k, 0);
            lo[j] = lam_o[v];
            dg[j] = __ldg(P.diag + v);
            av[j] = dadd(dg[j], lo[j]);
            dv[j] = fd[v];
            yv[j] = fy[v];
            uv[j] = __ldg(P.e + v);
            ln[j] = (k >= 0 && k + 1 < N) ? __ldg(P.w + v + 1) : 0.0;  // l_{k+1}
            bb[j] = __ldg(b + v);
            mo[j] = m_o[v];
            if (k >= 0) {
                const double rdk = 1.0 / dv[j];
                M = bwd_then<false>(M, BwdM{av[j], -(uv[j] * ln[j]), 1.0, 0.0, -uv[j] * rdk, yv[j] * rdk});
            }
        }
        M = bwd_then(M, bwd_identity());
        const BwdM E = warp_scan_excl_gen(M, bwd_identity(), [](const BwdM& f, const BwdM& g) { return bwd_then<true>(f, g); });
        double gnext, xnext;
        bwd_apply(E, gP, gQ, cx, gnext, xnext);
#pragma unroll
        for (int j = 0; j < kFLV; ++j) {
            const int k = k0 - j;
            if (k < 0) break;
            const int v = base + k;
            double xk, g;
            if (k == N - 1) {
                xk = ddiv(yv[j], dv[j]);
                g = av[j];
            } else {
                xk = ddiv(dsub(yv[j], dmul(uv[j], xnext)), dv[j]);
                g = dsub(av[j], dmul(uv[j], ddiv(ln[j], gnext)));
            }
            const double W = dsub(dadd(dv[j], g), av[j]);
            if (W == 0.0 || !isfinite(W)) bad = (region << 32) | (unsigned long long)(1 + k);
            if (REC) rec.W[v] = W;
            lam_n[v] = dsub(dsub(W, dg[j]), lo[j]);
            m_n[v] = dsub(dsub(dmul(W, xk), bb[j]), mo[j]);
            xnext = xk;
            gnext = g;
        }
        gP = __shfl_sync(0xffffffffu, gnext, 31);
        gQ = 1.0;
        cx = __shfl_sync(0xffffffffu, xnext, 31);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ob = __shfl_xor_sync(0xffffffffu, bad, o);
        bad = ob < bad ? ob : bad;
    }
    if (lane == 0 && bad != kNone) atomicMin(fail, bad);
}

constexpr int kFCW = 8;                 // columns per block (full phase)
constexpr int kFCT = 512;               // threads per block
constexpr int kFSeg = kFCT / kFCW;      // segments per column
constexpr int kMinSeg = 16;             // nodes per segment at least (short columns stay serial)

template <class T, bool REV, class Then>
__device__ __forceinline__ T seg_scan_excl_gen(T m, T ident, int sgm, int c, T (*sh)[kFCW], Then then) {
    for (int o = 1; o < kFSeg; o <<= 1) {
        sh[sgm][c] = m;
        __syncthreads();
        const int src = REV ? sgm + o : sgm - o;
        if (REV ? src < kFSeg : src >= 0) m = then(sh[src][c], m);
        __syncthreads();
    }
    sh[sgm][c] = m;
    __syncthreads();
    const int src = REV ? sgm + 1 : sgm - 1;
    const T e = (REV ? src < kFSeg : src >= 0) ? sh[src][c] : ident;
    __syncthreads();
    return e;
}

// columns phase: a block per kFCW adjacent columns, each cut into kFSeg segments
template <bool REC>
static __global__ void __launch_bounds__(kFCT, 2) k_line_full_cols(LineP P, const double* __restrict__ b,
                                                               const double* __restrict__ lam_o,
                                                               const double* __restrict__ m_o,
                                                               double* __restrict__ lam_n, double* __restrict__ m_n,
                                                               double* __restrict__ x, double* __restrict__ fd,
                                                               double* __restrict__ fy, unsigned long long* fail,
                                                               const int* done, LineRec rec) {
    __shared__ FwdM shf[kFSeg][kFCW];
    __shared__ int sing[kFCW];
    __shared__ int skip;
    if (threadIdx.x == 0)  // one read for the block: the barriers below need a uniform decision
        skip = (done && *(volatile const int*)done) || *(volatile unsigned long long*)fail != kNone;
    __syncthreads();
    if (skip) return;
    BwdM(*shb)[kFCW] = reinterpret_cast<BwdM(*)[kFCW]>(&shf[0][0]);  // same storage, after the forward scan
    const int c = threadIdx.x % kFCW, sgm = threadIdx.x / kFCW;
    const int col = blockIdx.x * kFCW + c;
    const bool ok = col < P.nx;
    const int nx = P.nx, N = P.ny;
    const int L = max((N + kFSeg - 1) / kFSeg, kMinSeg);
    const int k0 = min(N, sgm * L), k1 = min(N, k0 + L);
    const unsigned long long region = (unsigned long long)(P.ny + col);
    if (threadIdx.x < kFCW) sing[threadIdx.x] = 0;
    FwdM M = fwd_identity();
    if (ok)
        for (int k = k0; k < k1; ++k) {
            const int v = k * nx + col;
            const double a = dadd(__ldg(P.diag + v), lam_o[v]), bv = dadd(__ldg(b + v), m_o[v]);
            const double l = __ldg(P.s + v), u = k >= 1 ? __ldg(P.nn + v - nx) : 0.0;
            M = fwd_then(M, FwdM{a, -(l * u), 1.0, 0.0, bv, 0.0, -l});
        }
    const FwdM E = seg_scan_excl_gen<FwdM, false>(M, fwd_identity(), sgm, c, shf,
                                                   [](const FwdM& f, const FwdM& g) { return fwd_then<true>(f, g); });
    double dprev, yprev;
    fwd_apply(E, 1.0, 0.0, 0.0, dprev, yprev);
    // serial forward evaluation; the segment's backward map is composed on the way (C <- C o N_k)
    BwdM B = bwd_identity();
    bool singular = false;
    if (ok)
        for (int k = k0; k < k1; ++k) {
            const int v = k * nx + col;
            const double a = dadd(__ldg(P.diag + v), lam_o[v]), bv = dadd(__ldg(b + v), m_o[v]);
            const double l = __ldg(P.s + v);
            double d, y;
            if (k == 0) {
                d = a;
                y = bv;
                if (REC) rec.f[v] = 0.0;
            } else {
                const double f = ddiv(l, dprev);
                d = dsub(a, dmul(f, __ldg(P.nn + v - nx)));
                y = dsub(bv, dmul(f, yprev));
                if (REC) rec.f[v] = f;
            }
            if (d == 0.0 || !isfinite(d)) singular = true;
            if (REC) rec.rd[v] = ddiv(1.0, d);
            fd[v] = d;
            fy[v] = y;
            dprev = d;
            yprev = y;
            const double u = __ldg(P.nn + v), ln = k + 1 < N ? __ldg(P.s + v + nx) : 0.0;
            const double rdk = 1.0 / d;
            B = bwd_then(BwdM{a, -(u * ln), 1.0, 0.0, -u * rdk, y * rdk}, B);
        }
    if (singular) atomicOr(&sing[c], 1);
    __syncthreads();
    if (sing[c]) {  // uniform per column; the block still joins the barriers below
        if (sgm == 0 && ok) atomicMin(fail, region << 32);
    }
    const BwdM EB = seg_scan_excl_gen<BwdM, true>(B, bwd_identity(), sgm, c, shb,
                                                   [](const BwdM& f, const BwdM& g) { return bwd_then<true>(f, g); });
    if (sing[c] || !ok) return;
    double gnext, xnext;
    bwd_apply(EB, 1.0, 0.0, 0.0, gnext, xnext);
    unsigned long long bad = kNone;
    for (int k = k1 - 1; k >= k0; --k) {
        const int v = k * nx + col;
        const double lo = lam_o[v], dg = __ldg(P.diag + v);
        const double a = dadd(dg, lo), d = fd[v], y = fy[v], u = __ldg(P.nn + v);
        double xk, g;
        if (k == N - 1) {
            xk = ddiv(y, d);
            g = a;
        } else {
            xk = ddiv(dsub(y, dmul(u, xnext)), d);
            g = dsub(a, dmul(u, ddiv(__ldg(P.s + v + nx), gnext)));
        }
        const double W = dsub(dadd(d, g), a);
        if (W == 0.0 || !isfinite(W)) bad = (region << 32) | (unsigned long long)(1 + k);
        if (REC) rec.W[v] = W;
        lam_n[v] = dsub(dsub(W, dg), lo);
        m_n[v] = dsub(dsub(dmul(W, xk), __ldg(b + v)), m_o[v]);
        if (x) x[v] = xk;
        xnext = xk;
        gnext = g;
    }
    if (bad != kNone) atomicMin(fail, bad);
}

// r = b - A x in CSR column order (sparse.cpp:104-115) and its NaN-skipping inf-norm
static __global__ void k_line_residual(LineP P, const double* __restrict__ b, const double* __restrict__ x,
                                       double* __restrict__ r, unsigned long long* rmax, const int* done) {
    if (done && *(volatile const int*)done) return;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    double ra = 0.0;
    if (v < P.n) {  // loads issued independent of the mask (k_residual_dia)
        const int n = P.n;
        const uint32_t mk = P.mask[v];
        const double xs = x[max(v - P.nx, 0)], xw = x[max(v - 1, 0)], xc = x[v], xe = x[min(v + 1, n - 1)],
                     xn = x[min(v + P.nx, n - 1)];
        const double cs = __ldg(P.s + v), cw = __ldg(P.w + v), cd = __ldg(P.diag + v), ce = __ldg(P.e + v),
                     cn = __ldg(P.nn + v);
        double acc = b[v];
        if (mk & 1u) acc = dsub(acc, dmul(cs, xs));
        if (mk & 2u) acc = dsub(acc, dmul(cw, xw));
        acc = dsub(acc, dmul(cd, xc));
        if (mk & 4u) acc = dsub(acc, dmul(ce, xe));
        if (mk & 8u) acc = dsub(acc, dmul(cn, xn));
        if (r) r[v] = acc;
        ra = nan_skip_abs(acc);
    }
    if (rmax) block_max_red(rmax, ra);
}

struct LineCtrl {
    int done, status, iterations, step;
    unsigned long long rmax, fail, detail_key;
    double r0, tol, divergence;
    int max_iter, mode;
};

// RegionGabpEngine::solve's per-iteration test (region_gabp.cpp:172-197)
static __global__ void k_line_decide(LineCtrl* c, double* history, int kind_stop_on_fail) {
    if (c->done) return;
    const int it = c->step;
    c->iterations = it;
    if (c->fail != kNone) {
        c->status = 1;
        c->detail_key = c->fail;
        c->done = 1;
        return;
    }
    const double r = __longlong_as_double((long long)c->rmax);
    history[it] = r;
    c->rmax = 0ull;
    if (!isfinite(r) || r > c->divergence * c->r0) {
        c->status = 1;
        c->detail_key = kNone - 1;  // residual blowup
        c->done = 1;
        return;
    }
    if (r <= c->tol) {
        c->status = 0;
        c->done = 1;
        return;
    }
    if (it >= c->max_iter) {
        c->status = 2;
        c->done = 1;
        return;
    }
    c->step = it + 1;
    (void)kind_stop_on_fail;
}

// x += e, and the multigrid failure record for the level (see Engine::decode_failure kinds 6, 7)
static __global__ void k_line_check(Ctrl* c, const unsigned long long* fail, int seq) {
    if (c->halt || *fail == kNone) return;
    c->halt = 1;
    c->fail_seq = seq;
    c->detail_kind = (*fail & 0xffffffffull) ? 7 : 6;
    c->detail_key = *fail;
}

}  // namespace bgabp
