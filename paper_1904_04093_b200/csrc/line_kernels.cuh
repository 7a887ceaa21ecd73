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

// r = b - A x in CSR column order (sparse.cpp:104-115) and its NaN-skipping inf-norm
static __global__ void k_line_residual(LineP P, const double* __restrict__ b, const double* __restrict__ x,
                                       double* __restrict__ r, unsigned long long* rmax, const int* done) {
    if (done && *(volatile const int*)done) return;
    const int v = blockIdx.x * blockDim.x + threadIdx.x;
    double ra = 0.0;
    if (v < P.n) {
        const uint32_t mk = P.mask[v];
        double acc = b[v];
        if (mk & 1u) acc = dsub(acc, dmul(P.s[v], x[v - P.nx]));
        if (mk & 2u) acc = dsub(acc, dmul(P.w[v], x[v - 1]));
        acc = dsub(acc, dmul(P.diag[v], x[v]));
        if (mk & 4u) acc = dsub(acc, dmul(P.e[v], x[v + 1]));
        if (mk & 8u) acc = dsub(acc, dmul(P.nn[v], x[v + P.nx]));
        if (r) r[v] = acc;
        ra = nan_skip_abs(acc);
    }
    if (rmax) warp_max_commit(rmax, ra);
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
