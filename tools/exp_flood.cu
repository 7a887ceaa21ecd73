// Tuning experiment (not part of the product): times variants of the fused flood solve step of
// paper_1904_04093_b200/csrc/kernels.cuh on a symmetric grid Laplacian in the DIA layout.
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -fmad=false -o tools/exp_flood tools/exp_flood.cu
//   tools/exp_flood 2 2048      (2-D, 2048^2, S = 4)      tools/exp_flood 3 256   (3-D, 256^3, S = 6)
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "../paper_1904_04093_b200/csrc/kernels.cuh"

#define SYM_ROWS 1

using namespace bgabp;

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e_ = (x);                                                              \
        if (e_ != cudaSuccess) {                                                           \
            std::printf("CUDA %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

// the fused step as of commit 05b7882 (x in two plain buffers), for A/B timing
namespace bgabp {
template <int S, bool DELTA, bool SYM, int MINB = 4, bool DEFER = true, bool RES = true, bool ASYNC = false,
          bool UNC = true>
static __global__ void __launch_bounds__(256, MINB) k_old_solve(DiaP P, const double* __restrict__ b, double2* m0,
                                                              double2* m1, double* x0, double* x1, Ctrl* ctrl,
                                                              unsigned long long* spread) {
    if (ld_ctrl(&ctrl->done)) return;
    const int t = ld_ctrl(&ctrl->step);
    const double2* __restrict__ min = (t & 1) ? m0 : m1;
    double2* __restrict__ mout = (t & 1) ? m1 : m0;
    double* __restrict__ xw = ((t - 1) & 1) ? x1 : x0;        // x(t-1)
    const double* __restrict__ xr = ((t - 2) & 1) ? x1 : x0;  // x(t-2)
    const int n = P.n;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const bool res = RES && t >= 3;
    double dmax = 0.0, rabs = 0.0;
    // ASYNC: stage x(t-2) at j and j+off_s for the whole block into shared memory with LDGSTS
    // before the sweep, so the residual's loads are in flight during the message work without
    // holding registers.  Requires blockDim.x == 256.
    __shared__ double xs[ASYNC ? (S + 1) * 256 : 1];
    if (ASYNC && res) {
#pragma unroll
        for (int s = 0; s <= S; ++s) {
            const int o = s < S ? P.off[s] : 0;
            const long long q = (long long)j + o;
            cp_async8(&xs[s * 256 + threadIdx.x], xr + (q >= 0 && q < n ? q : 0), q >= 0 && q < n);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    }
    if (j < n) {
        const uint32_t mk = P.mask[j];
        const double dj = P.diag[j];
        const double bj = b[j];
        double sig = 0.0, acc = bj;
        double2 in[S];
        double cc[S], xn[S], rv[S];
        double xj = 0.0;
        // UNC: issue every load at once, independent of the mask (slot-major arrays are full
        // size, indices are clamped; the mask still selects every term below).  Predicating the
        // loads on the mask serialises a second DRAM round trip behind the mask load (ncu: the
        // mask test and the first message use were the two hottest stall sites).
#pragma unroll
        for (int s = 0; s < S; ++s) {
            in[s] = make_double2(0.0, 0.0);
            cc[s] = 0.0;
            xn[s] = 0.0;
            rv[s] = 0.0;
            const bool pin = UNC || (mk & (1u << s)), pout = UNC || (mk & (1u << (16 + s)));
            if (pin) in[s] = __ldg(min + s * n + j);
            // symmetric A stores every undirected edge twice; read the negative-offset slots from
            // the partner's positive slot (A_{j-d,j} = A_{j,j-d} = c[rev s][j-d]): same bits, and
            // those lines were just fetched for node j-d, so the coefficient DRAM traffic halves
            if (pout) {
                const double v = __ldg(SYM && s < P.nneg ? P.c + P.rev[s] * n + max(j + P.off[s], 0) : P.c + s * n + j);
                cc[s] = (mk & (1u << (16 + s))) ? v : 0.0;
            }
            if (!DEFER && res && pin) {
                const int q = j + P.off[s];
                xn[s] = xr[q < 0 ? 0 : (q >= n ? n - 1 : q)];
                if (!SYM) rv[s] = __ldg(P.rowv + s * n + j);
            }
        }
        if (!DEFER && res) xj = xr[j];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == P.nneg) sig = dadd(sig, dj);
            if (mk & (1u << s)) {
                acc = dadd(acc, in[s].y);
                if (mk & (1u << (16 + s))) sig = dadd(sig, dmul(in[s].x, cc[s]));
            }
        }
        if (P.nneg == S) sig = dadd(sig, dj);
        if (t >= 2) {  // x-stage of sweep t-1
            xw[j] = ddiv(acc, sig);
            if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
        }
        if (!DEFER && res) {  // residual of x(t-2) in CSR order (sparse.cpp:108-114)
            double r = bj;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xj));
                if (mk & (1u << s)) r = dsub(r, dmul(SYM ? cc[s] : rv[s], xn[s]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xj));
            rabs = nan_skip_abs(r);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!(mk & (1u << (16 + s)))) continue;
            const double den = dsub(sig, dmul(in[s].x, cc[s]));
            const int k = j + P.off[s];
            if (fabs(den) < kPivotFloor)
                atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)k);
            const double nl = ddiv(-cc[s], den);
            const double nm = dmul(nl, dsub(acc, in[s].y));
            double2* dst = mout + P.rev[s] * n + k;
            if (DELTA) {
                const double2 o = min[P.rev[s] * n + k];
                dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
            }
            *dst = make_double2(nl, nm);
        }
        if (ASYNC && res) {
            cp_async_wait_all();  // own copies only: each thread reads back what it staged
            double r = bj;
            const double xjj = xs[S * 256 + threadIdx.x];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xjj));
                if (mk & (1u << s))
                    r = dsub(r, dmul(SYM ? cc[s] : __ldg(P.rowv + s * n + j), xs[s * 256 + threadIdx.x]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xjj));
            rabs = nan_skip_abs(r);
        } else if (DEFER && res) {
            double r = bj;
            const double xjj = xr[j];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (mk & (1u << s)) {
                    xn[s] = xr[j + P.off[s]];
                    if (!SYM) rv[s] = __ldg(P.rowv + s * n + j);
                }
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xjj));
                if (mk & (1u << s)) r = dsub(r, dmul(SYM ? cc[s] : rv[s], xn[s]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xjj));
            rabs = nan_skip_abs(r);
        }
    }
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
    if (DELTA) warp_max_spread(spread + (size_t)(4 + (t & 3)) * kSpread, dmax);
}

template <int S, bool DELTA, bool SYM, int MINB = 4, bool DEFER = true, bool RES = true, bool ASYNC = false,
          bool UNC = true>
static __global__ void __launch_bounds__(256, MINB) k_old_nosm(DiaP P, const double* __restrict__ b, double2* m0,
                                                              double2* m1, double* x0, double* x1, Ctrl* ctrl,
                                                              unsigned long long* spread) {
    if (ld_ctrl(&ctrl->done)) return;
    const int t = ld_ctrl(&ctrl->step);
    const double2* __restrict__ min = (t & 1) ? m0 : m1;
    double2* __restrict__ mout = (t & 1) ? m1 : m0;
    double* __restrict__ xw = ((t - 1) & 1) ? x1 : x0;        // x(t-1)
    const double* __restrict__ xr = ((t - 2) & 1) ? x1 : x0;  // x(t-2)
    const int n = P.n;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const bool res = RES && t >= 3;
    double dmax = 0.0, rabs = 0.0;
    // ASYNC: stage x(t-2) at j and j+off_s for the whole block into shared memory with LDGSTS
    // before the sweep, so the residual's loads are in flight during the message work without
    // holding registers.  Requires blockDim.x == 256.
    double* xs = nullptr;
    if (ASYNC && res) {
#pragma unroll
        for (int s = 0; s <= S; ++s) {
            const int o = s < S ? P.off[s] : 0;
            const long long q = (long long)j + o;
            cp_async8(&xs[s * 256 + threadIdx.x], xr + (q >= 0 && q < n ? q : 0), q >= 0 && q < n);
        }
        asm volatile("cp.async.commit_group;\n" ::);
    }
    if (j < n) {
        const uint32_t mk = P.mask[j];
        const double dj = P.diag[j];
        const double bj = b[j];
        double sig = 0.0, acc = bj;
        double2 in[S];
        double cc[S], xn[S], rv[S];
        double xj = 0.0;
        // UNC: issue every load at once, independent of the mask (slot-major arrays are full
        // size, indices are clamped; the mask still selects every term below).  Predicating the
        // loads on the mask serialises a second DRAM round trip behind the mask load (ncu: the
        // mask test and the first message use were the two hottest stall sites).
#pragma unroll
        for (int s = 0; s < S; ++s) {
            in[s] = make_double2(0.0, 0.0);
            cc[s] = 0.0;
            xn[s] = 0.0;
            rv[s] = 0.0;
            const bool pin = UNC || (mk & (1u << s)), pout = UNC || (mk & (1u << (16 + s)));
            if (pin) in[s] = __ldg(min + s * n + j);
            // symmetric A stores every undirected edge twice; read the negative-offset slots from
            // the partner's positive slot (A_{j-d,j} = A_{j,j-d} = c[rev s][j-d]): same bits, and
            // those lines were just fetched for node j-d, so the coefficient DRAM traffic halves
            if (pout) {
                const double v = __ldg(SYM && s < P.nneg ? P.c + P.rev[s] * n + max(j + P.off[s], 0) : P.c + s * n + j);
                cc[s] = (mk & (1u << (16 + s))) ? v : 0.0;
            }
            if (!DEFER && res && pin) {
                const int q = j + P.off[s];
                xn[s] = xr[q < 0 ? 0 : (q >= n ? n - 1 : q)];
                if (!SYM) rv[s] = __ldg(P.rowv + s * n + j);
            }
        }
        if (!DEFER && res) xj = xr[j];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == P.nneg) sig = dadd(sig, dj);
            if (mk & (1u << s)) {
                acc = dadd(acc, in[s].y);
                if (mk & (1u << (16 + s))) sig = dadd(sig, dmul(in[s].x, cc[s]));
            }
        }
        if (P.nneg == S) sig = dadd(sig, dj);
        if (t >= 2) {  // x-stage of sweep t-1
            xw[j] = ddiv(acc, sig);
            if (fabs(sig) < kPivotFloor) atomicMin(&ctrl->npiv[(t - 1) & 3], (unsigned long long)j);
        }
        if (!DEFER && res) {  // residual of x(t-2) in CSR order (sparse.cpp:108-114)
            double r = bj;
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xj));
                if (mk & (1u << s)) r = dsub(r, dmul(SYM ? cc[s] : rv[s], xn[s]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xj));
            rabs = nan_skip_abs(r);
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (!(mk & (1u << (16 + s)))) continue;
            const double den = dsub(sig, dmul(in[s].x, cc[s]));
            const int k = j + P.off[s];
            if (fabs(den) < kPivotFloor)
                atomicMin(&ctrl->epiv[t & 3], ((unsigned long long)j << 32) | (unsigned)k);
            const double nl = ddiv(-cc[s], den);
            const double nm = dmul(nl, dsub(acc, in[s].y));
            double2* dst = mout + P.rev[s] * n + k;
            if (DELTA) {
                const double2 o = min[P.rev[s] * n + k];
                dmax = fmax(dmax, fmax(nan_skip_abs(dsub(nl, o.x)), nan_skip_abs(dsub(nm, o.y))));
            }
            *dst = make_double2(nl, nm);
        }
        if (ASYNC && res) {
            cp_async_wait_all();  // own copies only: each thread reads back what it staged
            double r = bj;
            const double xjj = xs[S * 256 + threadIdx.x];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xjj));
                if (mk & (1u << s))
                    r = dsub(r, dmul(SYM ? cc[s] : __ldg(P.rowv + s * n + j), xs[s * 256 + threadIdx.x]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xjj));
            rabs = nan_skip_abs(r);
        } else if (DEFER && res) {
            double r = bj;
            const double xjj = xr[j];
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (mk & (1u << s)) {
                    xn[s] = xr[j + P.off[s]];
                    if (!SYM) rv[s] = __ldg(P.rowv + s * n + j);
                }
            }
#pragma unroll
            for (int s = 0; s < S; ++s) {
                if (s == P.nneg) r = dsub(r, dmul(dj, xjj));
                if (mk & (1u << s)) r = dsub(r, dmul(SYM ? cc[s] : rv[s], xn[s]));
            }
            if (P.nneg == S) r = dsub(r, dmul(dj, xjj));
            rabs = nan_skip_abs(r);
        }
    }
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
    if (DELTA) warp_max_spread(spread + (size_t)(4 + (t & 3)) * kSpread, dmax);
}


// the current node body, launched with x(t-1) / x(t-2) as two separately passed buffers
template <int S, bool SYM, int MINB, bool DEFER>
static __global__ void __launch_bounds__(256, MINB) k_new_x01(DiaP P, const double* __restrict__ b, double2* m0,
                                                              double2* m1, double* x0, double* x1, Ctrl* ctrl,
                                                              unsigned long long* spread) {
    if (ld_ctrl(&ctrl->done)) return;
    const int t = ld_ctrl(&ctrl->step);
    const double2* __restrict__ min = (t & 1) ? m0 : m1;
    double2* __restrict__ mout = (t & 1) ? m1 : m0;
    double* __restrict__ xw = ((t - 1) & 1) ? x1 : x0;
    const double* __restrict__ xr = ((t - 2) & 1) ? x1 : x0;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const bool res = t >= 3;
    double dmax = 0.0, rabs = 0.0;
    if (j < P.n) flood_solve_node<S, false, SYM, DEFER, true, false, false>(P, b, min, mout, xw, xr, ctrl, t, res, j, rabs, dmax);
    if (res) warp_max_spread(spread + (size_t)((t - 2) & 3) * kSpread, rabs);
}

// residual variants: UNC = loads independent of the mask; RED = 0 none, 1 block + one atomic
// (warp_max_commit), 2 spread slots
template <int S, bool SYM, bool UNC, int RED>
static __global__ void __launch_bounds__(256) k_res_var(DiaP P, const double* __restrict__ b,
                                                        const double* __restrict__ x, double* __restrict__ r,
                                                        unsigned long long* rmax) {
    const int n = P.n;
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    double a = 0.0;
    if (j < n) {
        const uint32_t mk = P.mask[j];
        const double dj = P.diag[j], xj = x[j];
        double acc = b[j];
        double cv[S], xv[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool p = UNC || (mk & (1u << s));
            cv[s] = 0.0;
            xv[s] = 0.0;
            if (p) {
                const int q = j + P.off[s];
                const int qc = q < 0 ? 0 : (q >= n ? n - 1 : q);
                cv[s] = __ldg(SYM && s < P.nneg ? P.rowv + (size_t)P.rev[s] * n + qc : P.rowv + (size_t)s * n + j);
                xv[s] = __ldg(x + qc);
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == P.nneg) acc = dsub(acc, dmul(dj, xj));
            if (mk & (1u << s)) acc = dsub(acc, dmul(cv[s], xv[s]));
        }
        if (P.nneg == S) acc = dsub(acc, dmul(dj, xj));
        if (r) r[j] = acc;
        a = nan_skip_abs(acc);
    }
    if (RED == 1) warp_max_commit(rmax, a);
    if (RED == 2) warp_max_spread(rmax, a);
    if (RED == 5) {  // warp max to a per-warp partial, folded by k_fold_partials
        unsigned long long bits = __double_as_longlong(a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = ot > bits ? ot : bits;
        }
        if ((threadIdx.x & 31) == 0) rmax[(blockIdx.x * blockDim.x + threadIdx.x) >> 5] = bits;
    }
    if (RED >= 6 && RED <= 7) {  // 6: block max to a per-block partial (plain store); 7: atomic into 1024 slots
        __shared__ unsigned long long part2[8];
        unsigned long long bits = __double_as_longlong(a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = ot > bits ? ot : bits;
        }
        if ((threadIdx.x & 31) == 0) part2[threadIdx.x >> 5] = bits;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < 8; ++k) bits = part2[k] > bits ? part2[k] : bits;
            if (RED == 6) rmax[blockIdx.x] = bits;
            else if (bits) atomicMax(rmax + (blockIdx.x & 1023), bits);
        }
    }
    if (RED >= 3 && RED <= 4) {  // block max, then one fire-and-forget atomic (3: one word, 4: 64 block-indexed slots)
        __shared__ unsigned long long part[8];
        unsigned long long bits = __double_as_longlong(a);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long ot = __shfl_xor_sync(0xffffffffu, bits, o);
            bits = ot > bits ? ot : bits;
        }
        if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = bits;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int k = 1; k < 8; ++k) bits = part[k] > bits ? part[k] : bits;
            if (bits) atomicMax(RED == 3 ? rmax : rmax + (blockIdx.x & 63), bits);
        }
    }
}

// grid-stride residual: a fixed number of blocks, one block-level max and one atomic per block
template <int S, bool SYM, bool UNC>
static __global__ void __launch_bounds__(256) k_res_gs(DiaP P, const double* __restrict__ b,
                                                       const double* __restrict__ x, double* __restrict__ r,
                                                       unsigned long long* rmax) {
    const int n = P.n;
    double a = 0.0;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < n; j += gridDim.x * blockDim.x) {
        const uint32_t mk = P.mask[j];
        const double dj = P.diag[j], xj = x[j];
        double acc = b[j];
        double cv[S], xv[S];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const bool p = UNC || (mk & (1u << s));
            cv[s] = 0.0;
            xv[s] = 0.0;
            if (p) {
                const int q = j + P.off[s];
                const int qc = q < 0 ? 0 : (q >= n ? n - 1 : q);
                cv[s] = __ldg(SYM && s < P.nneg ? P.rowv + (size_t)P.rev[s] * n + qc : P.rowv + (size_t)s * n + j);
                xv[s] = __ldg(x + qc);
            }
        }
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == P.nneg) acc = dsub(acc, dmul(dj, xj));
            if (mk & (1u << s)) acc = dsub(acc, dmul(cv[s], xv[s]));
        }
        if (P.nneg == S) acc = dsub(acc, dmul(dj, xj));
        if (r) r[j] = acc;
        a = fmax(a, nan_skip_abs(acc));
    }
    warp_max_commit(rmax, a);
}

static __global__ void __launch_bounds__(1024) k_fold_partials(const unsigned long long* __restrict__ part, int np,
                                                              unsigned long long* out) {
    unsigned long long m = 0ull;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < np; i += gridDim.x * blockDim.x) m = part[i] > m ? part[i] : m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long ot = __shfl_xor_sync(0xffffffffu, m, o);
        m = ot > m ? ot : m;
    }
    if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// residual with PPT nodes per thread (block-strided), one block max + atomic at the end
template <int S, int PPT>
static __global__ void __launch_bounds__(256) k_res_ppt(DiaP P, const double* __restrict__ b,
                                                        const double* __restrict__ x, double* __restrict__ r,
                                                        unsigned long long* rmax) {
    const int n = P.n;
    const int j0 = blockIdx.x * blockDim.x * PPT + threadIdx.x;
    double a = 0.0;
    uint32_t mk[PPT];
    double cv[PPT][S], xv[PPT][S], dj[PPT], xj[PPT], bj[PPT];
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
        const int j = min(j0 + u * (int)blockDim.x, n - 1);
        mk[u] = P.mask[j];
        dj[u] = P.diag[j];
        xj[u] = x[j];
        bj[u] = b[j];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            const int q = j + P.off[s];
            const int qc = q < 0 ? 0 : (q >= n ? n - 1 : q);
            cv[u][s] = __ldg(s < P.nneg ? P.rowv + (size_t)P.rev[s] * n + qc : P.rowv + (size_t)s * n + j);
            xv[u][s] = __ldg(x + qc);
        }
    }
#pragma unroll
    for (int u = 0; u < PPT; ++u) {
        const int j = j0 + u * (int)blockDim.x;
        if (j >= n) continue;
        double acc = bj[u];
#pragma unroll
        for (int s = 0; s < S; ++s) {
            if (s == P.nneg) acc = dsub(acc, dmul(dj[u], xj[u]));
            if (mk[u] & (1u << s)) acc = dsub(acc, dmul(cv[u][s], xv[u][s]));
        }
        if (P.nneg == S) acc = dsub(acc, dmul(dj[u], xj[u]));
        if (r) r[j] = acc;
        a = fmax(a, nan_skip_abs(acc));
    }
    block_max_red(rmax, a);
}
}  // namespace bgabp

template <class T>
T* up(const std::vector<T>& v) {
    T* d;
    CK(cudaMalloc(&d, sizeof(T) * v.size()));
    CK(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return d;
}

template <int S>
void run(int N) {
    const int dims = S / 2;
    long long nn = 1;
    for (int d = 0; d < dims; ++d) nn *= N;
    const int n = (int)nn;
    DiaP P;
    std::memset(&P, 0, sizeof(P));
    P.n = n;
    P.j0 = 0;
    P.j1 = n;
    P.gofs = 0;
    P.S = S;
    P.nneg = S / 2;
    std::vector<int> st;
    int stride = 1;
    for (int d = 0; d < dims; ++d) {
        st.push_back(stride);
        stride *= N;
    }
    for (int s = 0; s < S; ++s) {
        P.off[s] = s < S / 2 ? -st[S / 2 - 1 - s] : st[s - S / 2];
        P.rev[s] = S - 1 - s;
    }
    std::vector<uint32_t> mask(n);
    std::vector<double> c((size_t)S * n, 0.0), diag(n, 2.0 * dims + 0.01), b(n);
    long long E = 0;
    std::vector<int> co(dims);
    for (int j = 0; j < n; ++j) {
        int rem = j;
        for (int d = 0; d < dims; ++d) {
            co[d] = rem % N;
            rem /= N;
        }
        for (int s = 0; s < S; ++s) {
            const int d = s < S / 2 ? (S / 2 - 1 - s) : (s - S / 2);
            const bool ok = s < S / 2 ? co[d] > 0 : co[d] < N - 1;
            if (ok) {
                mask[j] |= (1u << s) | (1u << (16 + s));
                c[(size_t)s * n + j] = -1.0;
                ++E;
            }
        }
        b[j] = std::sin(0.001 * j);
    }
    P.mask = up(mask);
    P.c = up(c);
    P.rowv = getenv("EXP_SHARED_ROWV") ? P.c : up(c);  // nonsymmetric variants read their own row copy
    P.diag = up(diag);
    double* db = up(b);
    double2 *m0, *m1;
    double *xr, *hist;
    CK(cudaMalloc(&m0, sizeof(double2) * S * n));
    CK(cudaMalloc(&m1, sizeof(double2) * S * n));
    CK(cudaMemset(m0, 0, sizeof(double2) * S * n));
    CK(cudaMemset(m1, 0, sizeof(double2) * S * n));
    CK(cudaMalloc(&xr, sizeof(double) * kXRing * n));
    CK(cudaMemset(xr, 0, sizeof(double) * kXRing * n));
    CK(cudaMalloc(&hist, sizeof(double) * 100000));
    Ctrl* ctrl;
    unsigned long long* spread;
    CK(cudaMalloc(&ctrl, sizeof(Ctrl)));
    CK(cudaMalloc(&spread, 8 * 64 * 8));
    CK(cudaMemset(spread, 0, 8 * 64 * 8));
    auto reset = [&]() {
        Ctrl h;
        std::memset(&h, 0, sizeof(h));
        for (int q = 0; q < 4; ++q) h.epiv[q] = h.npiv[q] = kNone;
        h.opiv = kNone;
        h.step = 1;
        h.r0 = 1.0;
        h.tol = 0.0;
        h.divergence = 1e300;
        h.max_iter = 1 << 30;
        CK(cudaMemcpy(ctrl, &h, sizeof(h), cudaMemcpyHostToDevice));
    };
    const unsigned g = (n + 255) / 256;
    const double bytes = 40.0 * E + 32.0 * n;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int steps = 40;
    auto timeit = [&](const char* name, auto&& launch) {
        reset();
        for (int k = 0; k < 5; ++k) launch();
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        for (int k = 0; k < steps; ++k) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double us = ms * 1e3 / steps;
        std::printf("S=%d %-44s %8.2f us/step  %7.1f GB/s  %.3f of 6557\n", S, name, us, bytes / us / 1e3,
                    bytes / us / 1e3 / 6557.4);
    };
#define W(NAME, MINB, DEFER, UNC)                                                                             \
    timeit(NAME, [&] {                                                                                        \
        k_flood_solve_dia<S, false, true, MINB, DEFER, UNC><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread); \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                                   \
    });
#define U(NAME, MINB, DEFER)                                                                                 \
    timeit(NAME, [&] {                                                                                        \
        P.uniform = 1;                                                                                        \
        k_flood_solve_dia<S, false, true, MINB, DEFER, true, true><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread); \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                                   \
        P.uniform = 0;                                                                                        \
    });
    if (getenv("EXP_RESIDUAL")) {
        double* rr;
        CK(cudaMalloc(&rr, sizeof(double) * n));
        const double rbytes = 8.0 * n * 4 + 4.0 * n + 8.0 * E / 2 * (SYM_ROWS ? 1 : 2);
        auto rt = [&](const char* name, auto&& launch) {
            for (int k = 0; k < 5; ++k) launch();
            CK(cudaDeviceSynchronize());
            cudaEventRecord(e0);
            for (int k = 0; k < steps; ++k) launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            CK(cudaGetLastError());
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double us = ms * 1e3 / steps;
            std::printf("S=%d %-44s %8.2f us  %7.1f GB/s\n", S, name, us, rbytes / us / 1e3);
        };
        rt("residual (product k_residual_dia, r + rmax)", [&] { k_residual_dia<S, true><<<g, 256>>>(P, db, xr, rr, spread, ctrl, MODE_PLAIN); });
        rt("residual (product, rmax only)", [&] { k_residual_dia<S, true><<<g, 256>>>(P, db, xr, nullptr, spread, ctrl, MODE_PLAIN); });
        rt("var predicated, block atomic", [&] { k_res_var<S, true, false, 1><<<g, 256>>>(P, db, xr, rr, spread); });
        rt("var UNC, block atomic", [&] { k_res_var<S, true, true, 1><<<g, 256>>>(P, db, xr, rr, spread); });
        rt("var UNC, spread", [&] { k_res_var<S, true, true, 2><<<g, 256>>>(P, db, xr, rr, spread); });
        rt("var UNC, block RED no precheck", [&] { k_res_var<S, true, true, 3><<<g, 256>>>(P, db, xr, rr, spread); });
        rt("var UNC, block RED 64 slots", [&] { k_res_var<S, true, true, 4><<<g, 256>>>(P, db, xr, rr, spread); });
        unsigned long long* parts;
        const int np = (int)((size_t)g * 256 / 32);
        CK(cudaMalloc(&parts, sizeof(unsigned long long) * np));
        rt("var UNC, warp partials + fold kernel", [&] {
            k_res_var<S, true, true, 5><<<g, 256>>>(P, db, xr, rr, parts);
            k_fold_partials<<<148, 1024>>>(parts, np, spread);
        });
        unsigned long long* bparts;
        CK(cudaMalloc(&bparts, sizeof(unsigned long long) * (g + 1024)));
        rt("var UNC, block partial store (no atomic)", [&] { k_res_var<S, true, true, 6><<<g, 256>>>(P, db, xr, rr, bparts); });
        rt("var UNC, block atomic 1024 slots", [&] { k_res_var<S, true, true, 7><<<g, 256>>>(P, db, xr, rr, bparts); });
        rt("var UNC, no reduction + k_inf_norm over r", [&] {
            k_res_var<S, true, true, 0><<<g, 256>>>(P, db, xr, rr, spread);
            k_inf_norm<<<1184, 256>>>(rr, n, spread);
        });
        rt("PPT=2 block RED", [&] { k_res_ppt<S, 2><<<(n + 511) / 512, 256>>>(P, db, xr, rr, spread); });
        rt("PPT=4 block RED", [&] { k_res_ppt<S, 4><<<(n + 1023) / 1024, 256>>>(P, db, xr, rr, spread); });
        rt("var UNC, no reduction", [&] { k_res_var<S, true, true, 0><<<g, 256>>>(P, db, xr, rr, spread); });
        for (int gb : {148 * 4, 148 * 8, 148 * 16, 148 * 32})
            rt(gb == 592 ? "grid-stride UNC 592 blocks" : gb == 1184 ? "grid-stride UNC 1184 blocks" : gb == 2368 ? "grid-stride UNC 2368 blocks" : "grid-stride UNC 4736 blocks",
               [&] { k_res_gs<S, true, true><<<gb, 256>>>(P, db, xr, rr, spread); });
        rt("var predicated, no reduction", [&] { k_res_var<S, true, false, 0><<<g, 256>>>(P, db, xr, rr, spread); });
        return;
    }
    for (int s = 0; s < S; ++s) P.cu[s] = -1.0;
    P.du = 2.0 * dims + 0.01;
    if (!getenv("EXP_ONLY_NONSYM")) {
    U("UNIF MINB=4 DEFER", 4, true)
    U("UNIF MINB=3 DEFER", 3, true)
    U("UNIF MINB=4 early-x", 4, false)
    U("UNIF MINB=3 early-x", 3, false)
    U("UNIF MINB=2 early-x", 2, false)
    U("UNIF MINB=5 early-x", 5, false)
    U("UNIF MINB=5 DEFER", 5, true)
    U("UNIF MINB=6 early-x", 6, false)
    U("UNIF MINB=6 DEFER", 6, true)
    }
#define NS(NAME, MINB, DEFER, UNC)                                                                            \
    timeit(NAME, [&] {                                                                                        \
        k_flood_solve_dia<S, false, false, MINB, DEFER, UNC><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread);   \
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);                                                   \
    });
    timeit("OLDK NONSYM MINB=3 early-x", [&] {
        k_old_solve<S, false, false, 3, false><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    timeit("OLDK no-smem NONSYM MINB=3 early-x", [&] {
        k_old_nosm<S, false, false, 3, false><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    timeit("NEW x0/x1 NONSYM MINB=3 early-x", [&] {
        k_new_x01<S, false, 3, false><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    NS("NONSYM MINB=3 early-x", 3, false, true)
    NS("NONSYM MINB=2 early-x", 2, false, true)
    NS("NONSYM MINB=4 early-x", 4, false, true)
    NS("NONSYM MINB=3 DEFER", 3, true, true)
    NS("NONSYM MINB=2 DEFER", 2, true, true)
    NS("NONSYM MINB=4 DEFER", 4, true, true)
    NS("NONSYM MINB=3 early-x predicated", 3, false, false)
    if (getenv("EXP_ONLY_NONSYM")) return;
    W("MINB=4 DEFER predicated", 4, true, false)
    W("MINB=4 DEFER unconditional", 4, true, true)
    W("MINB=3 DEFER unconditional", 3, true, true)
    W("MINB=4 early-x unconditional", 4, false, true)
    W("MINB=3 early-x unconditional", 3, false, true)
    W("MINB=2 early-x unconditional", 2, false, true)
    timeit("MINB=3 early-x unconditional DELTA", [&] {
        k_flood_solve_dia<S, true, true, 3, false, true><<<g, 256>>>(P, db, m0, m1, xr, xr + n, ctrl, spread);
        k_solve_decide_lag2<<<1, 64>>>(ctrl, hist, spread);
    });
    cudaFree(m0);
    cudaFree(m1);
}

int main(int argc, char** argv) {
    const int dims = argc > 1 ? std::atoi(argv[1]) : 2;
    const int N = argc > 2 ? std::atoi(argv[2]) : 2048;
    if (dims == 2) run<4>(N);
    if (dims == 3) run<6>(N);
    return 0;
}
