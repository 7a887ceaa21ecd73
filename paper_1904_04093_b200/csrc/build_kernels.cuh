// Device build of the DIA message-graph layout (build.cu, Engine::build_dia_device).
//
// The reference builds its message graph on the host (make_csr / transpose_pos, sparse.cpp:36-75;
// build_message_graph, gabp.cpp:8-27).  Here the canonical CSR goes to HBM once and these kernels
// derive everything the sweeps read: the per-node slot mask, the out-edge coefficients c[s][j],
// the row coefficients rowv[s][j], the diagonal, and the facts that pick kernel variants
// (bit-symmetric A, constant-coefficient stencil, 5-point grid without row wrap-around).  No
// transpose search is needed: the entry A_ij (row i, slot s of offset j - i) is the in-edge j->i
// of node i AND the coefficient of node j's outgoing message to i, i.e. c[rev s][j].
#pragma once

#include <cstdint>

#include "kernels.cuh"

namespace bgabp {

struct DiaOffs {
    int S;
    int off[kMaxDia], rev[kMaxDia];
};

// thread per row: scatter every off-diagonal entry into (mask, rowv) of its row node and
// (mask, c) of its column node; the diagonal into diag.  mask, c, rowv are zeroed beforehand.
static __global__ void k_dia_fill(int n, const int* __restrict__ ro, const int* __restrict__ ci,
                           const double* __restrict__ val, DiaOffs o, uint32_t* mask, double* c, double* rowv,
                           double* diag) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const int p1 = ro[i + 1];
        uint32_t in = 0u;
        for (int p = ro[i]; p < p1; ++p) {
            const int j = ci[p];
            const double v = val[p];
            if (j == i) {
                diag[i] = v;
                continue;
            }
            int s = 0;
            while (s < o.S && o.off[s] != j - i) ++s;  // <= 8 sorted offsets, found by the host scan
            if (s == o.S) continue;
            in |= 1u << s;
            rowv[(size_t)s * n + i] = v;
            const int rs = o.rev[s];
            c[(size_t)rs * n + j] = v;
            atomicOr(&mask[j], 1u << (16 + rs));
        }
        if (in) atomicOr(&mask[i], in);
    }
}

// layout facts, reduced over all nodes
struct DiaFacts {
    unsigned asym;                  // some in/out pair differs in structure or in bits
    unsigned wrap;                  // a 5-point grid row has a west edge at its first / east at its last node
    unsigned long long cmin[kMaxDia], cmax[kMaxDia];  // bit patterns of c over the slot's out-edges
    unsigned long long dmin, dmax;  // bit patterns of the diagonal
};

__device__ __forceinline__ unsigned long long warp_min_u64(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}
__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}

// gx > 0: also test the 5-point grid wrap-around condition for rows of gx nodes
static __global__ void k_dia_facts(int n, int S, const uint32_t* __restrict__ mask, const double* __restrict__ c,
                            const double* __restrict__ rowv, const double* __restrict__ diag, int gx,
                            DiaFacts* out) {
    unsigned asym = 0u, wrap = 0u;
    unsigned long long cmin[kMaxDia], cmax[kMaxDia];
    for (int s = 0; s < kMaxDia; ++s) {
        cmin[s] = ~0ull;
        cmax[s] = 0ull;
    }
    unsigned long long dmin = ~0ull, dmax = 0ull;
    const unsigned long long* cb = reinterpret_cast<const unsigned long long*>(c);
    const unsigned long long* rb = reinterpret_cast<const unsigned long long*>(rowv);
    const unsigned long long* db = reinterpret_cast<const unsigned long long*>(diag);
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        const uint32_t mk = mask[i];
        if ((mk & 0xffffu) != (mk >> 16)) asym = 1u;
        for (int s = 0; s < S; ++s) {
            if (!(mk & (1u << (16 + s)))) continue;
            const unsigned long long v = cb[(size_t)s * n + i];
            if ((mk & (1u << s)) && rb[(size_t)s * n + i] != v) asym = 1u;
            cmin[s] = v < cmin[s] ? v : cmin[s];
            cmax[s] = v > cmax[s] ? v : cmax[s];
        }
        const unsigned long long d = db[i];
        dmin = d < dmin ? d : dmin;
        dmax = d > dmax ? d : dmax;
        if (gx > 0) {
            const int col = i % gx;
            if (col == 0 && (mk & (2u | (2u << 16)))) wrap = 1u;
            if (col == gx - 1 && (mk & (4u | (4u << 16)))) wrap = 1u;
        }
    }
    asym = __any_sync(0xffffffffu, asym) ? 1u : 0u;
    wrap = __any_sync(0xffffffffu, wrap) ? 1u : 0u;
    for (int s = 0; s < S; ++s) {
        cmin[s] = warp_min_u64(cmin[s]);
        cmax[s] = warp_max_u64(cmax[s]);
    }
    dmin = warp_min_u64(dmin);
    dmax = warp_max_u64(dmax);
    if ((threadIdx.x & 31) == 0) {
        if (asym) atomicOr(&out->asym, 1u);
        if (wrap) atomicOr(&out->wrap, 1u);
        for (int s = 0; s < S; ++s) {
            if (cmin[s] != ~0ull) atomicMin(&out->cmin[s], cmin[s]);
            if (cmax[s]) atomicMax(&out->cmax[s], cmax[s]);
        }
        atomicMin(&out->dmin, dmin);
        atomicMax(&out->dmax, dmax);
    }
}

// CSR position -> message slot (s * n + i for the in-edge of row i at offset s; -1 on the diagonal),
// for get/set_state in CSR order (parity paths only, built on first use)
static __global__ void k_dia_csr2slot(int n, const int* __restrict__ ro, const int* __restrict__ ci, DiaOffs o,
                               long long* out) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        for (int p = ro[i]; p < ro[i + 1]; ++p) {
            const int j = ci[p];
            if (j == i) {
                out[p] = -1;
                continue;
            }
            int s = 0;
            while (s < o.S && o.off[s] != j - i) ++s;
            out[p] = s < o.S ? (long long)s * n + i : -1;
        }
    }
}

static __global__ void k_fill_value(double* v, long long n, double a) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
        v[i] = a;
}

}  // namespace bgabp
