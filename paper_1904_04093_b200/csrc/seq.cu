// Host side of the pipelined lexicographic sweep (seq_kernels.cuh).
#include <algorithm>
#include <cstdlib>
#include <vector>

#include "engine.h"

namespace bgabp {

void Engine::launch_seq_sweep(const double* b, double2* msg, double* x, bool delta, unsigned long long* dslot,
                              int mode, long long xstride) {
    const int nx = grid5_nx, ny = n / grid5_nx;
    const int strips = (ny + 31) / 32;
    if (!d_progress) d_progress = static_cast<int*>(dalloc(sizeof(int) * (size_t)strips));
    ck(cudaMemsetAsync(d_progress, 0, sizeof(int) * (size_t)strips, st), "memset progress");
    SeqP P{nx, ny, n, dia.mask, dia.c, dia.diag};
    void* args[] = {&P, (void*)&b, &msg, &x, &d_progress, &d_ctrl, &dslot, &mode, &xstride};
    // every strip spins on its predecessor: a cooperative launch guarantees co-residency (or fails)
    const void* fn = delta ? (const void*)k_seq_grid5<true> : (const void*)k_seq_grid5<false>;
    ck(cudaLaunchCooperativeKernel(fn, dim3(strips), dim3(32), args, 0, st), "sequential sweep launch");
}

static __global__ void k_pipe_reset(PipeRed* red, unsigned long long* prog, int nprog, int* ints) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < kPipeR) {
        red[i].rmax = red[i].delta = 0ull;
        red[i].opiv = kNone;
        red[i].count = 0u;
    }
    for (int k = i; k < nprog; k += gridDim.x * blockDim.x) prog[k] = 0ull;
    if (i == 0) ints[0] = ints[1] = 0;
}

void Engine::pipe_setup(bool ring) {
    const int strips = (n / grid5_nx + 31) / 32;
    // the x ring must outlast the deepest gate wait: with tickets in 2 * sweep + strip order a
    // block never waits on a later ticket as long as strips + 1 < 2 * kPipeR
    if (ring && !pipe_fits()) throw InvalidArg("sequential pipeline: grid too tall for the x ring");
    if (!d_pprog || strips != pipe_strips) {
        pipe_strips = strips;
        d_pprog = static_cast<unsigned long long*>(dalloc(sizeof(unsigned long long) * (size_t)kPipeR * strips));
        d_pred = static_cast<PipeRed*>(dalloc(sizeof(PipeRed) * kPipeR));
        d_pint = static_cast<int*>(dalloc(sizeof(int) * 2));
    }
    pipe_sn = (long long)strips * (grid5_nx + 31) * 32;
    // messages and the x ring live in the lane-skewed layout for the whole launch (both start
    // from zero: the solve's and a smoothing call's fresh state), so a strip's 32 lanes load and
    // store one or two lines per array and step instead of 32 rows' sectors
    if (!d_pmsg) d_pmsg = static_cast<double2*>(dalloc(sizeof(double2) * 4 * (size_t)pipe_sn));
    if (ring && !d_xring) d_xring = static_cast<double*>(dalloc(sizeof(double) * (size_t)kPipeR * pipe_sn));
    if (!d_skb) {  // lane-skewed read-only operands, built once per handle (b: every launch)
        const int nx = grid5_nx, ny = n / grid5_nx, sstep = nx + 31;
        const unsigned g = std::min<unsigned>(nblk_host(pipe_sn), 148u * 16u);
        d_skmask = static_cast<uint32_t*>(dalloc(sizeof(uint32_t) * (size_t)pipe_sn));
        k_pipe_skew<uint32_t><<<g, 256, 0, st>>>(dia.mask, d_skmask, nx, ny, sstep, pipe_sn, 1, pipe_sn, n);
        if (!dia.uniform || getenv("BGABP_PIPE_NOUNI")) {
            d_skc = static_cast<double*>(dalloc(sizeof(double) * 4 * (size_t)pipe_sn));
            d_skdiag = static_cast<double*>(dalloc(sizeof(double) * (size_t)pipe_sn));
            k_pipe_skew<double><<<g, 256, 0, st>>>(dia.c, d_skc, nx, ny, sstep, pipe_sn, 4, pipe_sn, n);
            k_pipe_skew<double><<<g, 256, 0, st>>>(dia.diag, d_skdiag, nx, ny, sstep, pipe_sn, 1, pipe_sn, n);
            if (!symmetric) {
                d_skrow = static_cast<double*>(dalloc(sizeof(double) * 4 * (size_t)pipe_sn));
                k_pipe_skew<double><<<g, 256, 0, st>>>(dia.rowv, d_skrow, nx, ny, sstep, pipe_sn, 4, pipe_sn, n);
            }
        }
        d_skb = static_cast<double*>(dalloc(sizeof(double) * (size_t)pipe_sn));
        ck(cudaGetLastError(), "pipeline skew");
    }
}

void Engine::pipe_reset() {
    const int np = kPipeR * pipe_strips;
    ck(cudaMemsetAsync(d_pmsg, 0, sizeof(double2) * 4 * (size_t)pipe_sn, st), "memset pipeline messages");
    k_pipe_reset<<<std::max(1, std::min((np + 255) / 256, 256)), 256, 0, st>>>(d_pred, d_pprog, np, d_pint);
}

void Engine::launch_pipe(const double* b, double* x, int t0, int nsweeps, bool solve, bool delta) {
    if (nsweeps <= 0 || n == 0) return;
    PipeP Q;
    Q.P = SeqP{grid5_nx, n / grid5_nx, n, dia.mask, dia.c, dia.diag};
    Q.rowv = dia.rowv;
    Q.b = b;
    Q.msg = d_pmsg;
    Q.x = x;
    Q.prog = d_pprog;
    Q.red = d_pred;
    Q.ticket = d_pint;
    Q.decided = d_pint + 1;
    Q.ctrl = d_ctrl;
    Q.hist = d_hist;
    auto it = pipe_orders.find(nsweeps);
    if (it == pipe_orders.end()) {  // blocks in order of 2 * sweep + strip (see k_seq_pipe)
        std::vector<int> ord;
        ord.reserve((size_t)nsweeps * pipe_strips);
        for (int d = 0; d <= 2 * (nsweeps - 1) + pipe_strips - 1; ++d)
            for (int tt = std::min(nsweeps - 1, d / 2); tt >= 0; --tt) {
                const int k = d - 2 * tt;
                if (k >= pipe_strips) break;
                ord.push_back((tt << 12) | k);
            }
        int* d_ord = static_cast<int*>(dalloc(sizeof(int) * ord.size()));
        ck(cudaMemcpyAsync(d_ord, ord.data(), sizeof(int) * ord.size(), cudaMemcpyHostToDevice, st), "order");
        ck(cudaStreamSynchronize(st), "sync");
        it = pipe_orders.emplace(nsweeps, d_ord).first;
    }
    Q.order = it->second;
    Q.strips = pipe_strips;
    Q.t0 = t0;
    Q.nsweeps = nsweeps;
    ck(cudaMemsetAsync(d_pint, 0, sizeof(int), st), "ticket");
    const dim3 grid((unsigned)((long long)nsweeps * pipe_strips));
    // 64 sweeps ahead of the stop decision.  Measured on 2048^2 (constant-stencil variant, 0.31 ms
    // per iteration) and no faster: a 128-slot ring, register caps of 168 / 128 (12 / 16 warps
    // per SM, with spills: 0.34 / 0.36 ms), publishing every 4 / 16 / 32 columns, L1 prefetch
    // distances 0-40, L2 prefetch of the east / north message lines, dependency flags polled one
    // step ahead with the boundary batches loaded a step before staging, and (unsafely) relaxed
    // progress stores without the release fence (-3 %).  Two pipelines on one GPU each run at half
    // speed: the kernel is bound by resident warps x per-step latency (8 warps per SM at 214
    // registers, ~640 instructions per warp step at ~8 cycles each), see DESIGN.md 4.  A
    // 164-register build of the constant-stencil kernel (12 warps per SM) ran 0.339 ms, and 0.325
    // ms with the lane-skewed operands (0.315 at 8 warps): the SM's warp-step rate stays at ~2.9
    // per us.  The lane-skewed operands took the general-coefficient kernel 0.393 -> 0.331 ms.
    // Two rows per lane (strips of 64 rows, two independent node chains per step, bit-identical)
    // ran 0.346 ms against 0.324 in the same run, and the spin / back-off of the progress polls
    // (16 x 64 ns ... 0 x 1 us) made no difference: the rate does not follow the warp count, the
    // chains per warp or the poll pressure.
    Q.gate = kPipeR;
    {  // b of this launch in the lane-skewed layout (the multigrid smoother passes a new residual)
        const int nx = grid5_nx, ny = n / grid5_nx;
        Q.sstep = nx + 31;
        Q.sslot = pipe_sn;
        const unsigned g = std::min<unsigned>(nblk_host(pipe_sn), 148u * 16u);
        k_pipe_skew<double><<<g, 256, 0, st>>>(b, d_skb, nx, ny, Q.sstep, pipe_sn, 1, pipe_sn, n);
        Q.smask = d_skmask;
        Q.sb = d_skb;
        Q.sc = d_skc;
        Q.sd = d_skdiag;
        Q.srow = d_skrow;
    }
    const bool uni = dia.uniform != 0 && getenv("BGABP_PIPE_NOUNI") == nullptr;  // NOUNI: A/B
    if (uni) {
        for (int q = 0; q < 4; ++q) Q.cu[q] = dia.cu[q];
        Q.du = dia.du;
    }
    if (solve) {
        if (uni) {  // constant stencil (config 2): no coefficient / diagonal loads
            if (delta) k_seq_pipe<true, true, true, true><<<grid, 32, 0, st>>>(Q);
            else k_seq_pipe<false, true, true, true><<<grid, 32, 0, st>>>(Q);
        } else if (symmetric) {
            if (delta) k_seq_pipe<true, true, true><<<grid, 32, 0, st>>>(Q);
            else k_seq_pipe<false, true, true><<<grid, 32, 0, st>>>(Q);
        } else {
            if (delta) k_seq_pipe<true, true, false><<<grid, 32, 0, st>>>(Q);
            else k_seq_pipe<false, true, false><<<grid, 32, 0, st>>>(Q);
        }
    } else {
        if (uni) k_seq_pipe<false, false, true, true><<<grid, 32, 0, st>>>(Q);
        else k_seq_pipe<false, false, true><<<grid, 32, 0, st>>>(Q);
        k_pipe_failure<<<1, 1, 0, st>>>(d_ctrl, d_pred, t0, nsweeps);
    }
    ck(cudaGetLastError(), "pipelined sequential sweeps");
}

// x(t) of the pipelined solve out of its lane-skewed ring slot (natural order); on a pivot stop
// node j < p takes xs, the rest xo (the reference's partly updated x)
static __global__ void k_pipe_x_out(const double* __restrict__ xs, const double* __restrict__ xo,
                                    double* __restrict__ out, int nx, int n, int sstep, long long p) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const int r = j / nx, c = j - r * nx, i = r & 31;
    const long long e = (long long)(r >> 5) * sstep * 32 + 32ll * (c + i) + i;
    out[j] = j < p ? xs[e] : xo[e];
}

const double* Engine::pipe_x_out(int slot, int oslot, long long p) {
    k_pipe_x_out<<<nblk_host(n), 256, 0, st>>>(d_xring + (size_t)slot * pipe_sn, d_xring + (size_t)oslot * pipe_sn, d_aux,
                                          grid5_nx, n, grid5_nx + 31, p);
    ck(cudaGetLastError(), "pipeline x");
    return d_aux;
}

}  // namespace bgabp
