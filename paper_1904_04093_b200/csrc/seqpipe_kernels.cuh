// Pipelined lexicographic GaBP: many sweeps of the sequential schedule in flight at once
// (reference GabpEngine::sweep_sequential + solve, gabp.cpp:49-100,
// 174-219, and the cold smoothing sweeps of multigrid.cpp:180-187).
//
// One sweep is latency-bound (k_seq_grid5: one warp per 32-row strip, critical path nx + ny - 1
// nodes).  But sweep t+1 only needs, at node (c, r), sweep t's messages from the east (c+1, r)
// and north (c, r+1) neighbours, so it can run right behind sweep t.  A launch covers a batch of
// sweeps: each block is one warp = (sweep t, strip k), numbered by an atomic ticket so that a
// block only ever waits for blocks with lower tickets (already running: no deadlock without a
// cooperative launch).  Dependencies are tagged progress counters (sweep << 32 | columns):
//   south   (t, k-1) has published column c            -- strip boundary, staged in batches
//   east    (t-1, k) has published column c+2          -- previous sweep, same strip
//   north   (t-1, k+1) has published column c+1        -- lane 31 only
// The read-only node operands (mask, b, coefficients, diagonal) are read from lane-skewed copies
// (k_pipe_skew): at every step the 32 lanes of a strip read 32 consecutive elements (one line per
// array) instead of 32 rows' streams through L1.
// Every write-after-read hazard of the in-place message array is ordered by these waits (a slot
// is rewritten by sweep t+1 only after sweep t+1's node passed a point that itself waited for
// sweep t's reader).  Messages written by other sweeps are read through L2 (ld.cg).
//
// SOLVE: each sweep writes x(t) into a ring slot, and the residual of x(t) is evaluated inside the
// wavefront from register / shuffle x values two columns behind (no extra memory traffic); the
// last block of sweep t takes the reference's stop decision for iteration t, in order.  Sweeps run
// speculatively past the decision; the ring (kPipeR slots) bounds how far, and the reported x is
// the decided iteration's slot (composed with the previous one on a pivot stop, which is exactly
// the reference's partly updated x).
#pragma once

#include "seq_kernels.cuh"

namespace bgabp {

constexpr int kPipeR = 64;
constexpr int kPipeChunk = 4096;  // sweeps per launch of a pipelined solve (engine.cu solve_run_to_end)

struct PipeRed {  // per-sweep reductions, ring slot t % kPipeR
    unsigned long long rmax, delta, opiv;
    unsigned int count, pad;
};

struct PipeP {
    SeqP P;
    const double* rowv;  // [4][n] A_{j,j+off} (residual); == P.c when A is bit-symmetric
    const double* b;
    double2* msg;              // [4][sslot] in-slot messages, lane-skewed like the operands below
    double* x;                 // SOLVE: ring [kPipeR][sslot], lane-skewed; smoothing: x of the last sweep (natural)
    unsigned long long* prog;  // [kPipeR][strips]
    PipeRed* red;              // [kPipeR]
    int* ticket;
    int* decided;  // SOLVE: last sweep whose stop test is done
    Ctrl* ctrl;
    double* hist;
    const int* order;  // ticket -> (sweep - t0) << 12 | strip, in order of 2 * sweep + strip
    int strips, t0, nsweeps;
    int gate;  // sweeps that may run ahead of the last stop decision (<= kPipeR)
    // constant-coefficient stencil (DiaP::uniform: bit-symmetric, one out-edge coefficient per
    // slot, one diagonal): the UNI kernels take cu / du instead of loading c / rowv / diag
    double cu[4], du;
    // lane-skewed read-only operands (Engine::pipe_sn): element (strip k, step s, lane i) holds
    // node (32k + i, s - i); sstep = nx + 31 steps per strip, sslot = the per-slot stride
    const uint32_t* smask;
    const double *sb, *sc, *sd, *srow;
    long long sslot;
    int sstep;
};

// lane-skewed copy of `nslots` node arrays [q][n] -> [q][sslot] (zero where the (row, column)
// falls outside the grid); consecutive elements are consecutive lanes of one strip step
template <typename T>
static __global__ void k_pipe_skew(const T* __restrict__ src, T* __restrict__ dst, int nx, int ny, int sstep,
                                   long long total, int nslots, long long sslot, long long n) {
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long per = (long long)sstep * 32, k = e / per, rem = e - k * per;
        const int s = (int)(rem >> 5), i = (int)(rem & 31);
        const long long r = k * 32 + i;
        const int c = s - i;
        const bool ok = r < ny && c >= 0 && c < nx;
        for (int q = 0; q < nslots; ++q) dst[q * sslot + e] = ok ? src[q * n + r * nx + c] : T(0);
    }
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
    return *(volatile const unsigned long long*)p;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// wait (lane 0) until `p` shows sweep `t` with at least `cols` columns; returns the columns seen.
// The flag is read with a volatile (L2) load, not ld.acquire: on sm_100 an acquire invalidates the
// SM's whole L1 (CCTL.IVALL), which wiped the read-only operands every other block on the SM keeps
// there (ncu: L1 hit rate 0.8 %).  The data the flag guards is only ever read through L2 (ld.cg)
// after the loop exits (no load is issued before the branch that depends on the flag resolves),
// and the producer's fence orders its writes before the flag.  Waiting warps back off.
__device__ __forceinline__ int pipe_wait(const unsigned long long* p, int t, int cols) {
    const unsigned long long want = ((unsigned long long)t << 32) | (unsigned)cols;
    unsigned long long v;
    int spins = 0;
    while ((v = ld_volatile_u64(p)) < want) {
        if (++spins > 16) __nanosleep(64);
    }
    asm volatile("" ::: "memory");
    const unsigned long long got = v & 0xffffffffull;  // 0xffffffff: that block stopped early
    return (v >> 32) == (unsigned long long)t && got < 0x7fffffffull ? (int)got : 0x7fffffff;
}

struct PipeNode {
    uint32_t mk;
    double cc[4], rv[4];
    double2 inE, inN;
    double b, d;
    double2 old[4];
};

// lane-skewed index of the out-slot node q of the node at skewed index e (lane `lane`): the
// south node (r-1, c) is lane - 1 one step earlier (lane 0: lane 31 of the previous strip, step
// c + 31), west / east the same lane one step earlier / later, north (r+1, c) lane + 1 one step
// later (lane 31: lane 0 of the next strip, step c); ss = elements per strip (sstep * 32)
__device__ __forceinline__ long long pipe_nbr(long long e, int q, int lane, long long ss) {
    switch (q) {
        case 0: return lane > 0 ? e - 33 : e - ss + 1023;
        case 1: return e - 32;
        case 2: return e + 32;
        default: return lane < 31 ? e + 33 : e + ss - 1023;
    }
}

// e: the node's lane-skewed index (messages and read-only operands)
template <bool DELTA, bool SOLVE, bool SYMR, bool UNI>
__device__ __forceinline__ void pipe_load(PipeNode& o, const PipeP& Q, int lane, long long e, bool valid) {
    o.mk = 0u;
    o.b = o.d = 0.0;
    o.inE = o.inN = make_double2(0.0, 0.0);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        o.cc[q] = o.rv[q] = 0.0;
        o.old[q] = make_double2(0.0, 0.0);
    }
    if (!valid) return;
    o.mk = __ldg(Q.smask + e);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        if (!UNI) o.cc[q] = __ldg(Q.sc + q * Q.sslot + e);
        if (SOLVE && !SYMR) o.rv[q] = __ldg(Q.srow + q * Q.sslot + e);
    }
    o.inE = __ldcg(Q.msg + 2 * Q.sslot + e);  // written by sweep t-1 on another SM
    o.inN = __ldcg(Q.msg + 3 * Q.sslot + e);
    o.b = __ldg(Q.sb + e);
    if (!UNI) o.d = __ldg(Q.sd + e);
    if (DELTA) {  // previous-sweep values of this node's four out-slots (only this node writes them)
        const long long ss = (long long)Q.sstep * 32;
#pragma unroll
        for (int q = 0; q < 4; ++q) {  // outside the grid (mask bit clear): any in-range element
            const long long k = pipe_nbr(e, q, lane, ss);
            o.old[q] = __ldcg(Q.msg + (size_t)(3 - q) * Q.sslot + (k < 0 ? 0 : (k >= Q.sslot ? Q.sslot - 1 : k)));
        }
    }
}

// residual term b_j - sum_k A_jk x_k in CSR column order (sparse.cpp:108-114): south, west,
// diagonal, east, north
__device__ __forceinline__ double pipe_residual(uint32_t mk, double bj, double dj, const double* rv, double xs,
                                                double xw, double xj, double xe, double xn) {
    double r = bj;
    if (mk & 1u) r = dsub(r, dmul(rv[0], xs));
    if (mk & 2u) r = dsub(r, dmul(rv[1], xw));
    r = dsub(r, dmul(dj, xj));
    if (mk & 4u) r = dsub(r, dmul(rv[2], xe));
    if (mk & 8u) r = dsub(r, dmul(rv[3], xn));
    return nan_skip_abs(r);
}

// the reference's per-iteration test for the sequential schedule (gabp.cpp:187-218)
__device__ __forceinline__ void pipe_decide(volatile Ctrl* c, double* history, int t, unsigned long long opiv,
                                            unsigned long long rmax, unsigned long long delta) {
    c->iterations = t;
    c->solx = t;
    if (opiv != kNone) {
        c->status = 1;
        c->detail_kind = 4;
        c->detail_key = opiv;
        c->done = 1;
        return;
    }
    const double r = __longlong_as_double((long long)rmax);
    history[t] = r;
    if (!isfinite(r) || r > c->divergence * c->r0) {
        c->status = 1;
        c->detail_kind = 3;
        c->done = 1;
        return;
    }
    const double dl = __longlong_as_double((long long)delta);
    if (c->stop == 0 ? (r <= c->tol) : (dl <= c->tol)) {
        c->status = 0;
        c->done = 1;
        return;
    }
    if (t >= c->max_iter) {
        c->status = 2;
        c->done = 1;
    }
}

// SYMR: A is bit-symmetric, so the residual's row coefficients are the out-edge coefficients;
// UNI (implies SYMR): constant stencil, coefficients and diagonal from Q.cu / Q.du
template <bool DELTA, bool SOLVE, bool SYMR, bool UNI = false, int MINB = 1>
static __global__ void __launch_bounds__(32, MINB) k_seq_pipe(PipeP Q) {
    constexpr unsigned FULL = 0xffffffffu;
    const int lane = threadIdx.x;
    // Tickets follow 2 * sweep + strip: every dependency of a block -- (t, k-1), (t-1, k),
    // (t-1, k+1) -- has a smaller key, and blocks are handed out roughly when they can start
    // (sweep order would park whole sweeps of warps that wait for the strips above them)
    int id = 0;
    if (lane == 0) id = atomicAdd(Q.ticket, 1);
    id = __ldg(Q.order + __shfl_sync(FULL, id, 0));
    const int t = Q.t0 + (id >> 12), strip = id & 4095;
    const int slot = t % kPipeR, pslot = (t + kPipeR - 1) % kPipeR;
    const SeqP& P = Q.P;
    const int nx = P.nx, ny = P.ny, n = P.n;
    unsigned long long* myprog = Q.prog + (size_t)slot * Q.strips + strip;
    const unsigned long long* prev_same = Q.prog + (size_t)pslot * Q.strips + strip;
    const unsigned long long* prev_next = prev_same + 1;
    const unsigned long long* south_prog = myprog - 1;
    volatile Ctrl* vc = Q.ctrl;
    const unsigned long long mytag = (unsigned long long)t << 32;

    if (!SOLVE && vc->halt) {  // an earlier smoothing call of this cycle already failed
        if (lane == 0) *(volatile unsigned long long*)myprog = mytag | 0xffffffffull;
        return;
    }
    // gate: ring slot t % R is free once sweep t - R + 1 is decided (its x(t - R) was the last use)
    if (SOLVE) {
        int go = 1;
        if (lane == 0) {
            while (true) {
                if (vc->done) {
                    go = 0;
                    break;
                }
                if (*(volatile int*)Q.decided >= t - Q.gate + 1) break;
                __nanosleep(256);
            }
        }
        go = __shfl_sync(FULL, go, 0);
        if (!go) {  // the solve already stopped: release everything waiting on this block
            if (lane == 0) *(volatile unsigned long long*)myprog = mytag | 0xffffffffull;
            return;
        }
    }

    const int r = strip * 32 + lane;
    const int r0 = strip * 32;
    const bool row_ok = r < ny;
    const bool last_lane = lane == 31 || r == ny - 1;
    const bool has_prev = t > 1;  // sweep 0 does not exist: its messages are the initial state
    const bool north_strip = strip + 1 < Q.strips && r0 + 31 + 1 < ny;
    const bool boundary = strip > 0 && r0 < ny;
    double* xt = SOLVE ? Q.x + (size_t)slot * Q.sslot : Q.x;
    const long long ss = (long long)Q.sstep * 32;
    const bool write_x = SOLVE || t == Q.t0 + Q.nsweeps - 1;
    __shared__ double2 ring_m[kSeqRing];
    __shared__ double ring_x1[kSeqRing], ring_x2[kSeqRing];  // x(t) of rows r0-1, r0-2
    int seen = 0, seenE = 0, seenN = 0;

    // column 0 of lane 0 needs the previous sweep's east message at column 1
    if (has_prev) {
        int v = 0;
        if (lane == 0) v = pipe_wait(prev_same, t - 1, min(2, nx));
        seenE = __shfl_sync(FULL, v, 0);
        __syncwarp();
    }
    PipeNode cur, nxt;
    // this lane's skewed element at step s is ebase + 32 s; row r0 - 1 (lane 31 of the previous
    // strip) at column c is pbase + 32 (c + 31)
    const long long ebase = (long long)strip * Q.sstep * 32 + lane;
    const long long pbase = (long long)(strip - 1) * Q.sstep * 32 + 31;
    pipe_load<DELTA, SOLVE, SYMR, UNI>(cur, Q, lane, ebase, row_ok && lane == 0);
    double2 west = make_double2(0.0, 0.0), north_out = make_double2(0.0, 0.0);
    double dmax = 0.0, rmax = 0.0;
    // own-row history for the residual two columns behind: x, b, diag, mask, A row of c-1 / c-2
    double xh1 = 0.0, xh2 = 0.0, xh3 = 0.0, bh1 = 0.0, bh2 = 0.0, dh1 = 0.0, dh2 = 0.0;
    double rvh1[4] = {0.0, 0.0, 0.0, 0.0}, rvh2[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t mkh1 = 0u, mkh2 = 0u;
    // lane 0 of strip > 0: the operands of row r0-1 two columns behind (its residual)
    double pb = 0.0, pd = 0.0, prv[4] = {0.0, 0.0, 0.0, 0.0};
    uint32_t pmk = 0u;
    const int steps = nx + 31 + (SOLVE ? 2 : 0);
    // two node buffers in ping-pong (a copy `cur = nxt` would wait for this step's loads)
    auto step = [&](const int s, PipeNode& cu, PipeNode& nu) {
        const int c = s - lane;
        const bool act = row_ok && c >= 0 && c < nx;
        const int j = r * nx + c;
        const long long e = ebase + 32ll * s;
        // previous sweep far enough ahead for next step's prefetch (east: lane 0 is the most
        // demanding lane; north: lane 31 reads the next strip's first row)
        if (has_prev) {
            const int needE = min(s + 3, nx), needN = north_strip ? min(s - 29, nx) : 0;
            const bool wE = seenE < needE, wN = needN > 0 && seenN < needN;
            if (wE || wN) {
                int v1 = seenE, v2 = seenN;
                if (lane == 0) {
                    if (wE) v1 = pipe_wait(prev_same, t - 1, needE);
                    if (wN) v2 = pipe_wait(prev_next, t - 1, needN);
                }
                seenE = __shfl_sync(FULL, v1, 0);
                seenN = __shfl_sync(FULL, v2, 0);
                __syncwarp();
            }
        }
        // next node: the skewed operands of step s + 1 are one coalesced line per array
        pipe_load<DELTA, SOLVE, SYMR, UNI>(nu, Q, lane, e + 32, row_ok && c + 1 >= 0 && c + 1 < nx);
        double2 south;
        south.x = __shfl_up_sync(FULL, north_out.x, 1);
        south.y = __shfl_up_sync(FULL, north_out.y, 1);
        // strip boundary: stage the previous strip's published batch (messages into row r0, and
        // x(t) of rows r0-1, r0-2 for the residual) with the whole warp
        if (boundary && s < nx && s >= seen) {
            int v = 0;
            if (lane == 0) v = pipe_wait(south_prog, t, s + 1);
            v = __shfl_sync(FULL, v, 0);
            __syncwarp();
            v = min(min(v, nx), s + kSeqRing - 4);
            // skewed: row r0 column cc is lane 0 of this strip at step cc; rows r0-1 / r0-2 are
            // lanes 31 / 30 of the previous strip at steps cc + 31 / cc + 30
            const long long mb = (long long)strip * ss, xb = mb - ss;
            for (int cc = seen + lane; cc < v; cc += 32) {
                ring_m[cc & (kSeqRing - 1)] = __ldcg(Q.msg + mb + 32ll * cc);
                if (SOLVE) {
                    ring_x1[cc & (kSeqRing - 1)] = __ldcg(xt + xb + 32ll * (cc + 31) + 31);
                    ring_x2[cc & (kSeqRing - 1)] = __ldcg(xt + xb + 32ll * (cc + 30) + 30);
                }
            }
            __syncwarp();
            seen = v;
        }
        if (act && lane == 0 && r > 0) south = ring_m[c & (kSeqRing - 1)];
        double2 nout = make_double2(0.0, 0.0);
        double xj = 0.0;
        if (act) {
            const uint32_t mk = cu.mk;
            double2 in[4];
            in[0] = (mk & 1u) ? south : make_double2(0.0, 0.0);
            in[1] = (mk & 2u) ? west : make_double2(0.0, 0.0);
            in[2] = (mk & 4u) ? cu.inE : make_double2(0.0, 0.0);
            in[3] = (mk & 8u) ? cu.inN : make_double2(0.0, 0.0);
            double cc[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) cc[q] = (mk & (1u << (16 + q))) ? (UNI ? Q.cu[q] : cu.cc[q]) : 0.0;
            double sig = 0.0, acc = cu.b;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q == 2) sig = dadd(sig, UNI ? Q.du : cu.d);
                const bool iq = mk & (1u << q), both = iq && (mk & (1u << (16 + q)));
                const double a2 = dadd(acc, in[q].y), s2 = dadd(sig, dmul(in[q].x, cc[q]));
                acc = iq ? a2 : acc;
                sig = both ? s2 : sig;
            }
            const unsigned long long pk = (unsigned long long)j << 32;
            const int off[4] = {-nx, -1, 1, nx};
            double num[4], den[4], nl[4];
            bool ok[5];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const bool oq = mk & (1u << (16 + q));
                const double d = dsub(sig, dmul(in[q].x, cc[q]));
                den[q] = oq ? d : 1.0;
                num[q] = oq ? -cc[q] : 1.0;
                nl[q] = ddiv_fast(num[q], den[q], ok[q]);
            }
            xj = ddiv_fast(acc, sig, ok[4]);
            if (!(ok[0] && ok[1] && ok[2] && ok[3] && ok[4])) {
#pragma unroll
                for (int q = 0; q < 4; ++q)
                    if (!ok[q]) nl[q] = ddiv(num[q], den[q]);
                if (!ok[4]) xj = ddiv(acc, sig);
            }
            double2 out[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) out[q] = make_double2(nl[q], dmul(nl[q], dsub(acc, in[q].y)));
            west = out[2];
            nout = out[3];
            if (fabs(sig) < kPivotFloor) atomicMin(&Q.red[slot].opiv, pk);
            if (SOLVE) xt[e] = xj;
            else if (write_x) xt[j] = xj;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (!(mk & (1u << (16 + q)))) continue;
                if (fabs(den[q]) < kPivotFloor) atomicMin(&Q.red[slot].opiv, pk | (unsigned)(j + off[q] + 1));
                if (DELTA)
                    dmax = fmax(dmax, fmax(nan_skip_abs(dsub(out[q].x, cu.old[q].x)),
                                           nan_skip_abs(dsub(out[q].y, cu.old[q].y))));
                // east- and north-going messages are consumed inside the strip by this sweep (the
                // `west` register, the south shuffle): only lane 31's north message crosses to the
                // next strip through memory.  Nothing reads the launch's final messages (the solve
                // and the smoothing calls start from zero and discard them), so the others are
                // stored only where the message delta needs the previous sweep's values.
                if (DELTA || q < 2 || (q == 3 && lane == 31))
                    Q.msg[(size_t)(3 - q) * Q.sslot + pipe_nbr(e, q, lane, ss)] = out[q];
            }
        }
        north_out = nout;
        if (SOLVE) {
            // residual of x(t) at column c-2: own row from the history, the row below from lane-1
            // (3 steps ago for it), the row above from lane+1 (its previous step)
            const double xb = __shfl_up_sync(FULL, xh3, 1);
            const double xa = __shfl_down_sync(FULL, xh1, 1);
            const int cr = c - 2;
            if (row_ok && cr >= 0 && cr < nx && (lane < 31 || r == ny - 1)) {
                const double below = lane == 0 ? ring_x1[cr & (kSeqRing - 1)] : xb;
                rmax = fmax(rmax, pipe_residual(mkh2, bh2, UNI ? Q.du : dh2, UNI ? Q.cu : rvh2, below, xh3, xh2, xh1, xa));
            }
            // lane 0 also closes row r0-1 of the previous strip (its lane 31 cannot see row r0)
            if (lane == 0 && boundary && cr >= 0 && cr < nx) {
                const double xw = cr > 0 ? ring_x1[(cr - 1) & (kSeqRing - 1)] : 0.0;
                const double xe = cr + 1 < nx ? ring_x1[(cr + 1) & (kSeqRing - 1)] : 0.0;
                rmax = fmax(rmax, pipe_residual(pmk, pb, UNI ? Q.du : pd, UNI ? Q.cu : prv, ring_x2[cr & (kSeqRing - 1)], xw,
                                                ring_x1[cr & (kSeqRing - 1)], xe, xh2));
            }
            // shift the histories; lane 0 fetches row r0-1's operands for the next step's column
            xh3 = xh2;
            xh2 = xh1;
            xh1 = xj;
            bh2 = bh1;
            if (!UNI) dh2 = dh1;
            mkh2 = mkh1;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!UNI) rvh2[q] = rvh1[q];
            bh1 = cu.b;
            if (!UNI) dh1 = cu.d;
            mkh1 = act ? cu.mk : 0u;
#pragma unroll
            for (int q = 0; q < 4; ++q)
                if (!UNI) rvh1[q] = SYMR ? cu.cc[q] : cu.rv[q];
            if (lane == 0 && boundary) {
                const int cn = c - 1;  // next step's residual column
                if (cn >= 0 && cn < nx) {
                    const long long ep = pbase + 32ll * (cn + 31);
                    pmk = __ldg(Q.smask + ep);
                    pb = __ldg(Q.sb + ep);
                    if (!UNI) pd = __ldg(Q.sd + ep);
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (!UNI) prv[q] = __ldg((SYMR ? Q.sc : Q.srow) + q * Q.sslot + ep);
                }
            }
        }
        if (act && last_lane && ((c % kSeqPublish) == kSeqPublish - 1 || c == nx - 1))
            st_release_u64(myprog, mytag | (unsigned)(c + 1));  // lane 30's x: ordered by the step's __syncwarp
        __syncwarp();
    };
    for (int s = 0; s < steps; s += 2) {
        step(s, cur, nxt);
        if (s + 1 < steps) step(s + 1, nxt, cur);
    }
    // per-sweep reductions; the last block of sweep t takes its stop decision
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        dmax = fmax(dmax, __shfl_xor_sync(FULL, dmax, o));
        rmax = fmax(rmax, __shfl_xor_sync(FULL, rmax, o));
    }
    if (lane == 0) {
        if (DELTA && dmax > 0.0) atomicMax(&Q.red[slot].delta, (unsigned long long)__double_as_longlong(dmax));
        if (SOLVE && rmax > 0.0) atomicMax(&Q.red[slot].rmax, (unsigned long long)__double_as_longlong(rmax));
        __threadfence();
        const unsigned prev = atomicAdd(&Q.red[slot].count, 1u);
        if (SOLVE && prev == (unsigned)Q.strips - 1) {
            __threadfence();
            while (!vc->done && *(volatile int*)Q.decided < t - 1) __nanosleep(32);
            PipeRed* R = Q.red + slot;
            const unsigned long long op = ld_volatile_u64(&R->opiv), rm = ld_volatile_u64(&R->rmax),
                                     dl = ld_volatile_u64(&R->delta);
            R->opiv = kNone;  // the slot is reused by sweep t + R
            R->rmax = 0ull;
            R->delta = 0ull;
            R->count = 0u;
            if (!vc->done) {
                pipe_decide(vc, Q.hist, t, op, rm, dl);
                __threadfence();
                *(volatile int*)Q.decided = t;
            }
        }
    }
}

// smoothing calls: the first failing sweep's first pivot (the reference stops there) -> ctrl->opiv
static __global__ void k_pipe_failure(Ctrl* c, PipeRed* red, int t0, int nsweeps) {
    for (int t = t0; t < t0 + nsweeps; ++t) {
        PipeRed& R = red[t % kPipeR];
        if (R.opiv != kNone && c->opiv == kNone) c->opiv = R.opiv;
        R.opiv = kNone;
        R.rmax = R.delta = 0ull;
        R.count = 0u;
    }
}

}  // namespace bgabp
