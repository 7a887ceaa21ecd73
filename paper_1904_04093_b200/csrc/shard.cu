// Sharded flood solve behind the C-ABI (include/gabp_b200.h, bgabp_shard_* / bgabp_ipc_*):
// one contiguous row block per shard.  Two transports: pack / unpack + a caller-driven MAX
// all-reduce (torch.distributed, paper_1904_04093_b200/shard.py), and peer memory, where the
// fused step stores halos and stop words straight into the neighbours' buffers (kernels.cuh:
// peer_msg / peer_x / k_shard_fold_p2p / k_shard_decide_p2p).
#include <algorithm>
#include <cstring>
#include <string>
#include <vector>

#include "engine.h"

namespace bgabp {

// captured multi-shard peer-memory iterations (bgabp_shard_p2p_steps), dropped with any of their
// engines or when one of them reallocates a captured buffer
// What a captured iteration bakes in per shard: its buffers (history generation), its node range
// and peer pointers (peer generation), and the solve's stop rule and right-hand side.
struct P2PKey {
    long long hist_gen, peer_gen;
    int stop;
    const double* b;
    bool operator==(const P2PKey& o) const {
        return hist_gen == o.hist_gen && peer_gen == o.peer_gen && stop == o.stop && b == o.b;
    }
};
static P2PKey p2p_key(const Engine& E) { return {E.hist_gen, E.peer_gen, E.solve_stop, E.solve_b}; }

struct P2PGraph {
    std::vector<Engine*> engines;
    std::vector<P2PKey> gens;
    cudaGraphExec_t exec = nullptr;
    std::vector<cudaEvent_t> join;
    cudaEvent_t fork = nullptr;
};
static std::vector<P2PGraph>& p2p_graphs() {
    static std::vector<P2PGraph>* g = new std::vector<P2PGraph>();
    return *g;
}
void p2p_forget(Engine* e) {
    auto& all = p2p_graphs();
    for (size_t i = 0; i < all.size();) {
        if (std::find(all[i].engines.begin(), all[i].engines.end(), e) != all[i].engines.end()) {
            if (all[i].exec) cudaGraphExecDestroy(all[i].exec);
            for (auto ev : all[i].join)
                if (ev) cudaEventDestroy(ev);
            if (all[i].fork) cudaEventDestroy(all[i].fork);
            all.erase(all.begin() + i);
        } else {
            ++i;
        }
    }
}

}  // namespace bgabp

using namespace bgabp;

static inline unsigned nblk(long long n, int t = 256) { return nblk_host(n, t); }

extern "C" {

// ---- sharded flood solve (one row block per rank; the driver moves halos and reduces) ---------
int bgabp_shard_set_range(bgabp_engine* h, int own_lo, int own_hi, int gofs) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (E.layout != BGABP_LAYOUT_DIA) throw InvalidArg("shard: DIA layout required");
        if (own_lo < 0 || own_hi > E.n || own_lo > own_hi) throw InvalidArg("shard: bad owned range");
        E.dia.j0 = own_lo;
        E.dia.j1 = own_hi;
        E.dia.gofs = gofs;
        ++E.peer_gen;  // captured multi-shard iterations hold the old range
        p2p_forget(&E);
        if (!E.d_red4) E.d_red4 = static_cast<unsigned long long*>(E.dalloc(sizeof(unsigned long long) * 4));
        if (!E.d_pack) {
            E.pack_cap = 0;
        }
        return BGABP_OK;
    })
}

int bgabp_shard_solve_begin(bgabp_engine* h, const double* b_dev, const bgabp_options* opt, double r0) {
    ABI_GUARD(nullptr, 0, {
        bgabp_schedule fl{};
        fl.kind = BGABP_SCHED_FLOOD;
        h->E.solve_begin(b_dev, fl, *opt, &r0);
        return BGABP_OK;
    })
}

int bgabp_shard_step_compute(bgabp_engine* h) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (!E.solve_fused || !E.d_red4) throw InvalidArg("shard: call set_range and shard_solve_begin first");
        E.enqueue_fused_kernel();
        k_shard_fold<<<1, kSpread, 0, E.st>>>(E.d_ctrl, E.d_spread, E.d_red4);
        ck(cudaGetLastError(), "shard compute");
        return BGABP_OK;
    })
}

void* bgabp_shard_reduce_buffer(bgabp_engine* h) { return (void*)h->E.d_red4; }

int bgabp_shard_step_decide(bgabp_engine* h) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        k_shard_decide<<<1, 1, 0, E.st>>>(E.d_ctrl, E.d_hist, E.d_red4);
        ck(cudaGetLastError(), "shard decide");
        return BGABP_OK;
    })
}

// ---- sharded solve with peer-memory halos and reduction (no pack/unpack, no collective) ----------
int bgabp_shard_peer_slots(bgabp_engine* h, void** slots) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (!E.d_slots) {
            const size_t bytes = sizeof(unsigned long long) * (kSlotWords + kMaxShards);
            E.d_slots = static_cast<unsigned long long*>(E.dalloc(bytes));
            ck(cudaMemsetAsync(E.d_slots, 0, bytes, E.st), "memset");
        }
        if (!E.d_xf) E.d_xf = static_cast<double*>(E.dalloc(sizeof(double) * kXRing * (size_t)std::max(E.n, 1)));
        *slots = E.d_slots;
        return BGABP_OK;
    })
}

int bgabp_shard_set_peers(bgabp_engine* h, int nranks, int rank, void* const* lower, int lower_n, int lower_delta,
                          void* const* upper, int upper_n, int upper_delta, int xlo_end, int xhi_begin,
                          void* const* slots) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (nranks < 1 || nranks > kMaxShards || rank < 0 || rank >= nranks)
            throw InvalidArg("shard: 1 <= nranks <= 8 and 0 <= rank < nranks");
        if (E.dia.j0 == 0 && E.dia.j1 == E.n && nranks > 1 && !E.d_red4)
            throw InvalidArg("shard: call set_range first");
        ++E.peer_gen;  // captured multi-shard iterations hold the old peer pointers
        p2p_forget(&E);
        PeerP& Q = E.peer;
        std::memset(&Q, 0, sizeof Q);
        for (int b2 = 0; b2 < 2; ++b2) {  // lower/upper = {msg0, msg1, x0, x1} of the neighbour (or null)
            Q.m[0][b2] = lower ? static_cast<double2*>(lower[b2]) : nullptr;
            Q.x[0][b2] = lower ? static_cast<double*>(lower[2 + b2]) : nullptr;
            Q.m[1][b2] = upper ? static_cast<double2*>(upper[b2]) : nullptr;
            Q.x[1][b2] = upper ? static_cast<double*>(upper[2 + b2]) : nullptr;
        }
        Q.nq[0] = lower_n;
        Q.nq[1] = upper_n;
        Q.delta[0] = lower_delta;
        Q.delta[1] = upper_delta;
        Q.xlo_end = xlo_end;
        Q.xhi_begin = xhi_begin;
        for (int q = 0; q < nranks; ++q) Q.red[q] = static_cast<unsigned long long*>(slots[q]);
        Q.nranks = nranks;
        Q.rank = rank;
        E.peer_on = true;
        if (!E.d_red4) E.d_red4 = static_cast<unsigned long long*>(E.dalloc(sizeof(unsigned long long) * 4));
        if (!E.step_ev) ck(cudaEventCreateWithFlags(&E.step_ev, cudaEventDisableTiming), "event");
        return BGABP_OK;
    })
}

// the fused step with peer stores, the fold into every shard's slots, and this shard's event
int bgabp_shard_p2p_compute(bgabp_engine* h) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (!E.solve_fused || !E.peer_on) throw InvalidArg("shard: call set_peers and shard_solve_begin first");
        E.enqueue_fused_kernel();
        k_shard_fold_p2p<<<1, kSpread, 0, E.st>>>(E.d_ctrl, E.d_spread, E.d_red4, E.peer);
        ck(cudaEventRecord(E.step_ev, E.st), "event");
        ck(cudaGetLastError(), "shard p2p compute");
        return BGABP_OK;
    })
}

// order this shard's stream after another shard's last p2p_compute (its peer stores and words)
int bgabp_shard_p2p_wait(bgabp_engine* h, bgabp_engine* other) {
    ABI_GUARD(nullptr, 0, {
        ck(cudaStreamWaitEvent(h->E.st, other->E.step_ev, 0), "wait");
        return BGABP_OK;
    })
}

int bgabp_shard_p2p_decide(bgabp_engine* h, int spin) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        k_shard_decide_p2p<<<1, 1, 0, E.st>>>(E.d_ctrl, E.d_hist, E.d_slots, E.peer.nranks, E.d_red4, E.peer.rank,
                                              spin);
        ck(cudaGetLastError(), "shard p2p decide");
        return BGABP_OK;
    })
}

// nsteps iterations of the peer-memory solve for `count` shards of one process (event-ordered),
// replayed from a CUDA graph of 16 iterations captured across all shards' streams (the kernels
// read the iteration index from the device, so one graph serves every position in the loop)

static void p2p_enqueue_iteration(bgabp_engine* const* sh, int count) {
    for (int k = 0; k < count; ++k) {
        Engine& E = sh[k]->E;
        E.enqueue_fused_kernel();
        k_shard_fold_p2p<<<1, kSpread, 0, E.st>>>(E.d_ctrl, E.d_spread, E.d_red4, E.peer);
        ck(cudaEventRecord(E.step_ev, E.st), "event");
    }
    for (int k = 0; k < count; ++k) {
        Engine& E = sh[k]->E;
        for (int q = 0; q < count; ++q)
            if (q != k) ck(cudaStreamWaitEvent(E.st, sh[q]->E.step_ev, 0), "wait");
        k_shard_decide_p2p<<<1, 1, 0, E.st>>>(E.d_ctrl, E.d_hist, E.d_slots, E.peer.nranks, E.d_red4, E.peer.rank, 0);
    }
}

// one process per shard (CUDA IPC peers): nsteps iterations of (step + peer stores + fold, then the
// decision after a device-side wait on the peers' step flags), enqueued without host round trips
int bgabp_shard_p2p_steps_ipc(bgabp_engine* h, int nsteps) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (!E.solve_fused || !E.peer_on) throw InvalidArg("shard: call set_peers and shard_solve_begin first");
        for (int k = 0; k < nsteps; ++k) {
            E.enqueue_fused_kernel();
            k_shard_fold_p2p<<<1, kSpread, 0, E.st>>>(E.d_ctrl, E.d_spread, E.d_red4, E.peer);
            k_shard_decide_p2p<<<1, 1, 0, E.st>>>(E.d_ctrl, E.d_hist, E.d_slots, E.peer.nranks, E.d_red4, E.peer.rank, 1);
        }
        ck(cudaGetLastError(), "p2p ipc steps");
        return BGABP_OK;
    })
}

int bgabp_shard_p2p_steps(bgabp_engine* const* shards, int count, int nsteps, int use_graph) {
    ABI_GUARD(nullptr, 0, {
        if (count < 1) throw InvalidArg("shard: no shards");
        for (int k = 0; k < count; ++k)
            if (!shards[k]->E.solve_fused || !shards[k]->E.peer_on)
                throw InvalidArg("shard: call set_peers and shard_solve_begin first");
        constexpr int kChunk = 16;
        P2PGraph* g = nullptr;
        if (use_graph && nsteps >= kChunk) {
            auto& all = p2p_graphs();
            for (auto& c : all) {
                if (c.engines.size() != (size_t)count) continue;
                bool same = true;
                for (int k = 0; k < count && same; ++k)
                    same = c.engines[k] == &shards[k]->E && c.gens[k] == p2p_key(shards[k]->E);
                if (same) g = &c;
            }
            if (!g) {
                P2PGraph c;
                for (int k = 0; k < count; ++k) {
                    c.engines.push_back(&shards[k]->E);
                    c.gens.push_back(p2p_key(shards[k]->E));
                }
                ck(cudaEventCreateWithFlags(&c.fork, cudaEventDisableTiming), "event");
                c.join.resize(count);
                for (auto& e : c.join) ck(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "event");
                cudaStream_t s0 = shards[0]->E.st;
                cudaGraph_t graph;
                ck(cudaStreamBeginCapture(s0, cudaStreamCaptureModeThreadLocal), "capture");
                ck(cudaEventRecord(c.fork, s0), "fork");
                for (int k = 1; k < count; ++k) ck(cudaStreamWaitEvent(shards[k]->E.st, c.fork, 0), "fork wait");
                for (int i = 0; i < kChunk; ++i) p2p_enqueue_iteration(shards, count);
                for (int k = 1; k < count; ++k) {
                    ck(cudaEventRecord(c.join[k], shards[k]->E.st), "join");
                    ck(cudaStreamWaitEvent(s0, c.join[k], 0), "join wait");
                }
                ck(cudaStreamEndCapture(s0, &graph), "capture end");
                ck(cudaGraphInstantiate(&c.exec, graph, 0), "graph instantiate");
                cudaGraphDestroy(graph);
                all.push_back(std::move(c));
                g = &all.back();
            }
        }
        int left = nsteps;
        while (g && left >= kChunk) {
            // order the graph after everything already on the other shards' streams, and them after it
            cudaStream_t s0 = shards[0]->E.st;
            for (int k = 1; k < count; ++k) {
                ck(cudaEventRecord(g->join[k], shards[k]->E.st), "pre");
                ck(cudaStreamWaitEvent(s0, g->join[k], 0), "pre wait");
            }
            ck(cudaGraphLaunch(g->exec, s0), "graph launch");
            ck(cudaEventRecord(g->fork, s0), "post");
            for (int k = 1; k < count; ++k) ck(cudaStreamWaitEvent(shards[k]->E.st, g->fork, 0), "post wait");
            left -= kChunk;
        }
        for (; left > 0; --left) p2p_enqueue_iteration(shards, count);
        ck(cudaGetLastError(), "p2p steps");
        return BGABP_OK;
    })
}

// CUDA IPC for shards in different processes (one process per GPU): export / open the device
// allocations a neighbour stores into (message buffers, x ring base, slot array)
int bgabp_ipc_get(const void* dev_ptr, void* handle_out) {
    ABI_GUARD(nullptr, 0, {
        cudaIpcMemHandle_t hd;
        ck(cudaIpcGetMemHandle(&hd, const_cast<void*>(dev_ptr)), "cudaIpcGetMemHandle");
        std::memcpy(handle_out, &hd, sizeof hd);
        return BGABP_OK;
    })
}
int bgabp_ipc_open(const void* handle, void** dev_ptr) {
    ABI_GUARD(nullptr, 0, {
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, handle, sizeof hd);
        ck(cudaIpcOpenMemHandle(dev_ptr, hd, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
        return BGABP_OK;
    })
}
int bgabp_ipc_close(void* dev_ptr) {
    ABI_GUARD(nullptr, 0, {
        ck(cudaIpcCloseMemHandle(dev_ptr), "cudaIpcCloseMemHandle");
        return BGABP_OK;
    })
}

int bgabp_dia_offsets(const bgabp_engine* h, int* off, int cap) {
    const Engine& E = h->E;
    if (E.layout != BGABP_LAYOUT_DIA) return -1;
    for (int s = 0; s < E.S && s < cap; ++s) off[s] = E.dia.off[s];
    return E.S;
}

void bgabp_trim_cache(void) { trim_block_cache(); }

void* bgabp_shard_msg(bgabp_engine* h, int which) { return (void*)h->E.d_msg[which & 1]; }
void* bgabp_shard_x(bgabp_engine* h, int which) {  // the slot holding x(which)
    Engine& E = h->E;
    if (!E.d_xf) E.d_xf = static_cast<double*>(E.dalloc(sizeof(double) * kXRing * (size_t)std::max(E.n, 1)));
    return (void*)xslot(E.d_xf, E.n, which);
}

int bgabp_shard_pack(bgabp_engine* h, int which, int lo, int len, void* out_dev) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (len > 0)
            k_shard_pack<<<nblk(len), 256, 0, E.st>>>(E.dia, E.d_msg[which & 1], static_cast<double2*>(out_dev), lo, len);
        ck(cudaGetLastError(), "shard pack");
        return BGABP_OK;
    })
}

int bgabp_shard_unpack(bgabp_engine* h, int which, const void* recv_dev, int lo, int len, int sender_lo,
                       int sender_hi) {
    ABI_GUARD(nullptr, 0, {
        Engine& E = h->E;
        if (len > 0)
            k_shard_unpack<<<nblk(len), 256, 0, E.st>>>(E.dia, E.d_msg[which & 1], static_cast<const double2*>(recv_dev),
                                                        lo, len, sender_lo, sender_hi);
        ck(cudaGetLastError(), "shard unpack");
        return BGABP_OK;
    })
}

int bgabp_shard_state(bgabp_engine* h, int* done, int* step) {
    ABI_GUARD(nullptr, 0, {
        h->E.read_ctrl();
        *done = h->E.h_ctrl->done;
        *step = h->E.h_ctrl->step;
        return BGABP_OK;
    })
}

}  // extern "C"
