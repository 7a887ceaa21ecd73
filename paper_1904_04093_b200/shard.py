"""Sharded synchronous GaBP solve: one contiguous row block per shard.

Each shard holds its owned rows plus ghost rows (halo width H = the largest neighbour offset)
and runs the fused flood step of the single-GPU solve (K1+K4) on its owned nodes only.  Per
iteration t:

    compute   sweep t + residual of x(t-2) on owned nodes, folded into 4 int64 words
    reduce    MAX all-reduce of those words (residual, message delta, encoded edge / node pivot)
    decide    the reference's stop logic (gabp.cpp:187-218) on the combined words, on every shard
    exchange  halo in-slot messages of sweep t and halo x(t-1) with the neighbouring shards

so every shard takes the same decision at the same iteration and the solve is bit-identical to
the single-engine one.  The transport is torch.distributed (NCCL between GPUs; gloo in the CPU
tests); shards of one process exchange by copies.  The compute side is the CUDA engine
(`GpuShard`); tests/shard_emu.py is a numpy stand-in with the same interface so this driver is
tested with world_size 2 over gloo on the CPU.
"""
from __future__ import annotations

import contextlib
import ctypes as C
from dataclasses import dataclass

import numpy as np

from .gabp import GabpEngine, GabpOptions, Layout, SparseMatrix, _raise, lib


@dataclass
class ShardLayout:
    """Global rows [lo, hi) owned by shard `index`; local arrays cover [glo, ghi) (ghosts around)."""
    index: int
    count: int
    n: int
    lo: int
    hi: int
    glo: int
    ghi: int

    @property
    def n_local(self):
        return self.ghi - self.glo

    @property
    def own_lo(self):
        return self.lo - self.glo

    @property
    def own_hi(self):
        return self.hi - self.glo

    @staticmethod
    def partition(n, halo, count, align=1):
        """`count` contiguous blocks of whole `align`-node units (e.g. grid rows), each >= halo."""
        units = n // align
        if units * align != n:
            raise ValueError("n is not a multiple of align")
        bounds = [(units * k) // count * align for k in range(count + 1)]
        out = []
        for k in range(count):
            lo, hi = bounds[k], bounds[k + 1]
            if hi - lo < halo:
                raise ValueError(f"shard {k} owns {hi - lo} nodes, fewer than the halo {halo}")
            out.append(ShardLayout(k, count, n, lo, hi, max(0, lo - halo), min(n, hi + halo)))
        return out


def dia_halo(A: SparseMatrix):
    """Largest |column - row| of A: the halo a row block needs."""
    rows = np.repeat(np.arange(A.n), np.diff(A.row_offsets))
    return int(np.max(np.abs(A.col_indices.astype(np.int64) - rows))) if A.nnz else 0


def local_matrix(A: SparseMatrix, L: ShardLayout) -> SparseMatrix:
    """Owned rows in full; ghost rows keep their diagonal and their couplings to owned nodes, which
    are the coefficients of the owned nodes' outgoing messages (gabp.cpp:120-139)."""
    ro = A.row_offsets
    s, e = int(ro[L.glo]), int(ro[L.ghi])
    rows = np.repeat(np.arange(L.glo, L.ghi), np.diff(ro[L.glo:L.ghi + 1]))
    cols = A.col_indices[s:e]
    vals = A.values[s:e]
    keep = ((rows >= L.lo) & (rows < L.hi)) | ((cols >= L.lo) & (cols < L.hi)) | (rows == cols)
    rows, cols, vals = rows[keep], cols[keep], vals[keep]
    counts = np.bincount(rows - L.glo, minlength=L.n_local)
    lro = np.zeros(L.n_local + 1, np.int32)
    np.cumsum(counts, out=lro[1:])
    return SparseMatrix(L.n_local, lro, (cols - L.glo).astype(np.int32), np.ascontiguousarray(vals, np.float64))


def _device_view(ptr, count, dtype, device):
    """A torch tensor over `count` elements of engine-owned device memory (no copy)."""
    import torch
    typestr = {torch.int64: "<i8", torch.float64: "<f8"}[dtype]

    class _Cai:
        __cuda_array_interface__ = {"shape": (count,), "typestr": typestr, "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_Cai(), device=device)


class GpuShard:
    """One row block on the GPU: the engine's fused step restricted to the owned nodes."""

    def __init__(self, A_local: SparseMatrix, L: ShardLayout, b_local, device="cuda"):
        import torch
        self.torch, self.L = torch, L
        self.eng = GabpEngine(A_local, Layout.Dia)
        _raise(lib().bgabp_shard_set_range(self.eng.handle, L.own_lo, L.own_hi, L.glo), "shard_set_range")
        self.S = int(self.eng.info["num_slots"])
        off = (C.c_int * 8)()
        cnt = lib().bgabp_dia_offsets(self.eng.handle, off, 8)
        self.offsets = tuple(off[:cnt])
        self.device = torch.device(device)
        self.stream = torch.cuda.ExternalStream(self.eng.stream(), device=self.device)
        self.b = torch.as_tensor(np.ascontiguousarray(b_local, np.float64), device=self.device)
        self.red4 = _device_view(lib().bgabp_shard_reduce_buffer(self.eng.handle), 4, torch.int64, self.device)
        # x(k) lives in slot k % 2 (kXRing in kernels.cuh); views of both slots
        self.x = [_device_view(lib().bgabp_shard_x(self.eng.handle, k), L.n_local, torch.float64, self.device)
                  for k in range(2)]

    def begin(self, opt: GabpOptions, r0: float):
        o = opt._c()
        _raise(lib().bgabp_shard_solve_begin(self.eng.handle, C.c_void_p(self.b.data_ptr()), C.byref(o),
                                             C.c_double(r0)), "shard_solve_begin")

    def compute(self):
        _raise(lib().bgabp_shard_step_compute(self.eng.handle), "shard_step_compute")

    def decide(self):
        _raise(lib().bgabp_shard_step_decide(self.eng.handle), "shard_step_decide")

    def pack(self, which, lo, length):
        out = self.torch.empty(self.S * length * 2, dtype=self.torch.float64, device=self.device)
        _raise(lib().bgabp_shard_pack(self.eng.handle, which, lo, length, C.c_void_p(out.data_ptr())), "pack")
        return out

    def unpack(self, which, buf, lo, length, sender_lo, sender_hi):
        _raise(lib().bgabp_shard_unpack(self.eng.handle, which, C.c_void_p(buf.data_ptr()), lo, length,
                                        sender_lo, sender_hi), "unpack")

    def new_buffer(self, count):
        return self.torch.empty(count, dtype=self.torch.float64, device=self.device)

    def done(self):
        d, _ = C.c_int(0), C.c_int(0)
        _raise(lib().bgabp_shard_state(self.eng.handle, C.byref(d), C.byref(_)), "shard_state")
        return bool(d.value)

    def end(self, max_iter):
        n = self.L.n_local
        x = self.torch.empty(n, dtype=self.torch.float64, device=self.device)
        hist = self.torch.empty(max_iter + 2, dtype=self.torch.float64, device=self.device)
        status, its, flops, detail = self.eng.solve_device_end(x.data_ptr(), hist.data_ptr())
        nh = its + (0 if int(status) == 1 and detail.startswith("zero pivot") else 1)  # gabp.cpp:193-199
        return (int(status), its, detail, x[self.L.own_lo:self.L.own_hi].cpu().numpy(),
                hist[:nh].cpu().numpy())


class Exchange:
    """MAX all-reduce and neighbour halo exchange between shards: copies within a process,
    torch.distributed point-to-point between processes."""

    def __init__(self, shards: dict, layouts, owner, world):
        self.shards, self.layouts, self.owner, self.world = shards, layouts, owner, world

    def allreduce_max(self):
        import torch
        mine = list(self.shards.values())
        acc = mine[0].red4.clone()
        for s in mine[1:]:
            acc = torch.maximum(acc, s.red4)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(acc, op=dist.ReduceOp.MAX)
        for s in mine:
            s.red4.copy_(acc)

    def halo(self, which_msg, which_x):
        """Messages of sweep t (buffer which_msg) and x(t-1) (x slot which_x)."""
        ops, pending = [], []
        P = len(self.layouts)
        for p in range(P):
            for q in (p - 1, p + 1):
                if q < 0 or q >= P:
                    continue
                sp, sq = self.shards.get(p), self.shards.get(q)
                if sp is None and sq is None:
                    continue
                Lp, Lq = self.layouts[p], self.layouts[q]
                items = []
                a, b = max(Lp.glo, Lq.lo), min(Lp.ghi, Lq.hi)  # q's nodes in p's halo: p computed their messages
                if b > a:
                    items.append(("msg", a, b))
                a, b = max(Lq.glo, Lp.lo), min(Lq.ghi, Lp.hi)  # p's nodes in q's halo: q needs their x
                if b > a:
                    items.append(("x", a, b))
                for kind, a, b in items:
                    tag = 4 * p + 2 * (q > p) + (kind == "x")
                    data = None
                    if sp is not None:
                        data = (sp.pack(which_msg, a - Lp.glo, b - a) if kind == "msg"
                                else sp.x[which_x][a - Lp.glo:b - Lp.glo].clone())
                    if sp is not None and sq is not None:
                        self._deliver(sq, kind, data, a, b, Lp, Lq, which_msg, which_x)
                    elif sp is not None:
                        import torch.distributed as dist
                        ops.append(dist.P2POp(dist.isend, data, self.owner[q], tag=tag))
                    else:
                        import torch.distributed as dist
                        buf = sq.new_buffer(sq.S * (b - a) * 2 if kind == "msg" else b - a)
                        ops.append(dist.P2POp(dist.irecv, buf, self.owner[p], tag=tag))
                        pending.append((sq, kind, buf, a, b, Lp, Lq))
        if ops:
            import torch.distributed as dist
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        for sq, kind, buf, a, b, Lp, Lq in pending:
            self._deliver(sq, kind, buf, a, b, Lp, Lq, which_msg, which_x)

    @staticmethod
    def _deliver(sq, kind, data, a, b, Lp, Lq, which_msg, which_x):
        if kind == "msg":  # only the in-slots whose sender p owns
            sq.unpack(which_msg, data, a - Lq.glo, b - a, Lp.lo - Lq.glo, Lp.hi - Lq.glo)
        else:
            sq.x[which_x][a - Lq.glo:b - Lq.glo].copy_(data)


def sharded_solve(shards: dict, layouts, owner, world, b_inf, opt: GabpOptions, poll_every=16):
    """Flood solve over all shards to the reference's stop rule.  `shards` maps global shard
    index -> shard object for this process; `owner` maps every shard index to its rank.
    Returns (status, iterations, detail, {shard: owned x}, residual history)."""
    import torch
    ex = Exchange(shards, layouts, owner, world)
    first = next(iter(shards.values()))
    gpu = isinstance(first, GpuShard)
    if gpu:  # every shard of every rank must hold the same DIA offsets
        mine = [s.offsets for s in shards.values()]
        if world > 1:
            import torch.distributed as dist
            every = [None] * world
            dist.all_gather_object(every, mine)
            mine = [o for r in every for o in r]
        check_offsets(mine)
    single = len(shards) == 1
    ctx = torch.cuda.stream(first.stream) if (gpu and single) else contextlib.nullcontext()
    sync = torch.cuda.synchronize if (gpu and not single) else (lambda: None)
    with ctx:
        for s in shards.values():
            s.begin(opt, b_inf)
        sync()
        t, cap = 1, opt.max_iter + 2
        done = first.done()
        while not done and t <= cap:
            for s in shards.values():
                s.compute()
            sync()
            ex.allreduce_max()
            sync()
            for s in shards.values():
                s.decide()
            sync()
            ex.halo(t & 1, (t - 1) & 1)
            sync()
            t += 1
            if t % poll_every == 0 or t > cap:
                done = first.done()
        out, res = {}, None
        for k, s in shards.items():
            status, its, detail, x, hist = s.end(opt.max_iter)
            out[k] = x
            res = (status, its, detail, hist)
    return res[0], res[1], res[2], out, res[3]


def check_offsets(offsets):
    """Halos move slot by slot (peer stores / pack / unpack use the neighbour's slot order), so
    every shard must hold the same DIA offsets; a row block that lacks one would land messages in
    the wrong slots."""
    offsets = list(offsets)
    if any(o != offsets[0] for o in offsets):
        raise ValueError(f"shard: the row blocks have different DIA neighbour offsets {sorted(set(offsets))}; "
                         "partition so that every block holds every stencil offset")


def connect_peers(shards: dict, layouts):
    """Wire every GpuShard of this process to its neighbours for the peer-memory step: each
    shard stores the halo messages / x it computes straight into the neighbour's buffers and its
    reduction words into every shard's slot array (bgabp_shard_set_peers).  Shards may live on
    different GPUs of one process (peer access enabled) or share one GPU."""
    L = lib()
    P = len(layouts)
    if sorted(shards) != list(range(P)):
        raise ValueError("connect_peers: every shard must live in this process")
    check_offsets(shards[k].offsets for k in range(P))
    slots = []
    for k in range(P):
        p = C.c_void_p()
        _raise(L.bgabp_shard_peer_slots(shards[k].eng.handle, C.byref(p)), "peer slots")
        slots.append(p.value)
    slot_arr = (C.c_void_p * P)(*slots)

    def bufs(k):
        h = shards[k].eng.handle
        return (C.c_void_p * 4)(L.bgabp_shard_msg(h, 0), L.bgabp_shard_msg(h, 1), L.bgabp_shard_x(h, 0),
                                L.bgabp_shard_x(h, 1))

    for k in range(P):
        Lk = layouts[k]
        lower = bufs(k - 1) if k > 0 else None
        upper = bufs(k + 1) if k + 1 < P else None
        lo_n = layouts[k - 1].n_local if k > 0 else 0
        up_n = layouts[k + 1].n_local if k + 1 < P else 0
        lo_d = Lk.glo - layouts[k - 1].glo if k > 0 else 0
        up_d = Lk.glo - layouts[k + 1].glo if k + 1 < P else 0
        xlo_end = layouts[k - 1].ghi - Lk.glo if k > 0 else 0          # own nodes in the lower one's halo
        xhi_begin = layouts[k + 1].glo - Lk.glo if k + 1 < P else Lk.n_local  # ... in the upper one's
        _raise(L.bgabp_shard_set_peers(shards[k].eng.handle, P, k, lower, lo_n, lo_d, upper, up_n, up_d,
                                       xlo_end, xhi_begin, slot_arr), "set peers")


def sharded_solve_p2p(shards: dict, layouts, b_inf, opt: GabpOptions, poll_every=16, spin=False, graph=False):
    """The sharded flood solve with the halo exchange and the stop-word reduction done by the
    step kernels themselves through peer memory (no pack / unpack kernels, no collective, no host
    synchronisation inside the loop): per iteration every shard enqueues its fused step (+ peer
    stores) and fold, then waits on every other shard's step event and decides.  Bit-identical to
    the single-engine solve.  Returns (status, iterations, detail, {shard: owned x}, history)."""
    connect_peers(shards, layouts)
    L = lib()
    order = sorted(shards)
    for k in order:
        shards[k].begin(opt, b_inf)
    shards[order[0]].torch.cuda.synchronize()  # every shard reset before any peer stores into it
    t, cap = 1, opt.max_iter + 2
    done = shards[order[0]].done()
    if graph:  # whole chunks of iterations from a CUDA graph across the shards' streams
        arr = (C.c_void_p * len(order))(*[shards[k].eng.handle.value for k in order])
        chunk = 4 * 16
        while not done and t <= cap:
            _raise(L.bgabp_shard_p2p_steps(arr, len(order), chunk, 1), "p2p steps")
            t += chunk
            done = shards[order[0]].done()
    while not done and t <= cap:
        for k in order:
            _raise(L.bgabp_shard_p2p_compute(shards[k].eng.handle), "p2p compute")
        if spin:  # the device-flag wait of the multi-process path, exercised with every flag already set
            shards[order[0]].torch.cuda.synchronize()
        for k in order:
            for q in order:
                if q != k and not spin:
                    _raise(L.bgabp_shard_p2p_wait(shards[k].eng.handle, shards[q].eng.handle), "p2p wait")
            _raise(L.bgabp_shard_p2p_decide(shards[k].eng.handle, 1 if spin else 0), "p2p decide")
        t += 1
        if t % poll_every == 0 or t > cap:
            done = shards[order[0]].done()
    out, res = {}, None
    for k in order:
        status, its, detail, x, hist = shards[k].end(opt.max_iter)
        out[k] = x
        res = (status, its, detail, hist)
    return res[0], res[1], res[2], out, res[3]


class IpcSolve:
    """The one-shard-per-process peer-memory solve as a stepping object (bench.py's multi-GPU
    mode): connect() maps the neighbours' buffers and every rank's slot array with CUDA IPC,
    begin() resets this rank, steps(k) enqueues k iterations (fused step with peer stores, fold,
    device-side wait on the peers' step flags, decision) with no host synchronisation, end()
    returns (status, iterations, detail, owned x, history)."""

    def __init__(self, shard, layouts, host_barrier=False):
        import torch.distributed as dist
        self.dist, self.shard, self.layouts, self.host_barrier = dist, shard, layouts, host_barrier
        self.L = lib()
        self.rank, self.P = dist.get_rank(), dist.get_world_size()
        if len(layouts) != self.P:
            raise ValueError("sharded_solve_ipc: one shard per rank")
        self.opened = []

    def connect(self):
        L, h, rank, P, layouts, dist = self.L, self.shard.eng.handle, self.rank, self.P, self.layouts, self.dist
        slots = C.c_void_p()
        _raise(L.bgabp_shard_peer_slots(h, C.byref(slots)), "peer slots")

        def export(ptr):
            buf = C.create_string_buffer(64)
            _raise(L.bgabp_ipc_get(C.c_void_p(ptr), buf), "ipc get")
            return buf.raw

        mine = {"msg0": export(L.bgabp_shard_msg(h, 0)), "msg1": export(L.bgabp_shard_msg(h, 1)),
                "x": export(L.bgabp_shard_x(h, 0)), "slots": export(slots.value), "offsets": self.shard.offsets}
        peers = [None] * P
        dist.all_gather_object(peers, mine)
        check_offsets(p["offsets"] for p in peers)

        def imp(handle):
            p = C.c_void_p()
            _raise(L.bgabp_ipc_open(handle, C.byref(p)), "ipc open")
            self.opened.append(p.value)
            return p.value

        slot_ptrs = [slots.value if q == rank else imp(peers[q]["slots"]) for q in range(P)]

        def nbr(q):
            xb = imp(peers[q]["x"])
            return (C.c_void_p * 4)(imp(peers[q]["msg0"]), imp(peers[q]["msg1"]), xb, xb + 8 * layouts[q].n_local)

        Lk = layouts[rank]
        lower = nbr(rank - 1) if rank > 0 else None
        upper = nbr(rank + 1) if rank + 1 < P else None
        _raise(L.bgabp_shard_set_peers(h, P, rank, lower, layouts[rank - 1].n_local if rank > 0 else 0,
                                       Lk.glo - layouts[rank - 1].glo if rank > 0 else 0, upper,
                                       layouts[rank + 1].n_local if rank + 1 < P else 0,
                                       Lk.glo - layouts[rank + 1].glo if rank + 1 < P else 0,
                                       layouts[rank - 1].ghi - Lk.glo if rank > 0 else 0,
                                       layouts[rank + 1].glo - Lk.glo if rank + 1 < P else Lk.n_local,
                                       (C.c_void_p * P)(*slot_ptrs)), "set peers")

    def begin(self, opt: GabpOptions, r0: float):
        import torch
        self.opt = opt
        self.shard.begin(opt, r0)  # zeroes this rank's buffers and slots
        torch.cuda.synchronize()
        self.dist.barrier()  # nobody stores into a peer before every peer has been reset

    def steps(self, k):
        import torch
        if not self.host_barrier:
            _raise(self.L.bgabp_shard_p2p_steps_ipc(self.shard.eng.handle, int(k)), "p2p ipc steps")
            return
        h = self.shard.eng.handle
        for _ in range(k):
            _raise(self.L.bgabp_shard_p2p_compute(h), "p2p compute")
            torch.cuda.synchronize()
            self.dist.barrier()
            _raise(self.L.bgabp_shard_p2p_decide(h, 1), "p2p decide")

    def done(self):
        return self.shard.done()

    def end(self):
        return self.shard.end(self.opt.max_iter)

    def close(self):
        import torch
        torch.cuda.synchronize()
        self.dist.barrier()  # every peer is done storing before the mappings go
        for p in self.opened:
            self.L.bgabp_ipc_close(C.c_void_p(p))
        self.opened = []


def sharded_solve_ipc(shard, layouts, b_inf, opt: GabpOptions, poll_every=16, host_barrier=False):
    """One shard per process (one process per GPU, torch.distributed initialised): the neighbours'
    message buffers / x ring and every rank's slot array are mapped with CUDA IPC once, then each
    iteration is the peer-memory step (halos and stop words stored by the kernels into the
    peers' memory) followed by a device-side wait on the peers' step flags -- no host
    synchronisation and no collective inside the loop.  host_barrier=True puts a host barrier
    between the steps and the decisions (every peer flag is already set when a decision runs):
    the mode for ranks sharing one GPU, where device-side waits between processes must not be
    used.  Returns (status, iterations, detail, owned x, history)."""
    s = IpcSolve(shard, layouts, host_barrier)
    s.connect()
    try:
        s.begin(opt, b_inf)
        t, cap = 1, opt.max_iter + 2
        done = s.done()
        while not done and t <= cap:
            s.steps(1)
            t += 1
            if t % poll_every == 0 or t > cap or host_barrier:
                done = s.done()
        out = s.end()
    finally:
        s.close()
    return out
