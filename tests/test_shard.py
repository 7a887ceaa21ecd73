"""Sharded flood solve: row blocks + halo exchange + MAX all-reduce of the stop
words must reproduce the single-process solve bit for bit.

CPU: the driver (paper_1904_04093_b200.shard) over numpy shards (tests/shard_emu.py), in one
process and with world_size 2 over gloo, against the oracle's GabpEngine::solve.
GPU: the driver over CUDA shards (one process, peer memory, CUDA IPC) against the CPU oracle directly
and against the single-engine CUDA solve.
"""
import os
import socket

import numpy as np
import pytest

from paper_1904_04093_b200.gabp import GabpOptions, SparseMatrix
from paper_1904_04093_b200.shard import ShardLayout, dia_halo, local_matrix, sharded_solve

from oracle.oracle import Schedule
from tests.shard_emu import CpuShard


def _csr(n, rows, cols, vals):
    rows, cols, vals = map(np.asarray, (rows, cols, vals))
    o = np.lexsort((cols, rows))
    rows, cols, vals = rows[o], cols[o], vals[o].astype(np.float64)
    ro = np.zeros(n + 1, np.int32)
    np.cumsum(np.bincount(rows, minlength=n), out=ro[1:])
    return SparseMatrix(n, ro, cols.astype(np.int32), vals)


def grid5(nx, ny, beta=0.0):
    """5-point operator, x fastest; beta skews the x couplings (nonsymmetric upwind-like)."""
    r, c, v = [], [], []
    for j in range(ny):
        for i in range(nx):
            k = j * nx + i
            r.append(k), c.append(k), v.append(4.0)
            for di, dj, w in ((-1, 0, -1.0 - beta), (1, 0, -1.0 + beta), (0, -1, -1.0), (0, 1, -1.0)):
                ii, jj = i + di, j + dj
                if 0 <= ii < nx and 0 <= jj < ny:
                    r.append(k), c.append(jj * nx + ii), v.append(w)
    return _csr(nx * ny, r, c, v)


def grid7(nx, ny, nz):
    r, c, v = [], [], []
    for kz in range(nz):
        for j in range(ny):
            for i in range(nx):
                k = (kz * ny + j) * nx + i
                r.append(k), c.append(k), v.append(6.5)
                for d in ((-1, 0, 0), (1, 0, 0), (0, -1, 0), (0, 1, 0), (0, 0, -1), (0, 0, 1)):
                    ii, jj, kk = i + d[0], j + d[1], kz + d[2]
                    if 0 <= ii < nx and 0 <= jj < ny and 0 <= kk < nz:
                        r.append(k), c.append((kk * ny + jj) * nx + ii), v.append(-1.0)
    return _csr(nx * ny * nz, r, c, v)


PROBLEMS = {
    # name: (matrix builder, align (whole grid rows / planes), shards, options)
    "grid5_sym": (lambda: grid5(24, 18), 24, 3, GabpOptions(tol=1e-9, max_iter=4000)),
    "grid5_nonsym": (lambda: grid5(20, 16, beta=0.4), 20, 2, GabpOptions(tol=1e-9, max_iter=4000)),
    "grid5_delta": (lambda: grid5(16, 12), 16, 3, GabpOptions(tol=1e-7, max_iter=4000, stop=1)),
    "grid5_maxiter": (lambda: grid5(24, 24), 24, 4, GabpOptions(tol=1e-14, max_iter=37)),
    "grid7": (lambda: grid7(8, 6, 9), 48, 3, GabpOptions(tol=1e-9, max_iter=4000)),
    "pivot2": (lambda: _csr(2, [0, 0, 1, 1], [0, 1, 0, 1], [1.0, 1.0, 1.0, 1.0]), 1, 2, GabpOptions()),
}


def _rhs(n, seed=5):
    return np.random.RandomState(seed).uniform(-1.0, 1.0, n)


def _r0(b):
    a = np.abs(b)
    a = a[~np.isnan(a)]
    return float(a.max()) if a.size else 0.0


def _shards(A, b, layouts, mine, cls):
    return {k: cls(local_matrix(A, layouts[k]), layouts[k], b[layouts[k].glo:layouts[k].ghi]) for k in mine}


def _gather(layouts, xs):
    x = np.zeros(layouts[0].n)
    for k, xk in xs.items():
        x[layouts[k].lo:layouts[k].hi] = xk
    return x


def _oracle_solve(orc, A, b, opt):
    from oracle.oracle import Csr
    Ac = orc.canonical(Csr(A.n, A.row_offsets, A.col_indices, A.values))
    return orc.engine(Ac).solve(b, Schedule.parallel_flood(), tol=opt.tol, max_iter=opt.max_iter, stop=int(opt.stop),
                                divergence_factor=opt.divergence_factor)


def _assert_same(rep, status, its, detail, x, hist):
    assert (status, its) == (rep.status, rep.iterations), (status, its, rep.status, rep.iterations, detail, rep.detail)
    assert detail == rep.detail
    np.testing.assert_array_equal(x.view(np.uint64), rep.solution.view(np.uint64))
    np.testing.assert_array_equal(hist.view(np.uint64), rep.residual_history.view(np.uint64))


def test_partition_covers_rows_with_halo():
    A = grid5(10, 9)
    H = dia_halo(A)
    assert H == 10
    Ls = ShardLayout.partition(A.n, H, 3, align=10)
    assert Ls[0].lo == 0 and Ls[-1].hi == A.n
    assert all(a.hi == b.lo for a, b in zip(Ls, Ls[1:]))
    assert all(L.lo % 10 == 0 and L.hi - L.lo >= H for L in Ls)
    assert Ls[1].glo == Ls[1].lo - H and Ls[1].ghi == Ls[1].hi + H
    with pytest.raises(ValueError):
        ShardLayout.partition(A.n, H, 10, align=10)


def test_local_matrix_keeps_owned_rows_and_columns():
    A = grid5(8, 8, beta=0.3)
    L = ShardLayout.partition(A.n, dia_halo(A), 2, align=8)[1]
    Al = local_matrix(A, L)
    D, Dl = np.zeros((A.n, A.n)), np.zeros((Al.n, Al.n))
    for M, Dm in ((A, D), (Al, Dl)):
        rows = np.repeat(np.arange(M.n), np.diff(M.row_offsets))
        Dm[rows, M.col_indices] = M.values
    sub = D[L.glo:L.ghi, L.glo:L.ghi]
    own = slice(L.own_lo, L.own_hi)
    np.testing.assert_array_equal(Dl[own, :], sub[own, :])
    np.testing.assert_array_equal(Dl[:, own], sub[:, own])
    np.testing.assert_array_equal(np.diag(Dl), np.diag(sub))


@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_emulated_shards_match_oracle(orc, name):
    build, align, count, opt = PROBLEMS[name]
    A = build()
    b = _rhs(A.n)
    layouts = ShardLayout.partition(A.n, dia_halo(A), count, align=align)
    shards = _shards(A, b, layouts, range(count), CpuShard)
    status, its, detail, xs, hist = sharded_solve(shards, layouts, [0] * count, 1, _r0(b), opt)
    rep = _oracle_solve(orc, A, b, opt)
    _assert_same(rep, status, its, detail, _gather(layouts, xs), hist)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, name, owner, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        build, align, count, opt = PROBLEMS[name]
        A = build()
        b = _rhs(A.n)
        layouts = ShardLayout.partition(A.n, dia_halo(A), len(owner), align=align)
        mine = [k for k, r in enumerate(owner) if r == rank]
        shards = _shards(A, b, layouts, mine, CpuShard)
        status, its, detail, xs, hist = sharded_solve(shards, layouts, owner, world, _r0(b), opt)
        q.put((rank, status, its, detail, xs, hist))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,owner", [("grid5_sym", [0, 0, 1, 1]), ("grid5_nonsym", [0, 1, 0, 1]),
                                        ("grid7", [0, 1]), ("pivot2", [0, 1])])
def test_gloo_world2_matches_oracle(orc, name, owner):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, name, owner, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    build, align, count, opt = PROBLEMS[name]
    A = build()
    b = _rhs(A.n)
    layouts = ShardLayout.partition(A.n, dia_halo(A), len(owner), align=align)
    xs = {}
    for rank, status, its, detail, x, hist in outs:
        xs.update(x)
    assert outs[0][1:4] == outs[1][1:4]  # every rank took the same decision
    rep = _oracle_solve(orc, A, b, opt)
    _assert_same(rep, outs[0][1], outs[0][2], outs[0][3], _gather(layouts, xs), outs[0][5])


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PROBLEMS))
def test_gpu_shards_match_single_engine(orc, name):
    from paper_1904_04093_b200.gabp import GabpEngine, Layout
    from paper_1904_04093_b200.gabp import Schedule as GSchedule
    from paper_1904_04093_b200.shard import GpuShard
    build, align, count, opt = PROBLEMS[name]
    A = build()
    b = _rhs(A.n)
    layouts = ShardLayout.partition(A.n, dia_halo(A), count, align=align)
    shards = _shards(A, b, layouts, range(count), GpuShard)
    status, its, detail, xs, hist = sharded_solve(shards, layouts, [0] * count, 1, _r0(b), opt)
    rep = GabpEngine(A, Layout.Dia).solve(b, GSchedule.parallel_flood(), opt)
    _assert_same(rep, status, its, detail, _gather(layouts, xs), hist)
    _assert_same(_oracle_solve(orc, A, b, opt), status, its, detail, _gather(layouts, xs), hist)


@pytest.mark.gpu
@pytest.mark.parametrize("name", sorted(PROBLEMS))
@pytest.mark.parametrize("mode", ["event", "spin", "graph"])
def test_gpu_peer_shards_match_single_engine(orc, name, mode):
    """The peer-memory step (halo messages and x stored by the step kernel into the neighbour's
    buffers, stop words into every shard's slots; bgabp_shard_p2p_*) against the single engine."""
    from paper_1904_04093_b200.gabp import GabpEngine, Layout
    from paper_1904_04093_b200.gabp import Schedule as GSchedule
    from paper_1904_04093_b200.shard import GpuShard, sharded_solve_p2p
    build, align, count, opt = PROBLEMS[name]
    A = build()
    b = _rhs(A.n)
    layouts = ShardLayout.partition(A.n, dia_halo(A), count, align=align)
    shards = _shards(A, b, layouts, range(count), GpuShard)
    status, its, detail, xs, hist = sharded_solve_p2p(shards, layouts, _r0(b), opt, spin=mode == "spin",
                                                      graph=mode == "graph")
    rep = GabpEngine(A, Layout.Dia).solve(b, GSchedule.parallel_flood(), opt)
    _assert_same(rep, status, its, detail, _gather(layouts, xs), hist)
    _assert_same(_oracle_solve(orc, A, b, opt), status, its, detail, _gather(layouts, xs), hist)


@pytest.mark.gpu
def test_gpu_peer_shards_config2_slab(orc):
    """Eight peer-connected shards of a 512 x 512 Poisson system (the config-2 operator), 300
    iterations: bit-identical to the single engine."""
    import paper_1904_04093_b200 as g
    from paper_1904_04093_b200.shard import GpuShard, sharded_solve_p2p
    A = g.poisson5(512, 512)
    b = _rhs(A.n, 11)
    opt = GabpOptions(tol=0.0, max_iter=300)
    layouts = ShardLayout.partition(A.n, dia_halo(A), 8, align=512)
    shards = _shards(A, b, layouts, range(8), GpuShard)
    status, its, detail, xs, hist = sharded_solve_p2p(shards, layouts, _r0(b), opt, graph=True)
    rep = g.GabpEngine(A).solve(b, g.Schedule.parallel_flood(), opt)
    _assert_same(rep, status, its, detail, _gather(layouts, xs), hist)
    _assert_same(_oracle_solve(orc, A, b, opt), status, its, detail, _gather(layouts, xs), hist)


def _ipc_worker(rank, world, port, name, q):
    """One process per shard, CUDA IPC mappings, host barrier between steps and decisions (the
    ranks share one GPU: device-side waits between processes are not used here)."""
    import torch
    import torch.distributed as dist
    from paper_1904_04093_b200.shard import GpuShard, sharded_solve_ipc
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        build, align, count, opt = PROBLEMS[name]
        A = build()
        b = _rhs(A.n)
        layouts = ShardLayout.partition(A.n, dia_halo(A), world, align=align)
        L = layouts[rank]
        shard = GpuShard(local_matrix(A, L), L, b[L.glo:L.ghi])
        status, its, detail, x, hist = sharded_solve_ipc(shard, layouts, _r0(b), opt, host_barrier=True)
        q.put((rank, status, its, detail, {rank: x}, hist))
        torch.cuda.synchronize()
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["grid5_sym", "grid5_nonsym", "grid7"])
def test_gpu_ipc_ranks_match_single_engine(orc, name):
    """Two processes, one shard each, neighbour buffers and slot arrays mapped with CUDA IPC."""
    import torch.multiprocessing as mp
    from paper_1904_04093_b200.gabp import GabpEngine, Layout
    from paper_1904_04093_b200.gabp import Schedule as GSchedule
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_ipc_worker, args=(r, 2, port, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=300) for _ in range(2)]
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    build, align, count, opt = PROBLEMS[name]
    A = build()
    b = _rhs(A.n)
    layouts = ShardLayout.partition(A.n, dia_halo(A), 2, align=align)
    xs = {}
    for rank, status, its, detail, x, hist in outs:
        xs.update(x)
    assert outs[0][1:4] == outs[1][1:4]
    rep = GabpEngine(A, Layout.Dia).solve(b, GSchedule.parallel_flood(), opt)
    _assert_same(rep, outs[0][1], outs[0][2], outs[0][3], _gather(layouts, xs), outs[0][5])
    _assert_same(_oracle_solve(orc, A, b, opt), outs[0][1], outs[0][2], outs[0][3], _gather(layouts, xs), outs[0][5])
