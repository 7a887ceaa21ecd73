"""CPU stand-in for paper_1904_04093_b200.shard.GpuShard (test infrastructure only).

Implements, with numpy over the same DIA slot layout, exactly what the GPU shard calls do:
the fused flood step k_flood_solve_dia restricted to the owned nodes, k_shard_fold,
k_shard_decide + solve_decide_lag2, k_shard_pack / k_shard_unpack (kernels.cuh).  It lets the
sharded driver (halo exchange, MAX all-reduce, stop agreement) run under gloo with world_size 2
on a machine without a GPU; the tests check the result against the oracle's single-process solve.
numpy evaluates every elementwise op in IEEE binary64 with round-to-nearest, the same as the
kernel's __dadd_rn/__dmul_rn/__ddiv_rn, and the terms are accumulated in the kernel's slot order.
"""
from __future__ import annotations

import numpy as np
import torch

FLOOR = 1e-300
NONE = (1 << 64) - 1
TOP = (1 << 63) - 1


def _nan_skip_abs(v):
    a = np.abs(v)
    return np.where(np.isnan(a), 0.0, a)


def _bits(d: float) -> int:
    return int(np.array([d], np.float64).view(np.uint64)[0])


def _dbl(b: int) -> float:
    return float(np.array([b], np.uint64).view(np.float64)[0])


class CpuShard:
    def __init__(self, A_local, L, b_local):
        self.L = L
        n = A_local.n
        ro, ci, v = A_local.row_offsets, A_local.col_indices, A_local.values
        rows = np.repeat(np.arange(n), np.diff(ro))
        off = ci.astype(np.int64) - rows
        nd = off != 0
        offs = np.unique(np.concatenate([off[nd], -off[nd]]))
        self.off = offs
        self.S = S = len(offs)
        self.nneg = int(np.sum(offs < 0))
        slot = {int(o): s for s, o in enumerate(offs)}
        self.rev = np.array([slot[-int(o)] for o in offs], np.int64)
        self.diag = np.zeros(n)
        self.IN = np.zeros((S, n), bool)    # message j+off -> j exists (A_{j,j+off} stored)
        self.OUT = np.zeros((S, n), bool)   # message j -> j+off exists (A_{j+off,j} stored)
        self.rowv = np.zeros((S, n))        # A_{j,j+off}
        self.c = np.zeros((S, n))           # A_{j+off,j}
        d = ~nd
        self.diag[rows[d]] = v[d]
        for k in np.nonzero(nd)[0]:
            i, j, s = rows[k], ci[k], slot[int(off[k])]
            self.IN[s, i] = True
            self.rowv[s, i] = v[k]
            rs = self.rev[s]
            self.OUT[rs, j] = True
            self.c[rs, j] = v[k]
        self.n = n
        self.b = np.ascontiguousarray(b_local, np.float64)
        self.msg = [np.zeros((S, n, 2)), np.zeros((S, n, 2))]
        self.red4 = torch.zeros(4, dtype=torch.int64)
        self.x = [torch.zeros(n, dtype=torch.float64) for _ in range(2)]  # x(k) in slot k & 1

    # ---- control block (Ctrl) --------------------------------------------------------------
    def begin(self, opt, r0):
        for m in self.msg:
            m[:] = 0.0
        for x in self.x:
            x.zero_()
        self.tol, self.divergence, self.stop, self.max_iter = opt.tol, opt.divergence_factor, int(opt.stop), opt.max_iter
        self.r0 = r0
        self.hist = np.zeros(opt.max_iter + 2)
        self.hist[0] = r0
        self.done_, self.step, self.status, self.iterations, self.solx = 0, 1, 2, 0, 0
        self.detail_kind, self.detail_key = 0, 0
        self.epiv, self.npiv = [NONE] * 4, [NONE] * 4
        self.delta, self.rmax = [0] * 4, [0] * 4

    def compute(self):
        if self.done_:
            return
        t = self.step
        mi = self.msg[0] if t & 1 else self.msg[1]
        mo = self.msg[1] if t & 1 else self.msg[0]
        xw = self.x[(t - 1) & 1].numpy()
        xr = self.x[(t - 2) & 1].numpy()
        L, S, n, g = self.L, self.S, self.n, self.L.glo
        J = np.arange(L.own_lo, L.own_hi)
        IN, OUT = self.IN[:, J], self.OUT[:, J]
        lam = mi[:, J, 0]
        mm = mi[:, J, 1]
        cc = np.where(OUT, self.c[:, J], 0.0)
        dj, bj = self.diag[J], self.b[J]
        sig = np.zeros(len(J))
        acc = bj.copy()
        for s in range(S):
            if s == self.nneg:
                sig = sig + dj
            acc = np.where(IN[s], acc + mm[s], acc)
            sig = np.where(IN[s] & OUT[s], sig + lam[s] * cc[s], sig)
        if self.nneg == S:
            sig = sig + dj
        npiv = NONE
        if t >= 2:
            xw[J] = acc / sig
            bad = np.abs(sig) < FLOOR
            if bad.any():
                npiv = int(J[bad][0]) + g
        rmax = 0.0
        if t >= 3:
            r = bj.copy()
            for s in range(S):
                if s == self.nneg:
                    r = r - dj * xr[J]
                q = np.clip(J + self.off[s], 0, n - 1)
                r = np.where(IN[s], r - self.rowv[s, J] * xr[q], r)
            if self.nneg == S:
                r = r - dj * xr[J]
            rmax = float(np.max(_nan_skip_abs(r))) if len(J) else 0.0
        dmax, epiv = 0.0, NONE
        for s in range(S):
            o = OUT[s]
            if not o.any():
                continue
            js = J[o]
            k = js + self.off[s]
            den = sig[o] - lam[s][o] * cc[s][o]
            bad = np.abs(den) < FLOOR
            if bad.any():
                keys = ((js[bad] + g).astype(np.int64) << 32) | (k[bad] + g)
                epiv = min(epiv, int(keys.min()))
            nl = -cc[s][o] / den
            nm = nl * (acc[o] - mm[s][o])
            rs = self.rev[s]
            old = mi[rs, k]
            dmax = max(dmax, float(np.max(np.maximum(_nan_skip_abs(nl - old[:, 0]), _nan_skip_abs(nm - old[:, 1])))))
            mo[rs, k, 0] = nl
            mo[rs, k, 1] = nm
        # k_shard_fold
        self.red4[0] = _bits(rmax) if t >= 3 else 0
        self.red4[1] = _bits(dmax)
        self.red4[2] = 0 if epiv == NONE else TOP - epiv
        self.red4[3] = 0 if (t < 2 or npiv == NONE) else TOP - npiv

    def decide(self):  # k_shard_decide + solve_decide_lag2
        if self.done_:
            return
        t = self.step
        w = [int(v) for v in self.red4.tolist()]
        if t >= 3:
            self.rmax[(t - 2) & 3] = w[0]
        self.delta[t & 3] = w[1]
        self.epiv[t & 3] = TOP - w[2] if w[2] else NONE
        if t >= 2:
            self.npiv[(t - 1) & 3] = TOP - w[3] if w[3] else NONE
        if t >= 3:
            k = t - 2
            q = k & 3
            self.iterations, self.solx = k, k
            if self.npiv[q] != NONE:
                self.status, self.detail_kind, self.detail_key, self.done_ = 1, 1, self.npiv[q], 1
                return
            r = _dbl(self.rmax[q])
            self.hist[k] = r
            if not np.isfinite(r) or r > self.divergence * self.r0:
                self.status, self.detail_kind, self.done_ = 1, 3, 1
                return
            if (r <= self.tol) if self.stop == 0 else (_dbl(self.delta[q]) <= self.tol):
                self.status, self.done_ = 0, 1
                return
            if k >= self.max_iter:
                self.status, self.done_ = 2, 1
                return
            self.npiv[q], self.rmax[q], self.delta[q] = NONE, 0, 0
        if t >= 2:
            q = (t - 1) & 3
            if self.epiv[q] != NONE:
                self.status, self.iterations, self.solx = 1, t - 1, t - 2
                self.detail_kind, self.detail_key, self.done_ = 2, self.epiv[q], 1
                return
            self.epiv[q] = NONE
            if self.npiv[q] != NONE:  # node pivot of x-stage t-1, decided one step early
                self.status, self.iterations, self.solx = 1, t - 1, t - 1
                self.detail_kind, self.detail_key, self.done_ = 1, self.npiv[q], 1
                return
        self.step = t + 1

    # ---- halo --------------------------------------------------------------------------------
    def pack(self, which, lo, length):
        return torch.from_numpy(np.ascontiguousarray(self.msg[which][:, lo:lo + length, :]).reshape(-1))

    def unpack(self, which, buf, lo, length, sender_lo, sender_hi):
        recv = buf.numpy().reshape(self.S, length, 2)
        node = np.arange(lo, lo + length)
        for s in range(self.S):
            snd = node + self.off[s]
            sel = (snd >= sender_lo) & (snd < sender_hi)
            self.msg[which][s, node[sel]] = recv[s, sel]

    def new_buffer(self, count):
        return torch.empty(count, dtype=torch.float64)

    def done(self):
        return bool(self.done_)

    def end(self, max_iter):
        detail = {1: f"zero pivot at node {self.detail_key}",
                  2: f"zero pivot on edge {self.detail_key >> 32}->{self.detail_key & 0xffffffff}",
                  3: "residual blowup"}.get(self.detail_kind, "") if self.status == 1 else ""
        x = self.x[self.solx & 1].numpy().copy()
        if self.status == 1 and self.detail_kind == 1:  # x(k) below the pivot node, x(k-1) from it on
            glob = np.arange(self.n) + self.L.glo
            x = np.where(glob < self.detail_key, x, self.x[(self.solx - 1) & 1].numpy())
        x = x[self.L.own_lo:self.L.own_hi]
        nh = self.iterations + (0 if self.status == 1 and detail.startswith("zero pivot") else 1)
        return self.status, self.iterations, detail, x, self.hist[:nh].copy()
