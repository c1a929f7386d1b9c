"""TEST HELPER: a torch-CPU implementation of the dist.py rank-operator protocol, so the
multi-rank protocol (maps, halo exchange + rank-ordered combine, owned reductions,
Jacobi / PCG loops, TorchTransport) can run over gloo on CPU without a GPU.  The local
element operator is the oracle's (j, e)-ordered product; nothing here is product code."""

from __future__ import annotations

import numpy as np
import torch


class CpuRankOperator:
    def __init__(self, A_e, b_e, indt, n_nodes, nd, maps, p):
        self.rank = p
        lo, hi = int(maps["bounds"][p]), int(maps["bounds"][p + 1])
        gl = maps["local"][p]
        self.global_ids = gl
        self.global_of_int = gl            # internal numbering = sorted local ids
        self.n = gl.numel()
        conn = torch.searchsorted(gl, torch.as_tensor(indt[:, lo:hi], dtype=torch.int64))
        self.conn = conn
        self.A = torch.as_tensor(np.ascontiguousarray(A_e[:, :, lo:hi]))
        self.b_e = torch.as_tensor(np.ascontiguousarray(b_e[:, lo:hi]))
        self.if_idx = {q: torch.searchsorted(gl, ids) for q, ids in maps["interface"][p].items()}
        self.all_if = (torch.unique(torch.cat(list(self.if_idx.values())))
                       if self.if_idx else torch.empty(0, dtype=torch.int64))
        self.owned = (maps["owner"][gl] == p).to(torch.uint8)
        free = torch.ones(self.n, dtype=torch.uint8)
        nd = torch.as_tensor(nd, dtype=torch.int64)
        mine = nd[torch.isin(nd, gl)]
        free[torch.searchsorted(gl, mine)] = 0
        self.free = free

    def _scatter(self, vals):  # vals (nb, n_e_local) -> node sums in (j, e) order
        out = torch.zeros(self.n, dtype=torch.float64)
        out.index_add_(0, self.conn.reshape(-1), vals.reshape(-1))
        return out

    def to_internal(self, x_global):
        return x_global[self.global_of_int].clone()

    def scatter_owned(self, v, out_global):
        m = self.owned.bool()
        out_global[self.global_of_int[m]] = v[m]

    def matvec_partial(self, x, out):
        nb = self.conn.shape[0]
        xg = [x[self.conn[i]] for i in range(nb)]
        loc = torch.stack([sum(self.A[i, c] * xg[c] for c in range(nb)) for i in range(nb)])
        out.copy_(self._scatter(loc))

    def rhs_partial(self):
        return self._scatter(self.b_e)

    def diag_partial(self):
        nb = self.conn.shape[0]
        return self._scatter(torch.stack([self.A[j, j] for j in range(nb)]))

    def gather(self, idx, v):
        return v[idx].clone()

    def combine(self, v, recvs):
        if not self.if_idx:
            return
        acc = torch.zeros(self.n, dtype=torch.float64)
        own = v[self.all_if].clone()
        for r in sorted(set(recvs) | {self.rank}):
            if r == self.rank:
                acc.index_add_(0, self.all_if, own)
            else:
                acc.index_add_(0, self.if_idx[r], recvs[r])
        v[self.all_if] = acc[self.all_if]

    def vec_dinv(self, diag):
        f = self.free.bool()
        if diag is not None:
            f = f & (diag != 0)
        d = torch.zeros(self.n, dtype=torch.float64)
        d[f] = 1.0 / diag[f] if diag is not None else 1.0
        return d

    def vec_jacobi(self, omega, b, s, dinv, x, x_out, r_out, red):
        r = torch.where(self.free.bool(), b - s, torch.zeros_like(b))
        red.copy_((r[self.owned.bool()] ** 2).sum().reshape(1))
        if r_out is not None:
            r_out.copy_(r)
        if x_out is not None:
            x_out.copy_(x + omega * (dinv * r) if dinv is not None else x + omega * r)

    def vec_pcg_q(self, p, q, red):
        q.copy_(torch.where(self.free.bool(), q, torch.zeros_like(q)))
        red.copy_((p * q)[self.owned.bool()].sum().reshape(1))

    def vec_pcg_update(self, rz, pq, dinv, x, r, p, q, red):
        rz, pq = float(rz[0]), float(pq[0])
        alpha = rz / pq if pq != 0.0 else 0.0
        x.add_(alpha * p)
        r.sub_(alpha * q)
        o = self.owned.bool()
        red.copy_(torch.stack([(r[o] ** 2).sum(), (r * (dinv * r))[o].sum()]))

    def vec_pcg_direction(self, rz_old, rz_new, dinv, r, p):
        beta = float(rz_new[0]) / float(rz_old[0]) if float(rz_old[0]) != 0.0 else 0.0
        p.copy_(dinv * r + beta * p)

    def vec_cg1_update(self, cur, prev, rr0, tol, ctl, dinv, x, r, u, w, p, s, nxt):
        """ebs_vec_cg1_update (include/ebs.h) restated with torch CPU ops."""
        if int(ctl[0]):
            return
        gamma, delta, rr = (float(v) for v in cur[0:3])
        nk = rr ** 0.5 if rr >= 0 else float("nan")
        if not np.isfinite(nk) or (tol >= 0 and nk <= tol * float(rr0[0]) ** 0.5):
            ctl[1] = ctl[2]
            ctl[3] = 0 if np.isfinite(nk) else 1
            ctl[0] = 1
            return
        g_prev, a_prev = float(prev[0]), float(prev[3])
        beta = gamma / g_prev if g_prev != 0.0 else 0.0
        denom = delta - beta * gamma / a_prev if (beta != 0.0 and a_prev != 0.0) else delta
        alpha = gamma / denom if denom != 0.0 else 0.0
        p.copy_(u + beta * p)
        s.copy_(w + beta * s)
        x.add_(alpha * p)
        r.sub_(alpha * s)
        u.copy_(dinv * r)
        o = self.owned.bool()
        nxt[0] = (r * u)[o].sum()
        nxt[2] = (r * r)[o].sum()
        cur[3] = alpha
        ctl[2] += 1

    def dot_owned(self, x, y, red):
        red.copy_((x * y)[self.owned.bool()].sum().reshape(1))

    def zeros(self, n=None):
        return torch.zeros(self.n if n is None else n, dtype=torch.float64)
