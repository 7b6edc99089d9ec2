"""CPU stand-in for one rank's KfacEngine, used to test the sharded-step
orchestration (paper_2405_15603_b200/dist.py) under gloo without a GPU.

It implements the same phase contract as the device engine — phase 1 leaves
UNNORMALISED per-shard sums in ``reduce_buffer()``, phase 3 leaves per-candidate
sums of squared residuals in ``linesearch_buffer()``, normalisation by the
global point counts happens after the all-reduce — with the oracle's math.
Test infrastructure only.
"""

import numpy as np
import torch

from oracle import kfac_oracle as orc


class CpuShardEngine:
    def __init__(self, weights, biases, x_int, x_bnd, targets, problem, n_glob, nb_glob, *, ema,
                 damping, momentum, ls_min_exp=-30, ls_max_exp=0):
        self.w = [np.array(w) for w in weights]
        self.b = [np.array(b) for b in biases]
        self.x, self.xb, self.tg = x_int, x_bnd, targets
        self.prob = problem
        self.cd = orc.coeffs_of(problem)
        self.ng, self.nbg = float(n_glob), float(nb_glob)
        self.ema, self.lam, self.mu = ema, damping, momentum
        self.grid = [2.0 ** e for e in range(ls_min_exp, ls_max_exp + 1)]
        L = len(self.w)
        ps = [w.shape[1] + 1 for w in self.w]
        qs = [w.shape[0] for w in self.w]
        self.kf = orc.OracleKfac([np.eye(p) for p in ps], [np.eye(q) for q in qs],
                                 [np.eye(p) for p in ps], [np.eye(q) for q in qs], ema, damping)
        self.prev = [np.zeros((q, p)) for p, q in zip(ps, qs)]
        self.sizes = [(p * p, q * q, q * p) for p, q in zip(ps, qs)]
        n_red = sum(2 * a + 2 * b + 2 * g for a, b, g in self.sizes) + 2
        self.red = torch.zeros(n_red, dtype=torch.float64)
        self.ls = torch.zeros(2 * len(self.grid), dtype=torch.float64)
        D = sum(g for _, _, g in self.sizes)
        self.gvb = torch.zeros(4 * D, dtype=torch.float64)
        self.L = L
        self.scalars = np.zeros(4)

    def reduce_buffer(self):
        return self.red

    def linesearch_buffer(self):
        return self.ls

    def gvp_buffer(self):
        return self.gvb

    def _pack(self, parts):
        flat = np.concatenate([np.asarray(p).ravel() for p in parts])
        self.red.copy_(torch.from_numpy(flat))

    def _unpack(self):
        v = self.red.numpy()
        off = 0
        out = {k: [] for k in ("ai", "bi", "ab", "bb", "gi", "gb")}
        for key, idx in (("ai", 0), ("bi", 1), ("ab", 0), ("bb", 1), ("gi", 2), ("gb", 2)):
            for l, sz in enumerate(self.sizes):
                n = sz[idx]
                shape = {0: (int(np.sqrt(n)),) * 2, 1: (int(np.sqrt(n)),) * 2,
                         2: self.prev[l].shape}[idx]
                out[key].append(v[off:off + n].reshape(shape))
                off += n
        return out, v[off], v[off + 1]

    def direction_buffer(self):
        return self.dirbuf

    def phase(self, name, owned=None):
        if name == "precondition_owned":
            self._precondition_owned(owned)
        else:
            getattr(self, "_" + name)()

    def _accumulate(self):
        lin_in, pre, (u, gu, lu) = orc.taylor_forward(self.w, self.b, self.x, self.cd)
        r = np.asarray(self.prob.residual(self.x, u, gu, lu))
        du, dg, dop = self.prob.residual_grads(self.x, u, gu, lu)
        n = self.x.shape[0]
        seeds = np.concatenate([np.broadcast_to(du, (n,))[:, None], np.broadcast_to(dg, self.x.shape),
                                np.broadcast_to(dop, (n,))[:, None]], axis=1)
        gbar = orc.taylor_backward(self.w, pre, seeds, self.cd)
        ub, bin_, bpre = orc.plain_forward(self.w, self.b, self.xb)
        res = ub - self.tg
        bgr = orc.plain_backward(self.w, bpre, np.ones(res.size))
        ai, bi, ab, bb, gi, gb = [], [], [], [], [], []
        for l in range(self.L):
            zh = orc._augment_rows(lin_in[l]).reshape(-1, lin_in[l].shape[2] + 1)
            g = gbar[l].reshape(zh.shape[0], -1)
            ai.append(zh.T @ zh)
            bi.append(g.T @ g)
            gi.append((gbar[l] * r[:, None, None]).reshape(zh.shape[0], -1).T @ zh)
            zb = np.hstack([bin_[l], np.ones((bin_[l].shape[0], 1))])
            ab.append(zb.T @ zb)
            bb.append(bgr[l].T @ bgr[l])
            gb.append((bgr[l] * res[:, None]).T @ zb)
        self._pack(ai + bi + ab + bb + gi + gb + [np.array([r @ r, res @ res])])

    def _precondition(self):
        s, ssi, ssb = self._unpack()
        S = self.x.shape[1] + 2
        beta = self.ema
        kf = self.kf
        kf.a_int = [beta * o + (1 - beta) * orc._sym(a / (self.ng * S)) for o, a in zip(kf.a_int, s["ai"])]
        kf.b_int = [beta * o + (1 - beta) * orc._sym(b / self.ng) for o, b in zip(kf.b_int, s["bi"])]
        kf.a_bnd = [beta * o + (1 - beta) * orc._sym(a / self.nbg) for o, a in zip(kf.a_bnd, s["ab"])]
        kf.b_bnd = [beta * o + (1 - beta) * orc._sym(b / self.nbg) for o, b in zip(kf.b_bnd, s["bb"])]
        grads = [gi / self.ng + gb / self.nbg for gi, gb in zip(s["gi"], s["gb"])]
        self.scalars[0] = ssi / (2 * self.ng)
        self.scalars[1] = ssb / (2 * self.nbg)
        delta = orc.precondition(kf, grads)
        self.delta = delta
        self.grads = grads
        self.dir = [d + self.mu * p for d, p in zip(delta, self.prev)]

    # distributed solves: Delta of the owned layers, zeros elsewhere, + 8 status slots
    def _precondition_owned(self, owned):
        self._precondition()
        parts = [d if own else np.zeros_like(d) for d, own in zip(self.delta, owned)]
        self.dirbuf = torch.from_numpy(np.concatenate([p.ravel() for p in parts] + [np.zeros(8)]))
        self.delta = None

    def _direction(self):
        v = self.dirbuf.numpy()
        assert not v[-8:].any()
        off, delta = 0, []
        for p in self.prev:
            delta.append(v[off:off + p.size].reshape(p.shape).copy())
            off += p.size
        self.delta = delta
        self.dir = [d + self.mu * p for d, p in zip(delta, self.prev)]

    def _linesearch(self):
        out = np.zeros(2 * len(self.grid))
        for k, a in enumerate(self.grid):
            ws = [w + a * m[:, :-1] for w, m in zip(self.w, self.dir)]
            bs = [b + a * m[:, -1] for b, m in zip(self.b, self.dir)]
            _, _, (u, gu, lu) = orc.taylor_forward(ws, bs, self.x, self.cd)
            r = np.asarray(self.prob.residual(self.x, u, gu, lu))
            ub, _, _ = orc.plain_forward(ws, bs, self.xb)
            res = ub - self.tg
            out[2 * k], out[2 * k + 1] = r @ r, res @ res
        self.ls.copy_(torch.from_numpy(out))

    def _update(self):
        v = self.ls.numpy()
        best, best_a = np.inf, None
        for k, a in enumerate(self.grid):
            loss = v[2 * k] / (2 * self.ng) + v[2 * k + 1] / (2 * self.nbg)
            if np.isfinite(loss) and loss < best:
                best, best_a = loss, a
        self.scalars[2] = best_a
        self.scalars[3] = self.mu
        self.w = [w + best_a * m[:, :-1] for w, m in zip(self.w, self.dir)]
        self.b = [b + best_a * m[:, -1] for b, m in zip(self.b, self.dir)]
        self.prev = [best_a * m for m in self.dir]

    # KFAC*: local (unnormalised) Gramian-vector products from this shard's Jacobian rows
    def _star_gvp(self):
        cd = self.cd
        x = self.x

        class B:  # minimal batch view for the oracle
            pass

        b = B()
        b.interior, b.boundary, b.boundary_targets = self.x, self.xb, self.tg
        ev = orc.evaluate_batch(self.w, self.b, b, self.prob, cd)
        ri, rb = orc.jacobian_rows(ev)
        dv, pv = orc._vec(self.delta), orc._vec(self.prev)
        parts = [ri.T @ (ri @ dv), rb.T @ (rb @ dv), ri.T @ (ri @ pv), rb.T @ (rb @ pv)]
        self.gvb.copy_(torch.from_numpy(np.concatenate(parts)))
        del x

    def _star_update(self):
        D = self.gvb.numel() // 4
        v = self.gvb.numpy()
        g_dv = v[:D] / self.ng + v[D:2 * D] / self.nbg
        g_pv = v[2 * D:3 * D] / self.ng + v[3 * D:] / self.nbg
        dv, pv, gv = orc._vec(self.delta), orc._vec(self.prev), orc._vec(self.grads)
        lam = self.lam
        m11, rhs1 = float(dv @ g_dv + lam * dv @ dv), float(dv @ gv)
        have_prev = bool(pv @ pv > 0.0)
        if have_prev:
            m12, m22, rhs2 = float(dv @ g_pv + lam * dv @ pv), float(pv @ g_pv + lam * pv @ pv), float(pv @ gv)
        else:
            m12 = m22 = rhs2 = 0.0
        alpha, mu = orc.solve_quadratic_model(have_prev, m11, m12, m22, rhs1, rhs2)
        upd = [alpha * d + mu * p for d, p in zip(self.delta, self.prev)]
        self.w = [w + u[:, :-1] for w, u in zip(self.w, upd)]
        self.b = [b + u[:, -1] for b, u in zip(self.b, upd)]
        self.prev = upd
        self.scalars[2], self.scalars[3] = alpha, mu

    def finish_step(self):
        return self.scalars.copy(), 0
