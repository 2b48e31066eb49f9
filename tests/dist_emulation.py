"""CPU emulation of the distributed path's local compute (test infrastructure).

Implements the `GpuBackend` interface of paper_1706_06844_b200.distributed
with torch CPU tensors and numpy, building every level from the CPU oracle
(coefficients, grid, weights, transfers) so the gloo tests exercise the real
partitioning / all-to-all / halo / agglomeration logic against the oracle."""
import math

import numpy as np
import torch

from oracles import spec


def toeplitz_dense(gamma, n, pq, orc):
    _, w = orc.weights(gamma, max(n, 2), pq)
    col = -w[1:n + 1]
    row = np.zeros(n)
    row[0] = -w[1]
    if n > 1:
        row[1] = -w[0]
    i, j = np.indices((n, n))
    return np.where(i >= j, col[np.clip(i - j, 0, n - 1)], row[np.clip(j - i, 0, n - 1)])


class _Level:
    pass


class EmuBackend:
    def __init__(self, orc, cfg, pq=None):
        self.orc, self.cfg = orc, cfg
        self.pq = pq

    def zeros(self, n):
        return torch.zeros(n, dtype=torch.float64)

    def to_host(self, t):
        return t.numpy().copy()

    def from_host(self, a):
        return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64)

    # full level description (scaled like build_geometric_hierarchy)
    def level(self, problem, fine, dims, steps):
        d1, d2 = dims
        s = spec(self.cfg, n1=d1, n2=d2, steps=steps)
        g = self.orc.grid(s)
        gf = self.orc.grid(spec(self.cfg, n1=fine[0], n2=fine[1], steps=steps))
        scale = 1.0 if tuple(dims) == tuple(fine) else math.pow(gf["hx"] / g["hx"], problem.alpha)
        dp, dm, ep, em = self.orc.coefficients(s)
        pq = problem.pq
        L = _Level()
        L.d1, L.d2 = d1, d2
        L.Ta = toeplitz_dense(problem.alpha, d1, pq, self.orc)
        L.Tb = toeplitz_dense(problem.beta, d2, pq, self.orc)
        diag = g["inv_r"] + (dp + dm) * L.Ta[0, 0] + g["s_over_r"] * (ep + em) * L.Tb[0, 0]
        L.inv_r, L.s_over_r = g["inv_r"] * scale, g["s_over_r"] * scale
        L.dp, L.dm, L.ep, L.em, L.diag = dp * scale, dm * scale, ep, em, diag * scale
        return L

    def slab(self, problem, fine, dims, steps, m, rows, cols):
        L = self.level(problem, fine, dims, steps)
        L.r0, L.r1, L.c0, L.c1 = rows[0], rows[1], cols[0], cols[1]
        return L, L.diag[L.r0 * L.d1:L.r1 * L.d1].copy()

    def ypass(self, L, xT, QT, sign):
        nc = L.c1 - L.c0
        X = xT.numpy().reshape(nc, L.d2)
        ep = L.ep.reshape(L.d2, L.d1)[:, L.c0:L.c1].T
        em = L.em.reshape(L.d2, L.d1)[:, L.c0:L.c1].T
        ty = X @ L.Tb.T
        tt = X @ L.Tb
        QT.copy_(torch.from_numpy((sign * L.s_over_r * (ep * ty + em * tt)).reshape(-1)))

    def xpass(self, L, x, Q, out, sign, epi, b=None, dinv=None, omega=0.0, src=None, src_scale=0.0):
        nr = L.r1 - L.r0
        X = x.numpy().reshape(nr, L.d1).copy()
        sl = slice(L.r0 * L.d1, L.r1 * L.d1)
        dp, dm = L.dp[sl].reshape(nr, L.d1), L.dm[sl].reshape(nr, L.d1)
        y = L.inv_r * X + sign * dp * (X @ L.Ta.T) + sign * dm * (X @ L.Ta) + Q.numpy().reshape(nr, L.d1)
        y = y.reshape(-1)
        if epi == 1:
            y = y + src_scale * src.numpy()
        elif epi == 2:
            y = b.numpy() - y
        elif epi == 3:
            y = X.reshape(-1) + omega * dinv.numpy() * (b.numpy() - y)
        out.copy_(torch.from_numpy(np.ascontiguousarray(y)))

    def transpose(self, inp, out, rows, cols):
        if rows and cols:
            out.copy_(inp.reshape(rows, cols).t().reshape(-1))

    def permute(self, inp, out, nc, d2, offsets, direction):
        if not (nc and d2):
            return
        full = torch.zeros(nc, d2, dtype=torch.float64)
        if direction == 0:
            for s in range(len(offsets) - 1):
                a, b = offsets[s], offsets[s + 1]
                full[:, a:b] = inp[nc * a:nc * b].reshape(nc, b - a)
            out.copy_(full.reshape(-1))
        else:
            src = inp.reshape(nc, d2)
            for s in range(len(offsets) - 1):
                a, b = offsets[s], offsets[s + 1]
                out[nc * a:nc * b] = src[:, a:b].reshape(-1)

    def transfer_rows(self, n1, n2, cx, cy, op, add, inp, in_lo, out, out_lo, out_rows):
        if not out_rows:
            return
        k1 = (n1 - n1 % 2) // 2 if cx else n1
        k2 = (n2 - n2 % 2) // 2 if cy else n2
        if op == 0:  # coarse rows window -> fine rows window
            full = np.zeros(k1 * k2)
            a = inp.numpy()
            full[in_lo * k1:in_lo * k1 + a.size] = a
            f = self.orc.transfer(n1, n2, cx, cy, 0, full)[out_lo * n1:(out_lo + out_rows) * n1]
            if add:
                out += torch.from_numpy(f)
            else:
                out.copy_(torch.from_numpy(f))
        else:
            full = np.zeros(n1 * n2)
            a = inp.numpy()
            full[in_lo * n1:in_lo * n1 + a.size] = a
            c = self.orc.transfer(n1, n2, cx, cy, op, full)[out_lo * k1:(out_lo + out_rows) * k1]
            out.copy_(torch.from_numpy(np.ascontiguousarray(c)))

    def vec(self, op, n, a, x, y, out):
        if not n:
            return
        if op == 0:
            out.copy_(a * x * y)
        elif op == 1:
            out += a * x
        elif op == 2:
            out += a * x * y
        else:
            out.copy_(x * a)

    def dot(self, x, y, out_slot):
        out_slot[0] = torch.dot(x, y)

    def axpy_dev(self, a_dev, sgn, x, out):
        out += sgn * a_dev[0] * x

    def coarse_vcycle_factory(self, problem, fine, dims_tail, steps, m, omega, coarse, sweeps):
        levels = []
        for d in dims_tail:
            L = self.level(problem, fine, d, steps)
            n = L.d1 * L.d2
            I1, I2 = np.eye(L.d1), np.eye(L.d2)
            A = (L.inv_r * np.eye(n) + np.diag(L.dp) @ np.kron(I2, L.Ta) + np.diag(L.dm) @ np.kron(I2, L.Ta.T)
                 + L.s_over_r * (np.diag(L.ep) @ np.kron(L.Tb, I1) + np.diag(L.em) @ np.kron(L.Tb.T, I1)))
            levels.append((A, 1.0 / L.diag, L.d1, L.d2))
        orc = self.orc

        def cycle(l, b, x, zero):
            A, dinv, d1, d2 = levels[l]
            if l + 1 == len(levels):
                if coarse == 0:
                    return np.linalg.solve(A, b)
                if coarse == 2:
                    return x
                x = omega * dinv * b if zero else x + omega * dinv * (b - A @ x)
                for _ in range(1, sweeps):
                    x = x + omega * dinv * (b - A @ x)
                return x
            x = omega * dinv * b if zero else x + omega * dinv * (b - A @ x)
            r = b - A @ x
            _, _, e1, e2 = levels[l + 1]
            cx, cy = e1 < d1, e2 < d2
            bc = orc.transfer(d1, d2, cx, cy, 1, r)
            xc = cycle(l + 1, bc, np.zeros_like(bc), True)
            x = x + orc.transfer(d1, d2, cx, cy, 0, xc)
            return x + omega * dinv * (b - A @ x)

        def run(b_full):
            b = b_full.numpy()
            return torch.from_numpy(cycle(0, b, np.zeros_like(b), True))
        return run
