"""Python statement of the y-slab multi-GPU time step.

The product path is C++ (csrc/dist.cu behind fde_dist_* / fde.SlabMarch, NCCL,
or virtual ranks on one GPU).  This module states the same algorithm over a
backend interface; tests/test_distributed.py runs it on a numpy backend with
gloo at world size 2 and 3 on CPU (partition, halo rules, GMRES control flow)
and tests/test_gpu_distributed.py on the library's slab kernels at world 1.

One process per GPU.  Rank r owns grid rows [r0, r1) of every multigrid level
(x index fastest, so a row is n1 contiguous doubles):

* row (x-direction) Toeplitz lines are slab-local;
* column (y-direction) lines need an all-to-all transpose: each rank sends
  its slab, transposed, column block by column block, runs the column pass
  on the columns it then owns, and sends the result Q back the same way;
* restriction / prolongation along y read one halo row from each neighbour
  (only on levels that coarsen y; semicoarsened x-only levels are local);
* levels below `agglomerate` unknowns are replicated: the restricted rhs is
  all-gathered and every rank runs the rest of the V-cycle locally, so the
  coarse tail pays no collective latency;
* Krylov inner products are local partials combined in rank order
  (all-gather + ordered sum: the same bits on every rank and every run).

The algorithm is the reference's exactly (same level plan, transfers,
smoothing, GMRES control flow); only the partitioning is new, so parity is
checked against the single-GPU path / CPU oracle.  Local compute goes through
a backend: `GpuBackend` (libfde_b200 kernels on CUDA tensors, NCCL) for real
runs, or a numpy emulation in the tests (gloo on CPU).
"""
from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np

from . import (COARSE_LU, COARSE_NONE, COARSE_SWEEPS, Problem, _check, _stream, load_library,
               plan_level_dims)

EPI_STORE, EPI_RHS, EPI_RESID, EPI_JACOBI = 0, 1, 2, 3


def split_ranges(n: int, parts: int) -> list:
    """Balanced contiguous ranges: offsets[0..parts]."""
    return [n * r // parts for r in range(parts + 1)]


def coarse_size(n: int) -> int:  # multigrid.cpp:114
    return (n - n % 2) // 2


def induced_coarse_rows(fine_offsets: list, d2: int, coarsen_y: bool) -> list:
    """Coarse row b belongs to the rank owning its centre fine row 2b+1-par."""
    if not coarsen_y:
        return list(fine_offsets)
    par = (d2 + 1) % 2
    k2 = coarse_size(d2)
    out = []
    for f in fine_offsets:  # first coarse row whose centre is >= f
        b = 0 if f <= 0 else max(0, -(-(f - 1 + par) // 2))
        out.append(min(b, k2))
    out[-1] = k2
    return out


# --------------------------------------------------------------------- backends
class GpuBackend:
    """Local compute on CUDA tensors through the C ABI (include/fde_b200.h)."""

    def __init__(self, device):
        import torch
        self.torch = torch
        self.device = device
        self.lib = load_library()

    def zeros(self, n):
        return self.torch.zeros(n, dtype=self.torch.float64, device=self.device)

    def to_host(self, t):
        return t.cpu().numpy()

    def from_host(self, a):
        return self.torch.tensor(np.ascontiguousarray(a), dtype=self.torch.float64, device=self.device)

    @staticmethod
    def _p(t):
        return t.data_ptr() if t is not None else None

    def slab(self, problem: Problem, fine, dims, steps, m, rows, cols):
        h = ctypes.c_void_p()
        s = problem.c_struct()
        _check(self.lib.fde_slab_create(ctypes.byref(s), fine[0], fine[1], dims[0], dims[1], steps, m,
                                        rows[0], rows[1], cols[0], cols[1], ctypes.byref(h)))
        nr = rows[1] - rows[0]
        d = np.zeros(nr * dims[0])
        _check(self.lib.fde_slab_diagonal(h, d.ctypes.data_as(ctypes.POINTER(ctypes.c_double))))
        return h, d

    def ypass(self, h, xT, QT, sign):
        _check(self.lib.fde_slab_ypass(h, self._p(xT), self._p(QT), sign, _stream()))

    def xpass(self, h, x, Q, out, sign, epi, b=None, dinv=None, omega=0.0, src=None, src_scale=0.0):
        _check(self.lib.fde_slab_xpass(h, self._p(x), self._p(Q), self._p(out), sign, epi, self._p(b),
                                       self._p(dinv), omega, self._p(src), src_scale, _stream()))

    def transpose(self, inp, out, rows, cols):
        if rows and cols:
            _check(self.lib.fde_transpose(self._p(inp), self._p(out), rows, cols, _stream()))

    def permute(self, inp, out, nc, d2, offsets, direction):
        if nc and d2:
            off = (ctypes.c_longlong * len(offsets))(*offsets)
            _check(self.lib.fde_block_permute(self._p(inp), self._p(out), nc, d2, off, len(offsets) - 1,
                                              direction, _stream()))

    def transfer_rows(self, n1, n2, cx, cy, op, add, inp, in_lo, out, out_lo, out_rows):
        if out_rows:
            _check(self.lib.fde_transfer_rows(n1, n2, int(cx), int(cy), op, int(add), self._p(inp), in_lo,
                                              self._p(out), out_lo, out_rows, _stream()))

    def vec(self, op, n, a, x, y, out):
        if n:
            _check(self.lib.fde_vec(op, n, a, self._p(x), self._p(y), self._p(out), _stream()))

    def dot(self, x, y, out_slot):
        _check(self.lib.fde_dot(x.numel(), self._p(x), self._p(y), self._p(out_slot), 0, _stream()))

    def axpy_dev(self, a_dev, sgn, x, out):
        if x.numel():
            _check(self.lib.fde_axpy_dev(x.numel(), self._p(a_dev), sgn, self._p(x), self._p(out), _stream()))

    def coarse_vcycle_factory(self, problem, fine, dims_tail, steps, m, omega, coarse, sweeps):
        from . import MgHierarchy, StructuredFdeOperator
        levels = []
        hx_f = (problem.bx - problem.ax) / (fine[0] + 1)
        for (d1, d2) in dims_tail:
            op = StructuredFdeOperator.assemble(problem, d1, d2, steps, m)
            if (d1, d2) != tuple(fine):
                op.scale(math.pow(hx_f / ((problem.bx - problem.ax) / (d1 + 1)), problem.alpha))
            levels.append(op)
        h = MgHierarchy.from_levels(levels, omega, coarse, sweeps)

        def run(b_full):
            return h.vcycle(b_full, None, True)
        return run


# --------------------------------------------------------------------- context
@dataclass
class DistContext:
    rank: int
    world: int
    backend: object

    def all_to_all(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist
        if self.world == 1:
            out.copy_(inp)
            return
        dist.all_to_all_single(out, inp, out_splits, in_splits)

    def ordered_sum(self, local_scalar):
        """Sum of one device scalar per rank, in rank order (deterministic)."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return local_scalar.reshape(())
        parts = torch.empty(self.world, dtype=local_scalar.dtype, device=local_scalar.device)
        dist.all_gather_into_tensor(parts, local_scalar.reshape(1))
        acc = parts[0].clone()
        for r in range(1, self.world):
            acc = acc + parts[r]
        return acc

    def gather_rows(self, local, offsets, width):
        """All ranks receive the full row-major vector from the row slabs."""
        import torch
        import torch.distributed as dist
        if self.world == 1:
            return local.clone()
        rows = [offsets[r + 1] - offsets[r] for r in range(self.world)]
        mx = max(rows)
        buf = torch.zeros(mx * width, dtype=local.dtype, device=local.device)
        buf[:local.numel()] = local
        allb = torch.empty(self.world * mx * width, dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(allb, buf)
        return torch.cat([allb[r * mx * width:r * mx * width + rows[r] * width]
                          for r in range(self.world)])

    def halo(self, local, width, lo_needed, hi_needed):
        """(row below the slab from rank-1, row above from rank+1) as requested."""
        import torch
        import torch.distributed as dist
        below = above = None
        ops = []
        empty = torch.empty(0, dtype=local.dtype, device=local.device)
        nrows = local.numel() // width if width else 0
        # send my first row down / last row up when the neighbour asks
        send_down = local[:width] if nrows else empty
        send_up = local[(nrows - 1) * width:] if nrows else empty
        if lo_needed[self.rank]:
            below = torch.empty(width, dtype=local.dtype, device=local.device)
            ops.append(dist.P2POp(dist.irecv, below, self.rank - 1))
        if hi_needed[self.rank]:
            above = torch.empty(width, dtype=local.dtype, device=local.device)
            ops.append(dist.P2POp(dist.irecv, above, self.rank + 1))
        if self.rank + 1 < self.world and lo_needed[self.rank + 1]:
            ops.append(dist.P2POp(dist.isend, send_up.contiguous(), self.rank + 1))
        if self.rank > 0 and hi_needed[self.rank - 1]:
            ops.append(dist.P2POp(dist.isend, send_down.contiguous(), self.rank - 1))
        if ops:
            for q in dist.batch_isend_irecv(ops):
                q.wait()
        return below, above


# --------------------------------------------------------------------- levels
class SlabLevel:
    """Rank-local piece of one level operator plus its all-to-all plumbing."""

    def __init__(self, ctx: DistContext, problem: Problem, fine, dims, row_offsets, steps, m):
        self.ctx, self.bk = ctx, ctx.backend
        self.d1, self.d2 = dims
        self.rows = list(row_offsets)
        self.cols = split_ranges(self.d1, ctx.world)
        r, P = ctx.rank, ctx.world
        self.r0, self.r1 = self.rows[r], self.rows[r + 1]
        self.c0, self.c1 = self.cols[r], self.cols[r + 1]
        self.nr, self.nc = self.r1 - self.r0, self.c1 - self.c0
        self.h, diag = self.bk.slab(problem, fine, dims, steps, m, (self.r0, self.r1), (self.c0, self.c1))
        if np.any(~(diag > 0.0)):
            raise ValueError("operator diagonal must be strictly positive")
        self.dinv = self.bk.from_host(1.0 / diag)
        z = self.bk.zeros
        self.xTl = z(self.d1 * self.nr)      # my rows, transposed: [d1][nr]
        self.recv = z(self.nc * self.d2)     # chunks from every rank
        self.xT = z(self.nc * self.d2)       # my columns: [nc][d2]
        self.QT = z(self.nc * self.d2)
        self.send2 = z(self.nc * self.d2)
        self.recv2 = z(self.d1 * self.nr)    # [d1][nr]
        self.Q = z(self.nr * self.d1)        # my rows: [nr][d1]
        self.split_send = [(self.cols[d + 1] - self.cols[d]) * self.nr for d in range(P)]
        self.split_recv = [self.nc * (self.rows[s + 1] - self.rows[s]) for s in range(P)]
        self.split_send2 = [self.nc * (self.rows[d + 1] - self.rows[d]) for d in range(P)]
        self.split_recv2 = [(self.cols[s + 1] - self.cols[s]) * self.nr for s in range(P)]

    @property
    def local_size(self):
        return self.nr * self.d1

    def run(self, x, out, sign=1.0, epi=EPI_STORE, b=None, dinv=None, omega=0.0, src=None, src_scale=0.0):
        """out = epilogue(A~ x) on my rows (structured.cpp:125-148, distributed)."""
        bk = self.bk
        bk.transpose(x, self.xTl, self.nr, self.d1)                    # [nr][d1] -> [d1][nr]
        self.ctx.all_to_all(self.recv, self.xTl, self.split_recv, self.split_send)
        bk.permute(self.recv, self.xT, self.nc, self.d2, self.rows, 0)  # -> [nc][d2]
        bk.ypass(self.h, self.xT, self.QT, sign)
        bk.permute(self.QT, self.send2, self.nc, self.d2, self.rows, 1)
        self.ctx.all_to_all(self.recv2, self.send2, self.split_recv2, self.split_send2)
        bk.transpose(self.recv2, self.Q, self.d1, self.nr)             # [d1][nr] -> [nr][d1]
        bk.xpass(self.h, x, self.Q, out, sign, epi, b, dinv, omega, src, src_scale)


class DistHierarchy:
    """Geometric V-cycle (multigrid.cpp:318-394) over y-slab levels, with the
    coarse tail replicated on every rank."""

    def __init__(self, ctx, problem: Problem, n1, n2, steps, m, omega, coarse=COARSE_SWEEPS,
                 coarse_sweeps=3, agglomerate=65536, ratio0=None, fine_level=None):
        self.ctx, self.bk = ctx, ctx.backend
        self.omega, self.coarse, self.sweeps = omega, coarse, coarse_sweeps
        self.fine_level = fine_level or SlabLevel(ctx, problem, (n1, n2), (n1, n2),
                                                  split_ranges(n2, ctx.world), steps, m)
        if ratio0 is None:
            from . import StructuredFdeOperator
            ratio0 = _anisotropy_host(problem, n1, n2, steps, m)
        self.dims = plan_level_dims(n1, n2, ratio0, problem.alpha, problem.beta)
        L = len(self.dims)
        # slab levels: while big enough and every rank keeps >= 2 rows
        self.levels = [self.fine_level]
        offsets = self.fine_level.rows
        ls = 1
        while ls < L:
            d1, d2 = self.dims[ls]
            pd1, pd2 = self.dims[ls - 1]
            nxt = induced_coarse_rows(offsets, pd2, d2 < pd2)
            if d1 * d2 <= agglomerate or min(nxt[r + 1] - nxt[r] for r in range(ctx.world)) < 2:
                break
            self.levels.append(SlabLevel(ctx, problem, (n1, n2), (d1, d2), nxt, steps, m))
            offsets = nxt
            ls += 1
        self.n_slab = ls
        self.tail = (self.bk.coarse_vcycle_factory(problem, (n1, n2), self.dims[ls:], steps, m, omega,
                                                   coarse, coarse_sweeps) if ls < L else None)
        # transfers between consecutive levels
        self.xfer = []
        for l in range(L - 1):
            (a1, a2), (b1, b2) = self.dims[l], self.dims[l + 1]
            self.xfer.append((a1, a2, b1 < a1, b2 < a2))
        z = self.bk.zeros
        self.r = [z(lv.local_size) for lv in self.levels]
        self.bc = [None] + [z(lv.local_size) for lv in self.levels[1:]]
        self.xc = [None] + [z(lv.local_size) for lv in self.levels[1:]]
        last = self.levels[-1]
        self.tail_rows = None
        if self.tail is not None:
            # coarse rows the last slab level's ranks hand to the replicated tail
            (a1, a2, cx, cy) = self.xfer[self.n_slab - 1]
            self.tail_rows = induced_coarse_rows(last.rows, a2, cy)
            k1 = self.dims[self.n_slab][0]
            nrt = self.tail_rows[ctx.rank + 1] - self.tail_rows[ctx.rank]
            self.tail_b = z(nrt * k1)

    def vcycle(self, b, x, zero_guess=True):
        self._cycle(0, b, x, zero_guess)

    def _sweep(self, l, b, x):
        lv = self.levels[l]
        lv.run(x, x, 1.0, EPI_JACOBI, b=b, dinv=lv.dinv, omega=self.omega)

    def _cycle(self, l, b, x, zero):
        lv, bk = self.levels[l], self.bk
        n = lv.local_size
        last_slab = l + 1 == self.n_slab
        if last_slab and self.tail is None:  # coarsest level is a slab level
            if self.coarse == COARSE_SWEEPS:
                if zero:
                    bk.vec(0, n, self.omega, lv.dinv, b, x)
                else:
                    self._sweep(l, b, x)
                for _ in range(1, self.sweeps):
                    self._sweep(l, b, x)
            elif self.coarse == COARSE_LU:
                raise NotImplementedError("LU coarsest on a slab level: raise `agglomerate`")
            return
        if zero:
            bk.vec(0, n, self.omega, lv.dinv, b, x)  # x = omega dinv b (multigrid.cpp:355-356)
        else:
            self._sweep(l, b, x)
        lv.run(x, self.r[l], 1.0, EPI_RESID, b=b)     # r = b - A x
        a1, a2, cx, cy = self.xfer[l]
        if last_slab:
            # restrict my share of the coarse rows, then replicate the tail
            lo, hi = self.tail_rows[self.ctx.rank], self.tail_rows[self.ctx.rank + 1]
            self._restrict(l, self.r[l], self.tail_b, lo, hi)
            b_full = self.ctx.gather_rows(self.tail_b, self.tail_rows, self.dims[l + 1][0])
            xc_full = self.tail(b_full)
            self._prolong_add_from_full(l, xc_full, x)
        else:
            nxt = self.levels[l + 1]
            self._restrict(l, self.r[l], self.bc[l + 1], nxt.r0, nxt.r1)
            self._cycle(l + 1, self.bc[l + 1], self.xc[l + 1], True)
            self._prolong_add(l, self.xc[l + 1], x, nxt)
        self._sweep(l, b, x)                          # post-smooth

    def _with_halo(self, lv_rows, rank_lo, local, width, need_lo, need_hi):
        import torch
        below, above = self.ctx.halo(local, width, need_lo, need_hi)
        parts = ([below] if below is not None else []) + [local] + ([above] if above is not None else [])
        buf = torch.cat(parts) if len(parts) > 1 else local
        return buf, rank_lo - (1 if below is not None else 0)

    def _restrict(self, l, r_local, out, c_lo, c_hi):
        a1, a2, cx, cy = self.xfer[l]
        lv = self.levels[l]
        P = self.ctx.world
        if not cy:
            self.bk.transfer_rows(a1, a2, cx, cy, 1, 0, r_local, lv.r0, out, c_lo, c_hi - c_lo)
            return
        par = (a2 + 1) % 2
        rows = lv.rows
        coarse = induced_coarse_rows(rows, a2, True)

        def need(rk):
            lo, hi = coarse[rk], coarse[rk + 1]
            if hi <= lo:
                return False, False
            f_lo, f_hi = 2 * lo + 1 - par - 1, 2 * (hi - 1) + 1 - par + 1
            return (f_lo < rows[rk] and f_lo >= 0), (f_hi >= rows[rk + 1] and f_hi < a2)
        nl = [need(rk)[0] for rk in range(P)]
        nh = [need(rk)[1] for rk in range(P)]
        buf, lo = self._with_halo(rows, lv.r0, r_local, a1, nl, nh)
        self.bk.transfer_rows(a1, a2, cx, cy, 1, 0, buf, lo, out, c_lo, c_hi - c_lo)

    def _prolong_add(self, l, xc_local, x, nxt):
        a1, a2, cx, cy = self.xfer[l]
        lv = self.levels[l]
        P = self.ctx.world
        k1 = self.dims[l + 1][0]
        if not cy:
            self.bk.transfer_rows(a1, a2, cx, cy, 0, 1, xc_local, nxt.r0, x, lv.r0, lv.nr)
            return
        par = (a2 + 1) % 2
        crow = nxt.rows

        def need(rk):
            f0, f1 = lv.rows[rk], lv.rows[rk + 1]
            if f1 <= f0:
                return False, False
            t0, t1 = f0 - 1 + par, (f1 - 1) - 1 + par
            lo = t0 // 2 if t0 % 2 == 0 else (t0 - 1) // 2
            hi = t1 // 2 if t1 % 2 == 0 else (t1 + 1) // 2
            k2 = self.dims[l + 1][1]
            return (0 <= lo < crow[rk]), (crow[rk + 1] <= hi < k2)
        nl = [need(rk)[0] for rk in range(P)]
        nh = [need(rk)[1] for rk in range(P)]
        buf, lo = self._with_halo(crow, nxt.r0, xc_local, k1, nl, nh)
        self.bk.transfer_rows(a1, a2, cx, cy, 0, 1, buf, lo, x, lv.r0, lv.nr)

    def _prolong_add_from_full(self, l, xc_full, x):
        a1, a2, cx, cy = self.xfer[l]
        lv = self.levels[l]
        self.bk.transfer_rows(a1, a2, cx, cy, 0, 1, xc_full, 0, x, lv.r0, lv.nr)


def _anisotropy_host(problem: Problem, n1, n2, steps, m):
    """anisotropy_ratio of the fine step operator (multigrid.cpp:116-128),
    evaluated through a host-side assembly of the coefficient means."""
    from . import StructuredFdeOperator
    op = StructuredFdeOperator.assemble(problem, n1, n2, steps, m)
    return op.anisotropy_ratio(problem.alpha, problem.beta)


# --------------------------------------------------------------------- Krylov
class DistGmres:
    """gmres (krylov.cpp:34-166) on slab vectors; identical control flow to the
    single-GPU KrylovWorkspace::gmres, including the reuse of bit-identical
    M^-1 (b - A x) evaluations."""

    def __init__(self, ctx, level: SlabLevel, precond: DistHierarchy | None, restart):
        self.ctx, self.bk, self.A, self.M = ctx, ctx.backend, level, precond
        n = level.local_size
        z = self.bk.zeros
        self.n = n
        self.v = [z(n) for _ in range(restart + 1)]
        self.t, self.r, self.zv, self.w, self.trial = z(n), z(n), z(n), z(n), z(n)
        self.slot = z(1)

    def _gdot(self, x, y):
        self.bk.dot(x, y, self.slot)
        return self.ctx.ordered_sum(self.slot)

    def _pc(self, r, z):
        if self.M is None:
            z.copy_(r)
        else:
            self.M.vcycle(r, z, True)

    def solve(self, b, x, tol, restart, max_outer):
        bk, A, n = self.bk, self.A, self.n
        x.zero_()
        self._pc(b, self.zv)
        norm_b = math.sqrt(float(self._gdot(self.zv, self.zv)))
        hist, its = [], 0
        if norm_b == 0.0:
            return 0, True, [0.0]
        ld = restart + 1
        h = np.zeros(ld * restart)
        cs, sn = np.zeros(restart), np.zeros(restart)
        state = {"xver": 0, "zver": 0, "zbeta": norm_b}
        xbuf = [x, self.trial]

        def residual_z():
            if state["zver"] == state["xver"]:
                return state["zbeta"]
            A.run(xbuf[0], self.r, 1.0, EPI_RESID, b=b)
            self._pc(self.r, self.zv)
            state["zbeta"] = math.sqrt(float(self._gdot(self.zv, self.zv)))
            state["zver"] = state["xver"]
            return state["zbeta"]

        def lincomb(dst, src, y):
            if dst is not src:
                dst.copy_(src)
            for k in range(len(y)):
                bk.vec(1, n, float(y[k]), self.v[k], None, dst)

        converged = False
        for outer in range(max_outer):
            if converged:
                break
            beta = residual_z()
            rel0 = beta / norm_b
            if outer == 0:
                hist.append(rel0)
            if rel0 <= tol:
                converged = True
                break
            g = np.zeros(ld)
            g[0] = beta
            bk.vec(3, n, 1.0 / beta, self.zv, None, self.v[0])
            spanned, done = 0, False
            for i in range(restart):
                if done:
                    break
                A.run(self.v[i], self.t)
                self._pc(self.t, self.w)
                norm0 = math.sqrt(float(self._gdot(self.w, self.w)))
                for k in range(i + 1):  # modified Gram-Schmidt
                    hk = self._gdot(self.v[k], self.w)
                    bk.axpy_dev(hk.reshape(1), -1.0, self.v[k], self.w)
                    h[i * ld + k] = float(hk)
                nrmw = math.sqrt(float(self._gdot(self.w, self.w)))
                if nrmw < 1e-8 * norm0:
                    for k in range(i + 1):
                        c = self._gdot(self.v[k], self.w)
                        bk.axpy_dev(c.reshape(1), -1.0, self.v[k], self.w)
                        h[i * ld + k] += float(c)
                    nrmw = math.sqrt(float(self._gdot(self.w, self.w)))
                hip = nrmw
                happy = hip <= 1e-14 * (norm0 if norm0 > 0.0 else 1.0)
                for k in range(i):
                    tmp = cs[k] * h[i * ld + k] + sn[k] * h[i * ld + k + 1]
                    h[i * ld + k + 1] = -sn[k] * h[i * ld + k] + cs[k] * h[i * ld + k + 1]
                    h[i * ld + k] = tmp
                denom = math.hypot(h[i * ld + i], hip)
                cs[i] = h[i * ld + i] / denom if denom > 0.0 else 1.0
                sn[i] = hip / denom if denom > 0.0 else 0.0
                h[i * ld + i] = denom
                g[i + 1] = -sn[i] * g[i]
                g[i] = cs[i] * g[i]
                its += 1
                spanned = i + 1
                est = abs(g[i + 1]) / norm_b
                hist.append(est)
                if not happy:
                    bk.vec(3, n, 1.0 / hip, self.w, None, self.v[i + 1])
                if est <= tol or happy:
                    y = _back_substitute(h, ld, g, spanned)
                    lincomb(xbuf[1], xbuf[0], y)
                    xbuf.reverse()
                    state["xver"] += 1
                    if residual_z() / norm_b <= tol:
                        converged, done = True, True
                    elif happy:
                        done = True
                    else:
                        xbuf.reverse()
                        state["xver"] += 1
            if not converged and not done:
                y = _back_substitute(h, ld, g, spanned)
                lincomb(xbuf[0], xbuf[0], y)
                state["xver"] += 1
        final_rel = residual_z() / norm_b
        if final_rel <= tol:
            converged = True
        if hist:
            hist[-1] = final_rel
        else:
            hist.append(final_rel)
        if xbuf[0] is not x:
            x.copy_(xbuf[0])
        return its, converged, hist


def _back_substitute(h, ld, g, k):  # krylov.cpp:19-30
    y = np.zeros(k)
    for i in range(k - 1, -1, -1):
        v = g[i]
        for j in range(i + 1, k):
            v -= h[j * ld + i] * y[j]
        y[i] = v / h[i * ld + i] if h[i * ld + i] != 0.0 else 0.0
    return y


# --------------------------------------------------------------------- march
class DistMarch:
    """time_march (driver.cpp:10-69) on y-slabs: u^m rows stay on their rank."""

    def __init__(self, ctx, problem: Problem, n1, n2, steps, tol=1e-8, restart=20, max_outer=100,
                 omega=0.7, coarse=COARSE_SWEEPS, coarse_sweeps=3, agglomerate=65536, precond=True,
                 ratio0=None):
        self.ctx, self.bk = ctx, ctx.backend
        if getattr(problem, "time_dependent_coeffs", False):
            # the operator and the hierarchy are built once (at m = 1): a
            # time-dependent problem needs the t^{m-1} operator for the rhs and
            # the step-m operator and V-cycle for the solve (driver.cpp:37-51)
            raise NotImplementedError("the y-slab march supports time-independent coefficients "
                                      "only; use the single-GPU March for time-dependent problems")
        self.problem, self.n1, self.n2, self.steps = problem, n1, n2, steps
        self.tol, self.restart, self.max_outer = tol, restart, max_outer
        rows = split_ranges(n2, ctx.world)
        self.level = SlabLevel(ctx, problem, (n1, n2), (n1, n2), rows, steps, 1)
        self.M = (DistHierarchy(ctx, problem, n1, n2, steps, 1, omega, coarse, coarse_sweeps,
                                agglomerate, ratio0=ratio0, fine_level=self.level)
                  if precond else None)
        self.solver = DistGmres(ctx, self.level, self.M, restart)
        lv = self.level
        u0 = problem.sample_initial(n1, n2, steps)[lv.r0 * n1:lv.r1 * n1]
        self.u = self.bk.from_host(u0)
        self.b = self.bk.zeros(lv.local_size)
        self.x = self.bk.zeros(lv.local_size)
        hx = (problem.bx - problem.ax) / (n1 + 1)
        self.scale = 2.0 * math.pow(hx, problem.alpha)  # problem.cpp:82
        self.m = 0

    def step(self, source_local=None):
        """source_local: this rank's rows of v(., t^{m-1/2}) (sampled if None)."""
        self.m += 1
        lv = self.level
        if source_local is None:
            v = self.problem.sample_source(self.n1, self.n2, self.steps, self.m)
            source_local = self.bk.from_host(v[lv.r0 * self.n1:lv.r1 * self.n1])
        lv.run(self.u, self.b, -1.0, EPI_RHS, src=source_local, src_scale=self.scale)
        its, conv, hist = self.solver.solve(self.b, self.x, self.tol, self.restart, self.max_outer)
        self.u, self.x = self.x, self.u
        return its, hist[-1]

    def solution_local(self):
        return self.bk.to_host(self.u)
