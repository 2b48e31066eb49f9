"""Multi-rank (gloo, CPU) tests of the y-slab path:
partitioning, all-to-all transposes, halo exchange, coarse agglomeration and
distributed GMRES, with local compute emulated from the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracles import oracle, spec

import paper_1706_06844_b200 as fde
from paper_1706_06844_b200 import distributed as D


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


def gather_full(ctx, local, offsets, width):
    return ctx.gather_rows(local, offsets, width).numpy()


def _worker(rank, world, port, task, resq):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from dist_emulation import EmuBackend
        orc = oracle()
        cfg, n1, n2, steps = task["cfg"], task["n1"], task["n2"], task["steps"]
        s = spec(cfg, n1=n1, n2=n2, steps=steps)
        problem = fde.Problem.preset_config(cfg, steps=steps)
        ctx = D.DistContext(rank, world, EmuBackend(orc, cfg))
        rows = D.split_ranges(n2, world)
        res = {}
        if task["what"] == "apply":
            lv = D.SlabLevel(ctx, problem, (n1, n2), (n1, n2), rows, steps, 1)
            x = np.random.default_rng(1).uniform(-1, 1, n1 * n2)
            xl = torch.tensor(x[lv.r0 * n1:lv.r1 * n1])
            for sign, epi in ((1.0, D.EPI_STORE), (-1.0, D.EPI_STORE), (1.0, D.EPI_RESID)):
                out = torch.zeros_like(xl)
                b = torch.ones_like(xl)
                lv.run(xl, out, sign, epi, b=b)
                full = gather_full(ctx, out, rows, n1)
                ref = orc.apply(s, x, int(sign))
                if epi == D.EPI_RESID:
                    ref = 1.0 - ref
                res[(sign, epi)] = rel(full, ref)
        elif task["what"] == "vcycle":
            dims, r0 = orc.plan(s)
            h = D.DistHierarchy(ctx, problem, n1, n2, steps, 1, 0.7, task.get("coarse", 1), 3,
                                agglomerate=task["agg"], ratio0=r0)
            res["n_slab"] = h.n_slab
            res["dims"] = h.dims == dims
            b = np.random.default_rng(2).uniform(-1, 1, n1 * n2)
            lv = h.levels[0]
            x = torch.zeros(lv.local_size, dtype=torch.float64)
            h.vcycle(torch.tensor(b[lv.r0 * n1:lv.r1 * n1]), x, True)
            full = gather_full(ctx, x, rows, n1)
            res["err"] = rel(full, orc.vcycle(spec(cfg, n1=n1, n2=n2, steps=steps, coarse=task.get("coarse", 1)), b))
        elif task["what"] == "march":
            _, r0 = orc.plan(s)
            m = D.DistMarch.__new__(D.DistMarch)
            # DistMarch with the oracle's anisotropy ratio (the GPU path computes it itself)
            D.DistMarch.__init__(m, ctx, problem, n1, n2, steps, tol=1e-8, restart=20, max_outer=100,
                                 omega=0.7, agglomerate=task["agg"], ratio0=r0)
            its = []
            sols = []
            for _ in range(steps):
                it, _res = m.step()
                its.append(it)
                sols.append(gather_full(ctx, m.u, rows, n1))
            ro = orc.march(s, record=True)
            res["its"] = its
            res["ref_its"] = ro["its"].tolist()
            res["err"] = max(rel(sols[k], ro["u_steps"][k]) for k in range(steps))
        if rank == 0:
            resq.put(res)
    finally:
        dist.destroy_process_group()


def run_dist(world, task):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, task, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue
    import time
    t0 = time.time()
    while True:
        try:
            res = q.get(timeout=1.0)
            break
        except queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs) or time.time() - t0 > 300:
                for p in procs:
                    p.kill()
                raise AssertionError("distributed worker failed")
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("world", [2, 3])
def test_distributed_apply_matches_oracle(world):
    res = run_dist(world, dict(what="apply", cfg=2, n1=40, n2=33, steps=2))
    for k, v in res.items():
        assert v <= 1e-13, (k, v)


@pytest.mark.parametrize("world,agg,coarse", [(2, 60, 1), (3, 60, 1), (2, 1000, 1), (2, 60, 0)])
def test_distributed_vcycle_matches_oracle(world, agg, coarse):
    res = run_dist(world, dict(what="vcycle", cfg=2, n1=40, n2=41, steps=2, agg=agg, coarse=coarse))
    assert res["dims"]
    assert res["n_slab"] >= 1
    assert res["err"] <= 1e-12, res


def test_distributed_vcycle_semicoarsened():
    """cfg4 orders/coefficients on a wide grid: x-only coarsening first (no halo)."""
    res = run_dist(2, dict(what="vcycle", cfg=4, n1=63, n2=31, steps=2, agg=100))
    assert res["n_slab"] >= 2
    assert res["err"] <= 1e-12, res


def test_distributed_march_matches_oracle():
    res = run_dist(2, dict(what="march", cfg=2, n1=40, n2=33, steps=2, agg=100))
    assert res["its"] == res["ref_its"], res
    assert res["err"] <= 1e-10, res


def test_partition_helpers():
    assert D.split_ranges(10, 3) == [0, 3, 6, 10]
    # coarse rows follow their centre fine rows: d2 = 9 (par 0): centres 1, 3, 5, 7
    assert D.induced_coarse_rows([0, 4, 9], 9, True) == [0, 2, 4]
    assert D.induced_coarse_rows([0, 5, 10], 10, True) == [0, 3, 5]  # par 1: centres 0,2,4,6,8
    assert D.induced_coarse_rows([0, 4, 9], 9, False) == [0, 4, 9]


def test_cxx_partition_matches_python():
    """The C++ march's row partition (csrc/dist.cu) equals the Python
    emulation's for every level of random plans (host only)."""
    import ctypes
    import paper_1706_06844_b200 as fde
    from paper_1706_06844_b200 import distributed as D
    lib = fde.load_library()
    rng = np.random.default_rng(0)
    for _ in range(300):
        P = int(rng.integers(1, 9))
        d2 = int(rng.integers(2 * P, 5000))
        arr = (ctypes.c_size_t * (P + 1))()
        assert lib.fde_dist_split_rows(d2, P, arr) == 0
        rows = [int(v) for v in arr]
        assert rows == D.split_ranges(d2, P)
        while d2 >= 4:
            for cy in (1, 0):
                out = (ctypes.c_size_t * (P + 1))()
                assert lib.fde_dist_induced_rows(arr, P, d2, cy, out) == 0
                assert [int(v) for v in out] == D.induced_coarse_rows(rows, d2, bool(cy)), (rows, d2, cy)
            rows = D.induced_coarse_rows(rows, d2, True)
            arr = (ctypes.c_size_t * (P + 1))(*rows)
            d2 = D.coarse_size(d2)
