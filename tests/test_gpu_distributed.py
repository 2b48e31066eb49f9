"""The y-slab path's GPU backend (libfde_b200 slab kernels, block permutes,
row-window transfers) on one rank: it must reproduce the single-GPU solver."""
from pathlib import Path

import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from golden_util import compare_summary
from paper_1706_06844_b200 import distributed as D

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def ctx1():
    import torch
    return D.DistContext(0, 1, D.GpuBackend(torch.device("cuda:0")))


@pytest.mark.parametrize("cfg,n1,n2", [(2, 255, 255), (4, 511, 300), (3, 127, 64)])
def test_slab_apply_matches_operator(cuda, cfg, n1, n2):
    import torch
    ctx = ctx1()
    p = fde.Problem.preset_config(cfg, steps=4)
    lv = D.SlabLevel(ctx, p, (n1, n2), (n1, n2), [0, n2], 4, 1)
    op = fde.StructuredFdeOperator.assemble(p, n1, n2, 4, 1)
    x = torch.rand(n1 * n2, dtype=torch.float64, device="cuda")
    out = torch.empty_like(x)
    for sign in (1.0, -1.0):
        lv.run(x, out, sign)
        ref = op.apply(x) if sign > 0 else op.apply_rhs(x)
        assert float(torch.linalg.norm(out - ref) / torch.linalg.norm(ref)) <= 1e-14


@pytest.mark.parametrize("agg", [4096, 65536])
def test_dist_vcycle_matches_hierarchy(cuda, agg):
    import torch
    ctx = ctx1()
    p = fde.Problem.preset_config(4, steps=8)
    n = 511
    h = D.DistHierarchy(ctx, p, n, n, 8, 1, 0.7, fde.COARSE_SWEEPS, 3, agglomerate=agg)
    ref = fde.MgHierarchy.build_geometric(p, n, n, 8, 1, 0.7, fde.COARSE_SWEEPS, 3)
    assert h.dims == ref.dims()
    b = torch.rand(n * n, dtype=torch.float64, device="cuda")
    x = torch.zeros_like(b)
    h.vcycle(b, x, True)
    xr = ref.vcycle(b)
    assert float(torch.linalg.norm(x - xr) / torch.linalg.norm(xr)) <= 1e-13


def test_dist_march_cfg2_vs_golden(cuda):
    gd = np.load(GOLD / "cfg2_4steps.npz")
    ctx = ctx1()
    p = fde.Problem.preset_config(2, steps=4)
    m = D.DistMarch(ctx, p, 255, 255, 4, tol=1e-8, restart=20, omega=0.7, agglomerate=4096)
    its, us = [], []
    for _ in range(4):
        it, _ = m.step()
        its.append(it)
        us.append(m.solution_local())
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(np.array(us), gd, 1e-10) <= 1e-10
