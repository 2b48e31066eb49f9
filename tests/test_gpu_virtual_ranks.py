"""The multi-GPU host code (csrc/dist.cu) on VIRTUAL ranks of one GPU.

P = 2 / 3 / 4 / 8 logical ranks run the same C++ solver the NCCL build runs
(slab levels, fde_slab-style column / row passes on rank-local pieces with
r0, c0 > 0, block permutes with P > 1, row-window transfers with halo rows,
the replicated coarse tail, rank-ordered inner products), each on its own
host thread; collectives are ordered device copies.  They must reproduce the
single-GPU solver: identical GMRES iteration counts, solutions to rounding
(per-line FFT results differ in the last bits when a line's 16-byte alignment
differs between the two layouts, and rank-ordered dot products sum in another
order, so the comparison is <= 1e-12, not bit-for-bit).  The NCCL transport
itself is covered at world size 1."""
from pathlib import Path

import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from golden_util import compare_summary

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def mg_cfg(**kw):
    d = dict(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7, cycles=1,
             coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
    d.update(kw)
    return fde.DriverConfig(**d)


@pytest.mark.parametrize("cfg,n1,n2,P", [(4, 511, 511, 2), (4, 511, 300, 3), (2, 255, 255, 4),
                                          (4, 2047, 2047, 8), (3, 127, 64, 5)])
def test_virtual_apply_matches_operator(cuda, cfg, n1, n2, P):
    import torch
    p = fde.Problem.preset_config(cfg, steps=4)
    op = fde.StructuredFdeOperator.assemble(p, n1, n2, 4, 1)
    x = np.random.default_rng(n1 + P).uniform(-1, 1, n1 * n2)
    ref = op.apply(torch.tensor(x, device="cuda")).cpu().numpy()
    y = fde.vdist_run(p, n1, n2, 4, mg_cfg(), P, "apply", inp=x)
    assert rel(y, ref) <= 1e-13


@pytest.mark.parametrize("n,P,agg", [(511, 2, 65536), (511, 4, 4096), (2047, 2, 65536),
                                     (2047, 4, 65536), (2047, 8, 65536), (1023, 3, 16384)])
def test_virtual_vcycle_matches_hierarchy(cuda, n, P, agg):
    """cfg4 V-cycle (incl. n = 2047, the BASELINE grid): slab levels with halo
    exchanges, semicoarsened levels, replicated tail."""
    import torch
    p = fde.Problem.preset_config(4, steps=8)
    ref_h = fde.MgHierarchy.build_geometric(p, n, n, 8, 1, 0.7, fde.COARSE_SWEEPS, 3)
    b = np.random.default_rng(n).uniform(-1, 1, n * n)
    ref = ref_h.vcycle(torch.tensor(b, device="cuda")).cpu().numpy()
    x = fde.vdist_run(p, n, n, 8, mg_cfg(), P, "vcycle", inp=b, agglomerate=agg)
    assert rel(x, ref) <= 1e-12


@pytest.mark.parametrize("P", [2, 4, 8])
def test_virtual_march_cfg4_n511_matches_single_gpu(cuda, P):
    """cfg4 at n = 511, all 8 steps: the distributed march against the
    single-GPU march (identical iteration counts every step)."""
    n, steps = 511, 8
    p = fde.Problem.preset_config(4, steps=steps)
    m = fde.March(p, n, n, steps, mg_cfg())
    its_ref = [m.step()[0] for _ in range(steps)]
    u_ref = m.solution()
    u, its, res, ncoll = fde.vdist_run(p, n, n, steps, mg_cfg(), P, "march", nrun=steps)
    assert its == its_ref
    assert max(res) <= 1e-8
    assert rel(u, u_ref) <= 1e-10
    assert ncoll > 0


def test_virtual_march_cfg2_vs_reference_golden(cuda):
    """cfg2 (n = 255), 4 steps on 3 uneven virtual ranks against the golden the
    unmodified reference produced."""
    gd = np.load(GOLD / "cfg2_4steps.npz")
    p = fde.Problem.preset_config(2, steps=4)
    us, its_all = [], []
    for k in range(1, 5):
        u, its, _, _ = fde.vdist_run(p, 255, 255, 4, mg_cfg(), 3, "march", nrun=k, agglomerate=4096)
        us.append(u)
        its_all = its
    np.testing.assert_array_equal(its_all, gd["its"])
    assert compare_summary(np.array(us), gd, 1e-10) <= 1e-10


def test_virtual_march_unpreconditioned_and_errors(cuda):
    p = fde.Problem.preset_config(1, steps=4)
    cfg = mg_cfg(precond=fde.PRECOND_NONE, max_outer=200)
    m = fde.March(p, 63, 63, 4, cfg)
    its_ref = [m.step()[0] for _ in range(2)]
    u, its, _, _ = fde.vdist_run(p, 63, 63, 4, cfg, 2, "march", nrun=2)
    assert its == its_ref and rel(u, m.solution()) <= 1e-10
    with pytest.raises(ValueError):  # more ranks than the grid can hold
        fde.vdist_run(p, 63, 63, 4, cfg, 40, "march", nrun=1)
    with pytest.raises(ValueError):  # LU coarsest on a slab level
        fde.vdist_run(p, 63, 63, 4, mg_cfg(coarse=fde.COARSE_LU), 2, "march", nrun=1, agglomerate=1)
    ex2 = fde.Problem.example(2, 1.5, 1.5)
    with pytest.raises(ValueError):  # time-dependent coefficients
        fde.vdist_run(ex2, 31, 31, 4, mg_cfg(), 2, "march", nrun=1)


def test_nccl_transport_world1(cuda):
    """The NCCL build of the same march at world size 1 (libnccl opened at run
    time, send/recv to self): cfg2, 4 steps against the reference golden."""
    import torch
    gd = np.load(GOLD / "cfg2_4steps.npz")
    p = fde.Problem.preset_config(2, steps=4)
    m = fde.SlabMarch(p, 255, 255, 4, mg_cfg(), rank=0, world=1, agglomerate=4096)
    assert (m.r0, m.r1) == (0, 255)
    its, us = [], []
    for _ in range(4):
        its.append(m.step()[0])
        us.append(m.solution_local())
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(np.array(us), gd, 1e-10) <= 1e-10
    assert m.collectives() > 0
    x = torch.rand(255 * 255, dtype=torch.float64, device="cuda")
    y = torch.empty_like(x)
    m.apply(x, y)
    op = fde.StructuredFdeOperator.assemble(p, 255, 255, 4, 1)
    ref = op.apply(x)
    assert float(torch.linalg.norm(y - ref) / torch.linalg.norm(ref)) <= 1e-13
