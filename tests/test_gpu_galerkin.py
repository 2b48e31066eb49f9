"""The reference's oracle-size preconditioner variants on the GPU (SURVEY.md
8(f)4): `p2-exact` (P2ExactPrecond, proj/src/precond.cpp:90-101: exact solve
with the banded order-2 companion) and `mgm-galerkin` (MgmGalerkinPrecond,
precond.cpp:115-133: Galerkin R A P levels of the full operator over the
anisotropy plan), against the reference's own classes (oracle/_ref).

The reference factors P2 with Eigen's SparseLU; Eigen is absent from the
image, so oracle/_ref links the clean-room shim's dense LU in its place --
parity for `p2-exact` is pinned to that factorisation.
"""
import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from oracles import spec

pytestmark = pytest.mark.gpu

DEFAULTS = {1: (1.8, 1.6), 2: (1.8, 1.9), 3: (1.8, 1.9)}  # problem.cpp:262-265


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def to_dev(a):
    import torch
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def ex_spec(which, n, **kw):
    kw.setdefault("steps", n)
    kw.setdefault("tol", 1e-7)
    kw.setdefault("omega", 0.9)
    return spec(100 + which, n1=n, n2=n, **kw)


@pytest.mark.parametrize("which,n,kind,coarse", [
    (1, 16, fde.PRECOND_P2_EXACT, fde.COARSE_SWEEPS), (2, 31, fde.PRECOND_P2_EXACT, fde.COARSE_SWEEPS),
    (1, 16, fde.PRECOND_MGM_GALERKIN, fde.COARSE_SWEEPS),
    (3, 31, fde.PRECOND_MGM_GALERKIN, fde.COARSE_LU),
    (2, 33, fde.PRECOND_MGM_GALERKIN, fde.COARSE_NONE)])
def test_precond_apply_matches_reference(cuda, ref, which, n, kind, coarse):
    a, b = DEFAULTS[which]
    p = fde.Problem.example(which, a, b)
    s = ex_spec(which, n, precond=kind, coarse=coarse, cycles=1)
    op = fde.StructuredFdeOperator.assemble(p, n, n, n, 1)
    pc = fde.make_preconditioner(kind, p, n, n, n, 1, op, 0.9, 1, coarse, 3)
    r = np.random.default_rng(n + kind).uniform(-1, 1, n * n)
    z = pc.apply(to_dev(r)).cpu().numpy()
    zr = ref.precond(s, r)
    assert rel(z, zr) <= 1e-12, rel(z, zr)


@pytest.mark.parametrize("which,n,kind", [(1, 16, fde.PRECOND_P2_EXACT),
                                          (3, 32, fde.PRECOND_P2_EXACT),
                                          (1, 32, fde.PRECOND_MGM_GALERKIN),
                                          (2, 16, fde.PRECOND_MGM_GALERKIN)])
def test_time_march_matches_reference(cuda, ref, which, n, kind):
    """time_march with the variant: identical iteration counts, final solution
    within 1e-10 of the reference's own time_march (driver.cpp:10-69)."""
    a, b = DEFAULTS[which]
    p = fde.Problem.example(which, a, b)
    cfg = fde.DriverConfig(precond=kind, tol=1e-7, restart=20, max_outer=100, omega=0.9,
                           cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
    m = fde.March(p, n, n, n, cfg)
    its = [m.step()[0] for _ in range(n)]
    ro = ref.time_march(ex_spec(which, n, precond=kind))
    assert its == list(ro["its"]), (its, list(ro["its"]))
    assert rel(m.solution(), ro["u"]) <= 1e-10


def test_galerkin_size_limit(cuda):
    """precond.cpp:121-123: the Galerkin variant is limited to 128 x 128 grids."""
    a, b = DEFAULTS[1]
    p = fde.Problem.example(1, a, b)
    op = fde.StructuredFdeOperator.assemble(p, 129, 129, 129, 1)
    with pytest.raises(Exception, match="128"):
        fde.make_preconditioner(fde.PRECOND_MGM_GALERKIN, p, 129, 129, 129, 1, op, 0.9, 1,
                                fde.COARSE_SWEEPS, 3)
