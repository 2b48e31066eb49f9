"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle.

Bars (BASELINE north_star): FP64 operator/V-cycle results within 1e-12
relative l2 of the oracle; time-step solutions within 1e-10 relative l2 per
step with identical GMRES iteration counts.
"""
import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from oracles import spec, CONFIGS

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def to_dev(a):
    import torch
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def problem_for(cfg, **kw):
    return fde.Problem.preset_config(cfg, seed=kw.get("seed", 0), source_kind=kw.get("source_kind", -1),
                                     steps=kw.get("steps", 0))


@pytest.mark.parametrize("n1,n2", [(7, 5), (8, 8), (31, 33), (33, 31), (63, 63), (64, 65),
                                   (127, 1), (1, 15), (255, 255), (100, 257), (1023, 15),
                                   (513, 64), (2047, 3), (1025, 17), (17, 1025),
                                   (2048, 5), (5, 2048), (1531, 601), (601, 1531)])
@pytest.mark.parametrize("sign", [1, -1])
def test_operator_apply_matches_oracle(cuda, orc, n1, n2, sign):
    s = spec(2, n1=n1, n2=n2, steps=4)
    p = problem_for(2, steps=4)
    op = fde.StructuredFdeOperator.assemble(p, n1, n2, 4, 1)
    rng = np.random.default_rng(n1 * 7919 + n2)
    x = rng.uniform(-1, 1, n1 * n2)
    y = (op.apply(to_dev(x)) if sign > 0 else op.apply_rhs(to_dev(x))).cpu().numpy()
    yo = orc.apply(s, x, sign)
    assert rel(y, yo) <= 1e-13, rel(y, yo)
    np.testing.assert_array_equal(op.diagonal(), orc.diagonal(s))


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_operator_apply_presets(cuda, orc, cfg):
    n = {1: 63, 3: 255, 5: 511}[cfg]
    s = spec(cfg, n1=n, n2=n, steps=2)
    p = problem_for(cfg, steps=2)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 2, 1)
    x = np.random.default_rng(cfg).uniform(-1, 1, n * n)
    assert rel(op.apply(to_dev(x)).cpu().numpy(), orc.apply(s, x)) <= 1e-13


@pytest.mark.parametrize("cfg,n,coarse", [(1, 63, 1), (2, 255, 1), (4, 255, 1), (3, 127, 0),
                                          (3, 127, 1), (5, 255, 1), (1, 63, 2), (2, 63, 0)])
def test_vcycle_matches_oracle(cuda, orc, cfg, n, coarse):
    s = spec(cfg, n1=n, n2=n, steps=4, coarse=coarse)
    p = problem_for(cfg, steps=4)
    h = fde.MgHierarchy.build_geometric(p, n, n, 4, 1, 0.7, coarse, 3)
    assert h.dims() == orc.plan(s)[0]
    b = np.random.default_rng(n).uniform(-1, 1, n * n)
    x = h.vcycle(to_dev(b)).cpu().numpy()
    xo = orc.vcycle(s, b)
    assert rel(x, xo) <= 1e-12, rel(x, xo)
    x0 = np.random.default_rng(n + 1).uniform(-1, 1, n * n)  # nonzero initial guess path
    x2 = h.vcycle(to_dev(b), to_dev(x0), zero_guess=False).cpu().numpy()
    assert rel(x2, orc.vcycle(s, b, x0)) <= 1e-12


@pytest.mark.parametrize("n1,n2,cx,cy", [(63, 63, 1, 1), (64, 31, 1, 1), (30, 17, 1, 0),
                                         (17, 30, 0, 1), (2047, 7, 1, 1)])
def test_transfers_bitexact(cuda, orc, n1, n2, cx, cy):
    rng = np.random.default_rng(n1 + n2)
    k1 = (n1 - n1 % 2) // 2 if cx else n1
    k2 = (n2 - n2 % 2) // 2 if cy else n2
    f = rng.uniform(-1, 1, n1 * n2)
    c = rng.uniform(-1, 1, k1 * k2)
    for op, src, nout in ((0, c, n1 * n2), (1, f, k1 * k2), (2, f, k1 * k2)):
        import torch
        out = torch.zeros(nout, dtype=torch.float64, device="cuda")
        fde.transfer(n1, n2, cx, cy, op, to_dev(src), out)
        np.testing.assert_array_equal(out.cpu().numpy(), orc.transfer(n1, n2, cx, cy, op, src))


@pytest.mark.parametrize("cfg,n,precond", [(1, 63, 2), (2, 127, 2), (1, 63, 1), (1, 63, 0)])
def test_gmres_matches_oracle(cuda, orc, cfg, n, precond):
    s = spec(cfg, n1=n, n2=n, steps=4, precond=precond)
    p = problem_for(cfg, steps=4)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 4, 1)
    pc = fde.make_preconditioner(precond, p, n, n, 4, 1, op, 0.7, 1, fde.COARSE_SWEEPS, 3)
    b = orc.rhs(s, 1, orc.initial(s))
    r = fde.gmres(op, fde.SolverConfig(1e-8, 20, 100), to_dev(b), pc if precond else None)
    xo, it, conv, hist = orc.gmres(s, b)
    assert r.total_iterations == it
    assert r.converged == conv
    assert rel(r.solution.cpu().numpy(), xo) <= 1e-10
    assert len(r.residual_history) == len(hist)


def test_time_march_cfg1_full(cuda, orc):
    """cfg1 (n=63, 64 steps): every step within 1e-10, identical iterations."""
    s = spec(1)
    ro = orc.march(s, record=True)
    p = problem_for(1)
    cfg = fde.DriverConfig(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7,
                           cycles=1, coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
    m = fde.March(p, 63, 63, 64, cfg)
    for k in range(64):
        it, res = m.step()
        u = m.solution()
        assert it == ro["its"][k], (k, it, ro["its"][k])
        assert rel(u, ro["u_steps"][k]) <= 1e-10, (k, rel(u, ro["u_steps"][k]))


@pytest.mark.parametrize("cfg,n,coarse", [(1, 63, 1), (1, 63, 2), (2, 255, 1), (3, 127, 1),
                                          (3, 255, 2), (5, 255, 1), (4, 511, 1)])
def test_vcycle_tail_matches_level_kernels(cuda, orc, monkeypatch, cfg, n, coarse):
    """The one-launch coarse tail (csrc/tail.cu) against the per-level kernel
    sequence on the same hierarchy plan: same V-cycle to rounding (direct vs
    FFT Toeplitz sums), fewer launches, and both against the oracle."""
    import torch
    p = problem_for(cfg, steps=4)
    b = to_dev(np.random.default_rng(n + cfg).uniform(-1, 1, n * n))
    out = {}
    for tail in ("1", "0"):
        monkeypatch.setenv("FDE_MG_TAIL", tail)
        h = fde.MgHierarchy.build_geometric(p, n, n, 4, 1, 0.7, coarse, 3)
        h.vcycle(b)  # warm (graph-free path, per-call launches)
        torch.cuda.synchronize()
        k0 = fde.kernel_launches()
        x = h.vcycle(b).cpu().numpy()
        out[tail] = (x, fde.kernel_launches() - k0)
    assert rel(out["1"][0], out["0"][0]) <= 1e-13, rel(out["1"][0], out["0"][0])
    assert out["1"][1] < out["0"][1], (out["1"][1], out["0"][1])
    xo = orc.vcycle(spec(cfg, n1=n, n2=n, steps=4, coarse=coarse), b.cpu().numpy())
    assert rel(out["1"][0], xo) <= 1e-12
