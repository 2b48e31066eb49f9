"""GPU parity at BASELINE sizes: against the oracle where it finishes in
seconds (operator apply / V-cycle up to n=4095), against the reference's
golden trajectories (tests/golden, made from oracle/_ref) for the time
marches, and through size-independent identities elsewhere."""
from pathlib import Path

import numpy as np
import pytest

import paper_1706_06844_b200 as fde
from golden_util import compare_summary, sample_idx
from oracles import spec

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def dev(a):
    import torch
    return torch.tensor(np.ascontiguousarray(a), dtype=torch.float64, device="cuda")


def mg_cfg(**kw):
    c = dict(precond=fde.PRECOND_MGM, tol=1e-8, restart=20, max_outer=100, omega=0.7, cycles=1,
             coarse=fde.COARSE_SWEEPS, coarse_sweeps=3)
    c.update(kw)
    return fde.DriverConfig(**c)


def run_march(cfg_id, n, steps, dcfg, record=True, source_kind=-1):
    p = fde.Problem.preset_config(cfg_id, steps=steps, source_kind=source_kind)
    m = fde.March(p, n, n, steps, dcfg)
    its, us = [], []
    for _ in range(steps):
        it, _res = m.step()
        its.append(it)
        if record:
            us.append(m.solution())
    return np.array(its), np.array(us) if record else m.solution()


@pytest.mark.parametrize("cfg,n", [(4, 2047), (5, 2047), (5, 4095), (3, 1023)])
def test_apply_fullsize_vs_oracle(cuda, orc, cfg, n):
    s = spec(cfg, n1=n, n2=n, steps=8)
    p = fde.Problem.preset_config(cfg, steps=8)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 8, 1)
    x = np.random.default_rng(n).uniform(-1, 1, n * n)
    assert rel(op.apply(dev(x)).cpu().numpy(), orc.apply(s, x)) <= 1e-13
    assert rel(op.apply_rhs(dev(x)).cpu().numpy(), orc.apply(s, x, -1)) <= 1e-13


@pytest.mark.parametrize("cfg,n", [(4, 2047), (5, 2047), (3, 1023), (5, 4095)])
def test_vcycle_fullsize_vs_oracle(cuda, orc, cfg, n):
    s = spec(cfg, n1=n, n2=n, steps=8)
    p = fde.Problem.preset_config(cfg, steps=8)
    h = fde.MgHierarchy.build_geometric(p, n, n, 8, 1, 0.7, fde.COARSE_SWEEPS, 3)
    assert h.dims() == orc.plan(s)[0]
    b = np.random.default_rng(n + 1).uniform(-1, 1, n * n)
    assert rel(h.vcycle(dev(b)).cpu().numpy(), orc.vcycle(s, b)) <= 1e-12


@pytest.mark.parametrize("n", [2047, 4095])
def test_apply_identities_fullsize(cuda, n):
    """apply + apply_rhs = 2 inv_r x and linearity."""
    import torch
    p = fde.Problem.preset_config(5, steps=1)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 1, 1)
    inv_r = p.grid(n, n, 1)["inv_r"]
    g = torch.Generator(device="cuda").manual_seed(1)
    x = torch.rand(n * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y = torch.rand(n * n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    ax = op.apply(x)
    s = ax + op.apply_rhs(x)
    # inv_r x is ~1e-4 of the structured terms: the bar is relative to ||A x||
    assert float(torch.linalg.norm(s - 2 * inv_r * x) / torch.linalg.norm(ax)) <= 1e-14
    lhs = op.apply(3.0 * x - 0.5 * y)
    rhs = 3.0 * op.apply(x) - 0.5 * op.apply(y)
    assert float(torch.linalg.norm(lhs - rhs) / torch.linalg.norm(rhs)) <= 1e-13


def test_march_cfg1_p2_vs_golden(cuda):
    gd = np.load(GOLD / "cfg1_p2.npz")
    its, us = run_march(1, 63, 64, mg_cfg(precond=fde.PRECOND_P2))
    np.testing.assert_array_equal(its, gd["its"])
    assert rel(us[-1], gd["u_final"]) <= 1e-10
    assert compare_summary(us, gd, 1e-10) <= 1e-10


def test_march_cfg2_vs_golden(cuda):
    gd = np.load(GOLD / "cfg2_4steps.npz")
    its, us = run_march(2, 255, 4, mg_cfg())
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(us, gd, 1e-10) <= 1e-10
    assert rel(us[-1][sample_idx(255 * 255)], gd["samples"]) <= 1e-10


def test_march_cfg2_full_vs_oracle(cuda, orc):
    """cfg2 (n=255, 32 steps) step by step against the C oracle."""
    ro = orc.march(spec(2), record=True)
    its, us = run_march(2, 255, 32, mg_cfg())
    np.testing.assert_array_equal(its, ro["its"])
    for k in range(32):
        assert rel(us[k], ro["u_steps"][k]) <= 1e-10, k


@pytest.mark.parametrize("name,coarse", [("cfg3_sweeps", fde.COARSE_SWEEPS), ("cfg3_lu", fde.COARSE_LU)])
def test_march_cfg3_gmres_vs_golden(cuda, name, coarse):
    path = GOLD / f"{name}.npz"
    if not path.exists():
        pytest.skip(f"{name} golden not generated")
    gd = np.load(path)
    its, us = run_march(3, 1023, 16, mg_cfg(tol=1e-10, restart=30, coarse=coarse))
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(us, gd, 1e-10) <= 1e-10
    assert rel(us[-1][sample_idx(1023 * 1023)], gd["samples"]) <= 1e-10


def test_march_cfg4_vs_golden(cuda):
    path = GOLD / "cfg4.npz"
    if not path.exists():
        pytest.skip("cfg4 golden not generated")
    gd = np.load(path)
    its, us = run_march(4, 2047, 8, mg_cfg())
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(us, gd, 1e-10) <= 1e-10
    assert rel(us[-1][sample_idx(2047 * 2047)], gd["samples"]) <= 1e-10


@pytest.mark.parametrize("coarse", [fde.COARSE_SWEEPS, fde.COARSE_LU])
def test_bicgstab_cfg3_reduced_vs_oracle(cuda, orc, coarse):
    """cfg3 orders/coefficients/(1,-1) weights at n=127: BiCGSTAB (not in the
    reference; oracle restatement) step by step."""
    s = spec(3, n1=127, n2=127, steps=4, coarse=coarse)
    ro = orc.march(s, record=True, solver=1)
    its, us = run_march(3, 127, 4, mg_cfg(tol=1e-10, restart=30, coarse=coarse, solver=1))
    np.testing.assert_array_equal(its, ro["its"])
    for k in range(4):
        assert rel(us[k], ro["u_steps"][k]) <= 1e-10, k


@pytest.mark.parametrize("coarse", [fde.COARSE_SWEEPS, fde.COARSE_LU])
def test_bicgstab_cfg3_full(cuda, coarse):
    path = GOLD / f"cfg3_bicgstab_{'lu' if coarse == fde.COARSE_LU else 'sweeps'}.npz"
    if not path.exists():
        pytest.skip("bicgstab golden not generated")
    gd = np.load(path)
    its, us = run_march(3, 1023, 16, mg_cfg(tol=1e-10, restart=30, coarse=coarse, solver=1))
    np.testing.assert_array_equal(its, gd["its"])
    assert compare_summary(us, gd, 1e-10) <= 1e-10


def test_march_pipelined_host_io(cuda):
    """prefetch_source / solution_async (pipelined host I/O) give the same
    trajectory as plain host-array steps (cfg2 grid, 4 steps)."""
    steps = 4
    p = fde.Problem.preset_config(2, steps=steps)
    n = p.n
    srcs = [np.ascontiguousarray(p.sample_source(n, n, steps, m)) for m in range(1, steps + 1)]
    ref = fde.March(p, n, n, steps, mg_cfg())
    want = []
    for m in range(steps):
        ref.step(srcs[m])
        want.append(ref.solution())
    pipe = fde.March(p, n, n, steps, mg_cfg())
    outs = [np.zeros(n * n) for _ in range(steps)]
    pipe.prefetch_source(srcs[0])
    pipe.prefetch_source(srcs[1])
    for m in range(steps):
        pipe.step(fde.March.PREFETCHED)
        if m + 2 < steps:
            pipe.prefetch_source(srcs[m + 2])
        pipe.solution_async(outs[m])
    pipe.wait()
    for m in range(steps):
        np.testing.assert_array_equal(outs[m], want[m])


def test_cfg5_largest_grid_n8191(cuda, orc):
    """cfg5's largest grid (n = 8191, 67 M unknowns, 16384-point circulants):
    the operator apply at 300 sampled points against direct Toeplitz sums
    built from the oracle's weights and coefficient fields, apply + apply_rhs
    = 2 inv_r x, and the zero-guess V-cycle's linearity in b."""
    import torch
    n = 8191
    s = spec(5, n1=n, n2=n, steps=1)
    p = fde.Problem.preset_config(5, steps=1)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 1, 1)
    g = orc.grid(s)
    dp, dm, ep, em = orc.coefficients(s)
    x = np.random.default_rng(8191).uniform(-1, 1, n * n)
    y = op.apply(dev(x)).cpu().numpy()
    # T = Toeplitz(col = -w_{1..n}, row = (-w_1, -w_0, 0, ...)) (structured.cpp:47-55)
    def colrow(gamma):
        _, w = orc.weights(gamma, n)
        col = -w[1:n + 1]
        row = np.zeros(n)
        row[0], row[1] = -w[1], -w[0]
        return col, row
    (ca, ra), (cb, rb) = colrow(1.7), colrow(1.3)
    k = np.arange(n)
    def tline(col, row, i, v):  # (T v)_i and (T^T v)_i
        t = np.where(i >= k, col[np.abs(i - k)], row[np.abs(k - i)])
        tt = np.where(k >= i, col[np.abs(k - i)], row[np.abs(i - k)])
        return t @ v, tt @ v
    X = x.reshape(n, n)  # [j, i], x fastest
    for q in np.random.default_rng(1).integers(0, n * n, 300):
        i, j = int(q % n), int(q // n)
        ty, tt = tline(ca, ra, i, X[j])
        qy, qt = tline(cb, rb, j, X[:, i])
        ref = g["inv_r"] * x[q] + dp[q] * ty + dm[q] * tt + g["s_over_r"] * (ep[q] * qy + em[q] * qt)
        assert abs(y[q] - ref) <= 1e-12 * np.abs(y).max(), (i, j, y[q], ref)
    xd = dev(x)
    ax = op.apply(xd)
    s2 = ax + op.apply_rhs(xd)
    assert float(torch.linalg.norm(s2 - 2 * g["inv_r"] * xd) / torch.linalg.norm(ax)) <= 1e-14
    del ax, s2
    h = fde.MgHierarchy.build_geometric(p, n, n, 1, 1, 0.7, fde.COARSE_SWEEPS, 3)
    assert h.dims() == orc.plan(s)[0]
    b1, b2 = xd, torch.flip(xd, [0])
    v = h.vcycle(3.0 * b1 - b2)
    v12 = 3.0 * h.vcycle(b1) - h.vcycle(b2)
    assert bool(torch.isfinite(v).all())
    assert float(torch.linalg.norm(v - v12) / torch.linalg.norm(v)) <= 1e-12


def test_cfg5_n8191_apply_full_vector_vs_oracle(cuda, orc):
    """cfg5's largest grid: every one of the 67 M outputs of one operator apply
    against the oracle's FFT apply (the sampled direct-sum check above pins
    the oracle's answer there)."""
    n = 8191
    s = spec(5, n1=n, n2=n, steps=1)
    p = fde.Problem.preset_config(5, steps=1)
    op = fde.StructuredFdeOperator.assemble(p, n, n, 1, 1)
    x = np.random.default_rng(5).uniform(-1, 1, n * n)
    y = op.apply(dev(x)).cpu().numpy()
    del op
    assert rel(y, orc.apply(s, x)) <= 1e-13
