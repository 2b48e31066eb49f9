"""Pin the CPU oracle (oracle/fde_oracle.c) before trusting it as the checker.

* known-answer values from the reference's own verify suite and SPEC
  (verify.cpp:133-181);
* golden vectors produced by the UNMODIFIED reference (tests/golden, made by
  tools/make_golden.py from oracle/_ref);
* the reference build itself (oracle/_ref) on seeded inputs, when present.
"""
import math
from pathlib import Path

import numpy as np
import pytest

from golden_util import compare_summary, sample_idx
from oracles import spec

GOLD = Path(__file__).parent / "golden"


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def gold(name):
    return np.load(GOLD / f"{name}.npz")


# ---------------------------------------------------------------- weights
def test_weight_hand_values(orc):
    """verify.cpp:163-181 'hand-values' (tolerance 1e-14)."""
    _, w = orc.weights(1.5, 8)
    assert abs(w[0] - 0.75) <= 1e-14 and abs(w[1] + 0.875) <= 1e-14
    assert abs(w[2] + 0.09375) <= 1e-14
    _, w = orc.weights(1.8, 8)
    assert abs(w[1] + 1.52) <= 1e-14
    g, _ = orc.weights(2.0, 3)
    np.testing.assert_allclose(g, [1.0, -2.0, 1.0, 0.0], atol=1e-14, rtol=0)


@pytest.mark.parametrize("gamma", [1.1, 1.3, 1.5, 1.77, 2.0])
def test_binom_closed_form(orc, gamma):
    """verify.cpp:146-161: g_k = (-1)^k binom(gamma, k) against log-gamma, <= 1e-10."""
    g, _ = orc.weights(gamma, 200)
    for k in range(0, 200, 7):
        if gamma - k + 1 <= 0 and float(gamma - k + 1).is_integer():
            exact = 0.0
        else:
            lg = math.lgamma(gamma + 1) - math.lgamma(k + 1) - math.lgamma(gamma - k + 1)
            sign = (-1) ** k * math.copysign(1.0, math.gamma(gamma - k + 1)) if gamma - k + 1 < 0 else (-1) ** k
            exact = sign * math.exp(lg)
        assert abs(g[k] - exact) <= 1e-10 * max(1.0, abs(exact))


@pytest.mark.parametrize("gamma", [1.1, 1.25, 1.5, 1.75, 1.9, 2.0])
def test_weight_invariants(orc, gamma):
    """weights.cpp:59-115 invariants on K = 10^4 (verify.cpp:133-144)."""
    K = 10000
    g, w = orc.weights(gamma, K)
    assert g[0] == 1.0 and abs(g[1] + gamma) <= 1e-12
    assert abs(w[0] - gamma / 2) <= 1e-12
    assert abs(w[1] - (2 - gamma - gamma * gamma) / 2) <= 1e-12 and w[1] < 0
    assert abs(w[2] - gamma * (gamma * gamma + gamma - 4) / 4) <= 1e-12
    tail = w[3:]
    assert np.all(tail >= -1e-12)
    assert tail[0] <= w[0] + 1e-12 and np.all(np.diff(tail) <= 1e-12)
    ps = np.cumsum(w)[2:]
    assert np.all(ps <= 1e-12) if gamma == 2.0 else np.all(ps < 0)


def test_weights_match_golden(orc):
    gd = gold("weights")
    for gamma in (1.1, 1.3, 1.5, 1.6, 1.7, 1.8, 1.9, 2.0):
        for pq in (0, 1):
            g, w = orc.weights(gamma, 64, pq)
            np.testing.assert_array_equal(g, gd[f"g_{gamma}_{pq}"])
            np.testing.assert_allclose(w, gd[f"w_{gamma}_{pq}"], rtol=0, atol=1e-15)


# ---------------------------------------------------------------- FFT / Toeplitz
@pytest.mark.parametrize("n", [1, 2, 8, 64, 256])
def test_fft_vs_naive_dft(orc, n):
    """FFT == direct DFT to 1e-12 on random vectors."""
    rng = np.random.default_rng(n)
    for _ in range(20):
        a = rng.normal(size=n) + 1j * rng.normal(size=n)
        for inv in (False, True):
            f, d = orc.fft(a, inv), orc.naive_dft(a, inv)
            assert np.max(np.abs(f - d)) <= 1e-12 * max(1.0, np.max(np.abs(d)))
            np.testing.assert_allclose(f, np.fft.ifft(a) if inv else np.fft.fft(a), atol=1e-12 * n)


def dense_toeplitz(col, row):
    n = len(col)
    return np.array([[col[i - j] if i >= j else row[j - i] for j in range(n)] for i in range(n)])


def test_toeplitz_spec_examples(orc):
    """n=4, gamma=2: ones -> [1,0,0,1]; e_1 -> first column."""
    y, _ = orc.toeplitz_both(2.0, np.ones(4))
    np.testing.assert_allclose(y, [1, 0, 0, 1], atol=1e-14)
    e1 = np.zeros(4)
    e1[0] = 1
    _, w = orc.weights(2.0, 4)
    y, _ = orc.toeplitz_both(2.0, e1)
    np.testing.assert_allclose(y, -w[1:5], atol=1e-14)


@pytest.mark.parametrize("n", [1, 7, 8, 31, 64, 129])
def test_toeplitz_vs_dense(orc, n):
    rng = np.random.default_rng(n)
    col, row = rng.normal(size=n), rng.normal(size=n)
    row[0] = col[0]
    x = rng.normal(size=n)
    y, yt = orc.toeplitz_colrow(col, row, x)
    T = dense_toeplitz(col, row)
    assert np.max(np.abs(y - T @ x)) <= 1e-12 * max(1, np.abs(T @ x).max())
    assert np.max(np.abs(yt - T.T @ x)) <= 1e-12 * max(1, np.abs(T.T @ x).max())


def test_toeplitz_matches_golden(orc):
    gd = gold("toeplitz")
    for n in (1, 2, 3, 7, 8, 31, 33, 64, 100):
        for gamma, pq in ((1.5, 0), (1.8, 0), (1.1, 1)):
            y, yt = orc.toeplitz_both(gamma, gd[f"x_{n}"], pq)
            assert rel(y, gd[f"y_{n}_{gamma}_{pq}"]) <= 1e-13
            assert rel(yt, gd[f"yt_{n}_{gamma}_{pq}"]) <= 1e-13


# ---------------------------------------------------------------- operator / MG
def test_apply_plus_rhs_identity(orc):
    """apply_M + apply_rhs = 2 inv_r u."""
    s = spec(2, n1=31, n2=47, steps=4)
    x = np.random.default_rng(3).uniform(-1, 1, 31 * 47)
    inv_r = orc.grid(s)["inv_r"]
    np.testing.assert_allclose(orc.apply(s, x) + orc.apply(s, x, -1), 2 * inv_r * x, rtol=1e-13,
                               atol=1e-13 * inv_r)


def test_apply_vs_dense_cfg1(orc, ref):
    """dense_assemble oracle (structured.cpp:194-216) at cfg1, N = 3969."""
    s = spec(1)
    A = ref.dense(s)
    x = np.random.default_rng(5).uniform(-1, 1, 63 * 63)
    assert rel(orc.apply(s, x), A @ x) <= 1e-13
    np.testing.assert_array_equal(orc.diagonal(s), np.diag(A))


def test_operator_and_vcycle_match_golden(orc):
    gd = gold("apply")
    for cfg, n1, n2 in ((1, 63, 63), (2, 31, 47), (3, 64, 33), (4, 47, 31), (5, 63, 63)):
        s = spec(cfg, n1=n1, n2=n2, steps=4)
        x = gd[f"x_{cfg}"]
        assert rel(orc.apply(s, x), gd[f"y_{cfg}"]) <= 1e-13
        assert rel(orc.apply(s, x, -1), gd[f"yr_{cfg}"]) <= 1e-13
        np.testing.assert_array_equal(orc.diagonal(s), gd[f"diag_{cfg}"])
        for coarse in (0, 1, 2):
            sc = spec(cfg, n1=n1, n2=n2, steps=4, coarse=coarse)
            assert rel(orc.vcycle(sc, x), gd[f"v_{cfg}_{coarse}"]) <= 1e-12, (cfg, coarse)
        assert rel(orc.vcycle(spec(cfg, n1=n1, n2=n2, steps=4, precond=1), x), gd[f"p2_{cfg}"]) <= 1e-12


def test_plans_match_golden(orc):
    gd = gold("plans")
    for cfg in (1, 2, 3, 4, 5):
        dims, r0 = orc.plan(spec(cfg))
        assert [tuple(d) for d in gd[f"plan_{cfg}"].tolist()] == dims
        assert abs(r0 - float(gd[f"ratio0_{cfg}"])) <= 1e-12 * abs(r0)
    for n in (511, 1023, 4095, 8191):
        assert [tuple(d) for d in gd[f"plan_5_{n}"].tolist()] == orc.plan(spec(5, n1=n, n2=n))[0]


@pytest.mark.parametrize("n1,n2,cx,cy", [(63, 63, 1, 1), (64, 31, 1, 1), (30, 17, 1, 0),
                                         (17, 30, 0, 1), (2, 2, 1, 1), (3, 9, 0, 1)])
def test_transfers_match_reference(orc, ref, n1, n2, cx, cy):
    rng = np.random.default_rng(n1 * 31 + n2)
    k1 = (n1 - n1 % 2) // 2 if cx else n1
    k2 = (n2 - n2 % 2) // 2 if cy else n2
    f, c = rng.uniform(-1, 1, n1 * n2), rng.uniform(-1, 1, k1 * k2)
    np.testing.assert_array_equal(orc.transfer(n1, n2, cx, cy, 0, c), ref.transfer(n1, n2, cx, cy, 0, c))
    for op in (1, 2):
        np.testing.assert_array_equal(orc.transfer(n1, n2, cx, cy, op, f), ref.transfer(n1, n2, cx, cy, op, f))


@pytest.mark.parametrize("cfg,n", [(2, 63), (3, 95), (4, 127), (5, 127)])
def test_vcycle_matches_reference(orc, ref, cfg, n):
    b = np.random.default_rng(n).uniform(-1, 1, n * n)
    for coarse in (0, 1):
        s = spec(cfg, n1=n, n2=n, steps=4, coarse=coarse)
        assert orc.plan(s)[0] == ref.plan(s)[0]
        assert rel(orc.vcycle(s, b), ref.vcycle(s, b)) <= 1e-12


# ---------------------------------------------------------------- Krylov / march
def test_gmres_matches_reference(orc, ref):
    s = spec(2, n1=63, n2=63, steps=4)
    b = orc.rhs(s, 1, orc.initial(s))
    xo, ito, co, ho = orc.gmres(s, b)
    xr, itr, cr, hr = ref.gmres(s, b)
    assert ito == itr and co == cr and len(ho) == len(hr)
    assert rel(xo, xr) <= 1e-12
    np.testing.assert_allclose(ho, hr, rtol=1e-8)


def test_march_cfg1_matches_golden(orc):
    """cfg1 (n=63, 64 steps, GMRES(20)+mgm): per-step iterations identical,
    trajectory summaries and sampled steps within 1e-12 of the reference."""
    gd = gold("cfg1")
    r = orc.march(spec(1), record=True)
    np.testing.assert_array_equal(r["its"], gd["its"])
    assert rel(r["u_steps"][0], gd["u_step1"]) <= 1e-12
    assert rel(r["u_steps"][31], gd["u_step32"]) <= 1e-12
    assert rel(r["u"], gd["u_final"]) <= 1e-12
    assert compare_summary(r["u_steps"], gd, 1e-12) <= 1e-12


def test_march_cfg1_p2_matches_golden(orc):
    gd = gold("cfg1_p2")
    r = orc.march(spec(1, precond=1), record=True)
    np.testing.assert_array_equal(r["its"], gd["its"])
    assert rel(r["u"], gd["u_final"]) <= 1e-12


def test_march_cfg2_matches_golden(orc):
    gd = gold("cfg2_4steps")
    r = orc.march(spec(2, steps=4), record=True)
    np.testing.assert_array_equal(r["its"], gd["its"])
    assert compare_summary(r["u_steps"], gd, 1e-12) <= 1e-12
    assert rel(r["u"][sample_idx(255 * 255)], gd["samples"]) <= 1e-12


def test_source_and_initial_match_reference(orc, ref):
    for cfg in (1, 3):
        s = spec(cfg, n1=40, n2=30, steps=4)
        np.testing.assert_array_equal(orc.source(s, 3), ref.source(s, 3))
        np.testing.assert_array_equal(orc.initial(s), ref.initial(s))
        for k, (a, b) in enumerate(zip(orc.coefficients(s), ref.coefficients(s))):
            np.testing.assert_array_equal(a, b)


def test_bicgstab_converges_and_is_deterministic(orc):
    """BiCGSTAB is not in the reference (unpinned): check it solves the
    left-preconditioned system to tol and agrees with GMRES's solution."""
    s = spec(3, n1=63, n2=63, steps=4, restart=30, tol=1e-10)
    b = orc.rhs(s, 1, orc.initial(s))
    xb, itb, cb, hb = orc.bicgstab(s, b)
    xg, itg, cg, hg = orc.gmres(s, b)
    assert cb and cg and hb[-1] <= 1e-10
    assert rel(xb, xg) <= 1e-8
    xb2, itb2, _, _ = orc.bicgstab(s, b)
    assert itb2 == itb and np.array_equal(xb, xb2)
