"""Independent pins for the two rows the reference cannot pin (SURVEY.md 8(a')):
the WSGD (p,q) = (1,-1) weight table and BiCGSTAB.

The reference implements neither, so these tests anchor them on sources
OUTSIDE this repo's own restatement:

* (1,-1) weights -- the weighted and shifted Gruenwald difference operators of
  Tian, Zhou and Deng, "A class of second order difference approximations for
  solving space fractional diffusion equations", Math. Comp. 84 (2015):
  lambda_1 = (gamma - 2q) / (2(p - q)), lambda_2 = (2p - gamma) / (2(p - q)),
  which for (1,-1) gives  w_0 = l1 g_0, w_1 = l1 g_1, w_k = l1 g_k + l2 g_{k-2}
  with l1 = (2 + gamma)/4, l2 = (2 - gamma)/4.  Checked three ways: exact hand
  values at gamma = 3/2, the same lambda formula reproducing the reference's
  own (1,0) table (proj/src/weights.cpp:44-47), and second-order convergence of
  the discrete Riemann-Liouville derivative of x^4 (1-x)^4, whose closed form
  is the power rule the reference's manufactured sources use
  (proj/src/problem.cpp:152-170; the exponent 4 makes the zero extension C^3,
  so the truncation error is second order uniformly up to the boundary -- with
  the reference's x^2 (1-x)^2 both tables, the reference's (1,0) included,
  drop to first order in the maximum norm at the first nodes).  A wrong shift or weight makes the operator
  first order (or inconsistent) and fails the ratio test.
* BiCGSTAB -- scipy.sparse.linalg.bicgstab (van der Vorst's recurrences) on the
  dense left-preconditioned system M^-1 A at n = 31: the iterates are unique
  given r^_0 = r_0, so the per-iteration residuals must coincide.
"""
import ctypes
import math

import numpy as np
import pytest

from oracles import oracle, spec


@pytest.fixture(scope="module")
def orc():
    return oracle()


def lib_weights(gamma, K, pq):
    """The product's own host weight table (fde_wsgd_weights, CPU callable)."""
    import paper_1706_06844_b200 as fde
    lib = fde.load_library()
    g, w = np.zeros(K + 1), np.zeros(K + 1)
    P = ctypes.POINTER(ctypes.c_double)
    rc = lib.fde_wsgd_weights(ctypes.c_double(gamma), K, pq, g.ctypes.data_as(P),
                              w.ctypes.data_as(P))
    assert rc == 0
    return g, w


def wsgd_by_lambda(gamma, K, p, q):
    """Tian-Zhou-Deng weights for integer shifts p > q >= -1 written from the
    paper's definition: the shift-p Gruenwald sum has g_k at offset k - p, and
    the matrix layout stores offset k - 1 (one node to the right of x_i)."""
    g = np.zeros(K + 1)
    g[0] = 1.0
    for k in range(1, K + 1):
        g[k] = g[k - 1] * (1.0 - (gamma + 1.0) / k)
    l1 = (gamma - 2.0 * q) / (2.0 * (p - q))
    l2 = (2.0 * p - gamma) / (2.0 * (p - q))
    w = np.zeros(K + 1)
    for k in range(K + 1):
        # offset (k - 1) = (kp - p) = (kq - q)
        kp, kq = k - 1 + p, k - 1 + q
        if 0 <= kp <= K:
            w[k] += l1 * g[kp]
        if 0 <= kq <= K:
            w[k] += l2 * g[kq]
    return w


@pytest.mark.parametrize("source", ["oracle", "library"])
def test_wsgd_1m1_hand_values(orc, source):
    # gamma = 3/2: g = 1, -3/2, 3/8, 1/16, 3/128; l1 = 7/8, l2 = 1/8 (dyadic: exact)
    g, w = orc.weights(1.5, 8, pq=1) if source == "oracle" else lib_weights(1.5, 8, 1)
    # (the recurrence g_k = g_{k-1} (1 - (gamma+1)/k) rounds at k = 3; the reference's own
    # hand-value check uses 1e-14, verify.cpp:163-181)
    np.testing.assert_allclose(g[:5], [1.0, -1.5, 0.375, 0.0625, 0.0234375], rtol=0, atol=1e-15)
    hand = [0.875, -1.3125, 0.453125, -0.1328125, 0.0673828125]
    np.testing.assert_allclose(w[:5], hand, rtol=0, atol=1e-15)


@pytest.mark.parametrize("gamma", [1.1, 1.5, 1.9, 2.0])
def test_wsgd_lambda_formula_reproduces_both_tables(orc, gamma):
    K = 64
    # (1,0): the reference's own table (weights.cpp:44-47, pinned by test_oracle_pins)
    np.testing.assert_allclose(orc.weights(gamma, K, pq=0)[1], wsgd_by_lambda(gamma, K, 1, 0),
                               rtol=1e-14, atol=1e-16)
    # (1,-1): the same definition with q = -1
    for w in (orc.weights(gamma, K, pq=1)[1], lib_weights(gamma, K, 1)[1]):
        np.testing.assert_allclose(w, wsgd_by_lambda(gamma, K, 1, -1), rtol=1e-14, atol=1e-16)


def rl_derivative_exact(gamma, x):
    """Left Riemann-Liouville derivative of u = x^4 (1-x)^4 = x^4 - 4 x^5 + 6 x^6 - 4 x^7 + x^8
    on [0, 1]: D^g x^m = Gamma(m+1) / Gamma(m+1-g) x^(m-g) (problem.cpp:152-170)."""
    def term(m):
        return math.gamma(m + 1) / math.gamma(m + 1 - gamma) * x ** (m - gamma)
    return term(4) - 4.0 * term(5) + 6.0 * term(6) - 4.0 * term(7) + term(8)


@pytest.mark.parametrize("gamma", [1.1, 1.5, 1.9])
@pytest.mark.parametrize("pq", [0, 1])
def test_wsgd_second_order_on_manufactured_solution(orc, gamma, pq):
    """max error of h^-gamma sum_k w_k u(x_{i-k+1}) against the exact derivative
    drops by ~4 per halving of h for both weight tables."""
    errs = []
    for n in (127, 255, 511, 1023):
        h = 1.0 / (n + 1)
        x = h * np.arange(0, n + 2)  # nodes 0..n+1, u(0) = u(1) = 0
        u = x ** 4 * (1.0 - x) ** 4
        w = orc.weights(gamma, n + 1, pq=pq)[1]
        d = np.zeros(n)
        for i in range(1, n + 1):
            k = np.arange(0, i + 2)  # u(x_{i-k+1}), k = 0 .. i+1
            d[i - 1] = np.dot(w[k], u[i - k + 1]) / h ** gamma
        errs.append(np.max(np.abs(d - rl_derivative_exact(gamma, x[1:n + 1]))))
    ratios = [errs[i] / errs[i + 1] for i in range(len(errs) - 1)]
    # second order: ratios approach 4 from below as h -> 0 (a first-order table gives 2)
    assert all(3.2 <= r <= 4.6 for r in ratios) and ratios[-1] >= 3.7, (errs, ratios)


def test_bicgstab_matches_scipy_on_dense_preconditioned_system(orc):
    from scipy.sparse.linalg import bicgstab

    n = 31
    s = spec(3, n1=n, n2=n, steps=4, restart=30, tol=1e-10)  # cfg3 orders, (1,-1), mgm sweeps
    N = n * n
    A = np.zeros((N, N))
    Minv = np.zeros((N, N))
    e = np.zeros(N)
    for j in range(N):
        e[j] = 1.0
        A[:, j] = orc.apply(s, e)
        Minv[:, j] = orc.precond(s, e)
        e[j] = 0.0
    b = orc.rhs(s, 1, orc.initial(s))
    B, c = Minv @ A, Minv @ b
    xs = []
    x_sp, info = bicgstab(B, c, x0=np.zeros(N), rtol=1e-13, atol=0.0, maxiter=200,
                          callback=lambda xk: xs.append(xk.copy()))
    assert info == 0
    x_or, its, conv, hist = orc.bicgstab(s, b)
    assert conv
    # hist[0] = 1 (zero guess), hist[k] = ||M^-1 (b - A x_k)|| / ||M^-1 b|| after full step k;
    # the last entry is the verified true residual of the accepted iterate
    nc = np.linalg.norm(c)
    res_sp = [np.linalg.norm(c - B @ xk) / nc for xk in xs]
    m = min(len(hist) - 2, len(res_sp))
    assert m >= 3, (len(hist), len(res_sp))
    for k in range(m):
        assert hist[k + 1] == pytest.approx(res_sp[k], rel=1e-5, abs=1e-13), (k, hist, res_sp)
    # and both reach the same solution of the preconditioned system
    assert np.linalg.norm(x_or - x_sp) / np.linalg.norm(x_sp) <= 1e-8
