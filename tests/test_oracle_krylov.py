"""Oracle pins for NEXT-1 (the paper's GMRES(6)-smoothed V-cycle inside flexible GMRES,
P:625): the pinned inner product (reading R-dot), the GMRES(m) smoothing step
(R-gmres6) and flexible GMRES (R-fgmres).  Each pin is independent of the oracle's
own arithmetic: exact rational arithmetic, closed forms, or textbook properties."""
import math
from fractions import Fraction

import numpy as np
import pytest


def _fma(a, b, c):
    return float(Fraction(a) * Fraction(b) + Fraction(c))   # correctly rounded (ties to even)


def pinned_dot_reference(a, b):
    """R-dot written out independently: 256-blocks of fma chains, pairwise tree."""
    n = len(a)
    if n == 0:
        return 0.0
    s = []
    for B in range(0, n, 256):
        acc = 0.0
        for i in range(B, min(n, B + 256)):
            acc = _fma(float(a[i]), float(b[i]), acc)
        s.append(acc)
    while len(s) > 1:
        t = [s[2 * k] + s[2 * k + 1] for k in range(len(s) // 2)]
        if len(s) % 2:
            t.append(s[-1])
        s = t
    return s[0]


@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 1000, 3000])
def test_dot_matches_exact_order(oracle_mod, n):
    rng = np.random.default_rng(n)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    assert oracle_mod.dot(a, b) == pinned_dot_reference(a, b)


def test_dot_exact_on_integers_and_error_bound(oracle_mod):
    a = np.arange(-500, 500, dtype=np.float64)
    assert oracle_mod.dot(a, a) == float(sum(int(v) ** 2 for v in a))
    rng = np.random.default_rng(1)
    x, y = rng.uniform(-1, 1, 100000), rng.uniform(-1, 1, 100000)
    exact = math.fsum(float(Fraction(u) * Fraction(v)) for u, v in zip(x[:2000], y[:2000]))
    got = oracle_mod.dot(x[:2000], y[:2000])
    assert abs(got - exact) <= 2000 * 2.0 ** -52 * np.sum(np.abs(x[:2000] * y[:2000]))


@pytest.fixture(scope="module")
def small(oracle_mod):
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c3", 4, 2)
    w, _, _ = workloads.draw(cfg, 1, 0)
    orc = oracle_mod.Oracle(cfg, w)
    n = orc.n()
    rng = np.random.default_rng(3)
    return orc, n, rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)


def _B(orc, r):
    return orc.sweep(r, np.zeros_like(r), x_is_zero=True)


def test_gmres_one_step_is_minimal_residual_richardson(small):
    """m = 1: x1 = x0 + alpha z, z = B r0, alpha = (Bt . z)/(Bt . Bt), t = A z (closed form
    of the one-dimensional least-squares problem of left-preconditioned GMRES)."""
    orc, n, b, x0 = small
    r0 = orc.residual(b, x0)
    z = _B(orc, r0)
    bt = _B(orc, orc.spmv(z))
    alpha = np.dot(bt, z) / np.dot(bt, bt)
    x1 = orc.gmres_smooth(b, x0, m=1)
    assert np.linalg.norm(x1 - (x0 + alpha * z)) <= 1e-9 * np.linalg.norm(alpha * z)


def test_gmres_preconditioned_residual_monotone(small):
    orc, n, b, x0 = small
    res = []
    for m in range(1, 9):
        x = orc.gmres_smooth(b, x0, m=m)
        res.append(np.linalg.norm(_B(orc, orc.residual(b, x))))
    assert all(res[k + 1] <= res[k] * (1 + 1e-10) for k in range(len(res) - 1))
    assert res[-1] < 0.5 * np.linalg.norm(_B(orc, orc.residual(b, x0)))


def test_gmres_full_krylov_space_is_direct_solve(oracle_mod):
    """m = n: the Krylov space of B A is the whole space, so one smoothing step solves
    A x = b (up to rounding amplified by the condition number)."""
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c1", 2, 2)          # finest n = 9
    w, _, _ = workloads.draw(cfg, 1, 2)
    orc = oracle_mod.Oracle(cfg, w)
    n = orc.n()
    assert n == 9
    b = np.random.default_rng(4).uniform(-1, 1, n)
    A = orc.csr().to_scipy().toarray()
    x = orc.gmres_smooth(b, np.zeros(n), m=n, x_is_zero=True)
    assert np.linalg.norm(A @ x - b) <= 1e-12 * np.linalg.cond(A) * np.linalg.norm(b)
    x2 = orc.gmres_smooth(b, np.zeros(n), m=n - 3, x_is_zero=True)
    assert np.linalg.norm(A @ x2 - b) > np.linalg.norm(A @ x - b)


def test_fgmres_converges_and_meets_tolerance(oracle_mod):
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c1", 8, 2)
    w, b, _ = workloads.draw(cfg, 225, 0)
    orc = oracle_mod.Oracle(cfg, w)
    orc.set_smoother("gmres", 6)
    x, its, hist, conv = orc.fgmres(b)
    assert conv and its <= 20
    A = orc.csr().to_scipy()
    assert np.linalg.norm(b - A @ x) <= 1.01 * max(1e-7 * np.linalg.norm(b), 1e-7)
    assert np.all(np.diff(hist) <= 1e-12 * hist[0])       # GMRES residual estimates never grow


def test_fgmres_with_exact_preconditioner_one_iteration(oracle_mod):
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c1", 4, 1)
    w, b, _ = workloads.draw(cfg, 49, 0)
    orc = oracle_mod.Oracle(cfg, w)          # one level: the V-cycle is the coarse LU solve
    orc.set_smoother("gmres", 6)
    x, its, _, conv = orc.fgmres(b)
    assert conv and its == 1
