"""Oracle pins for NEXT-3: the coupled Newton system over [u | p | E | B] (P:223-239,
Table 1) and the paper's outer solver (FGMRES with the block upper-triangular
preconditioner).  Pins are algebraic identities of the continuous forms
(computed by different formulas in the oracle), degenerate cases with known answers,
and convergence of the outer solver."""
import dataclasses

import numpy as np
import pytest


def _case(oracle_mod, dim, N, L, S=1.0, bn=True, **kw):
    from paper_2104_14855_b200 import workloads
    cfg = dataclasses.replace(workloads.small("c3" if dim == 2 else "c5", N, L), Re=1.0, Rem=1.0, gamma=1.0, S=S, **kw)
    w, _, _ = workloads.draw(cfg, 1, 0)
    bnp = workloads.magnetic_potential(cfg, 0) if bn else None
    return cfg, oracle_mod.CoupledOracle(cfg, w, bnp)


@pytest.mark.parametrize("dim,N", [(2, 4), (3, 2)])
def test_block_identities(oracle_mod, dim, N):
    """J = S G^T ((B^n x E).v = E.(v x B^n)); the p rows are the transpose of the p
    columns (B = (B^T)^T); B^T annihilates constant pressures (-(1, div v) = 0)."""
    cfg, c = _case(oracle_mod, dim, N, 1, S=2.5)
    A = c.csr().to_scipy(c.n).toarray()
    u, p, E = slice(0, c.nu), slice(c.nu, c.nu + c.np_), slice(c.nu + c.np_, c.nu + c.np_ + c.nE)
    J, G = A[u, E], A[E, u]
    assert np.abs(G).max() > 0
    assert np.allclose(J, 2.5 * G.T, rtol=1e-12, atol=1e-12 * np.abs(J).max())
    Bt, B = A[u, p], A[p, u]
    assert np.array_equal(B, Bt.T)
    assert np.abs(Bt @ np.ones(c.np_)).max() <= 1e-12 * np.abs(Bt).max()


def test_decoupled_limit(oracle_mod):
    """S = 0 and B^n = 0: J = D~ = G = 0, the system is block diagonal and the E-B part
    of the FGMRES solution solves the E-B block alone."""
    cfg, c = _case(oracle_mod, 2, 4, 2, S=0.0, bn=False)
    A = c.csr().to_scipy(c.n).toarray()
    nup = c.nu + c.np_
    assert np.abs(A[:nup, nup:]).max() == 0 and np.abs(A[nup:, :nup]).max() == 0
    b = np.random.default_rng(1).uniform(-1, 1, c.n)
    b[c.nu:nup] -= b[c.nu:nup].mean()            # consistent pressure data (constants in the kernel)
    x, its, _, conv = c.fgmres(b, maxit=80)
    assert conv
    N_ = A[nup:, nup:]
    assert np.linalg.norm(N_ @ x[nup:] - b[nup:]) <= 1e-6 * np.linalg.norm(b)


@pytest.mark.parametrize("dim,N,L", [(2, 8, 2), (3, 4, 2)])
def test_outer_fgmres_converges(oracle_mod, dim, N, L):
    cfg, c = _case(oracle_mod, dim, N, L, S=1.0)
    b = np.random.default_rng(2).uniform(-1, 1, c.n)
    b[c.nu:c.nu + c.np_] -= b[c.nu:c.nu + c.np_].mean()
    x, its, hist, conv = c.fgmres(b, maxit=60)
    assert conv and its < 60
    r = b - c.apply(x)
    assert np.linalg.norm(r) <= 1.05 * max(1e-7 * np.linalg.norm(b), 1e-7)


def test_preconditioner_is_linear_in_exact_arithmetic_limit(oracle_mod):
    """The block preconditioner with FGMRES(2) inner solves is nonlinear in general, but
    its output scales with the input: P(alpha r) = alpha P(r) for alpha a power of two
    (every operation commutes exactly with the scaling)."""
    cfg, c = _case(oracle_mod, 2, 4, 2)
    r = np.random.default_rng(3).uniform(-1, 1, c.n)
    y1 = c.precondition(r)
    y2 = c.precondition(4.0 * r)
    assert np.array_equal(4.0 * y1, y2)
