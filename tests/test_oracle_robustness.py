"""Oracle pins from the paper's solver claims (CPU, test infrastructure).

The paper's central claim for the hot path is robustness of the star-patch multigrid:
* AL velocity block: the vertex-star patches capture the kernel of the div-div term,
  so the V-cycle is robust in gamma (Schoberl's framework);
* E-B block, Picard linearisation: a mixed vector Laplacian, Re_m-robust;
* outer block preconditioner: with exact inner solves the Schur complement
  approximation S~ "works very well" -- in 2D with Picard a handful of outer
  iterations.
These fix qualitative behaviour, not values: a plausible mistake in the patches, the
operators or the block structure (a missing patch DoF, a dropped coupling block, a wrong
sign) breaks them.  The gamma pin carries its own negative control (point-Jacobi
patches degrade with gamma), so it cannot pass vacuously.
Also: structural pins of the block upper-triangular preconditioner.
"""
import dataclasses

import numpy as np
import pytest


def _cfg(name, N, L, **kw):
    from paper_2104_14855_b200 import workloads
    return dataclasses.replace(workloads.small(name, N, L), **kw)


def _fgmres_its(orc, seed=3, maxit=60):
    n = orc.csr(orc.nlev - 1).rp.size - 1
    b = np.random.default_rng(seed).standard_normal(n)
    _, its, _, conv = orc.fgmres(b, maxit=maxit)
    return its if conv else None


@pytest.mark.parametrize("name,N,L,cap", [("c3", 16, 3, 14), ("c5", 4, 2, 8)], ids=["2D", "3D"])
def test_al_velocity_multigrid_is_gamma_robust(oracle_mod, name, N, L, cap):
    """FGMRES(GMRES(6)-smoothed V-cycle) counts do not grow with gamma."""
    from paper_2104_14855_b200 import workloads
    its = []
    for g in (1e2, 1e4, 1e6, 1e8):
        cfg = _cfg(name, N, L, Re=1.0, gamma=g)
        w, _, _ = workloads.draw(cfg, 1, 6)
        o = oracle_mod.Oracle(cfg, w)
        o.set_smoother("gmres", 6)
        its.append(_fgmres_its(o))
    assert None not in its and max(its) <= cap and max(its) - min(its) <= 1, its
    # negative control: one-DoF patches (point Jacobi) are not kernel-capturing
    ctrl = []
    for g in (1e2, 1e6):
        cfg = _cfg(name, N, L, Re=1.0, gamma=g)
        w, _, _ = workloads.draw(cfg, 1, 6)
        o = oracle_mod.Oracle(cfg, w)
        o.set_smoother("gmres", 6)
        for lev in range(1, o.nlev):
            n = o.csr(lev).rp.size - 1
            o.set_patches(np.arange(n + 1), np.arange(n), lev)
        ctrl.append(_fgmres_its(o))
    assert ctrl[0] is not None and (ctrl[1] is None or ctrl[1] >= ctrl[0] + 10), ctrl


@pytest.mark.parametrize("name,N,L,cap,rems", [("c2", 32, 3, 12, (10.0, 1e2, 1e3, 1e4)),
                                               ("c4", 8, 3, 8, (10.0, 1e3, 1e4))], ids=["2D", "3D"])
def test_picard_eb_multigrid_is_Rem_robust(oracle_mod, name, N, L, cap, rems):
    """Picard (delta = 0) E-B block = mixed vector Laplacian: Re_m-robust."""
    from paper_2104_14855_b200 import workloads
    its = []
    for rem in rems:
        cfg = _cfg(name, N, L, Re=rem, Rem=rem, picard=1)
        w, _, _ = workloads.draw(cfg, 1, 6)
        o = oracle_mod.Oracle(cfg, w)
        o.set_smoother("gmres", 6)
        its.append(_fgmres_its(o))
    assert None not in its and max(its) <= cap, its


def _fgmres_np(A, P, b, m, tol):
    """Plain flexible GMRES (numpy, least squares on the Hessenberg) for the pins."""
    n = len(b); beta = np.linalg.norm(b)
    V = np.zeros((m + 1, n)); H = np.zeros((m + 1, m))
    V[0] = b / beta
    for k in range(m):
        w = A(P(V[k]))
        for i in range(k + 1):
            H[i, k] = w @ V[i]; w = w - H[i, k] * V[i]
        H[k + 1, k] = np.linalg.norm(w); V[k + 1] = w / H[k + 1, k]
        e = np.zeros(k + 2); e[0] = beta
        y = np.linalg.lstsq(H[:k + 2, :k + 1], e, rcond=None)[0]
        if np.linalg.norm(H[:k + 2, :k + 1] @ y - e) <= tol * beta:
            return k + 1
    return None


@pytest.mark.parametrize("S,Re,gamma", [(1.0, 10.0, 1e2), (1e2, 1e2, 1e4), (1e3, 1e3, 1e4)])
def test_outer_schur_approximation_with_exact_inner_solves(oracle_mod, S, Re, gamma):
    """2D Picard: with exact (sparse LU) inner solves, the block upper-triangular
    preconditioner built on the oracle's coupled operator needs <= 4 outer FGMRES
    iterations for S up to 1e3 (P:635 'works very well as a preconditioner')."""
    import scipy.sparse as sp
    import scipy.sparse.linalg as sla
    from paper_2104_14855_b200 import workloads
    cfg = _cfg("c3", 16, 3, Re=Re, Rem=Re, gamma=gamma, S=S, picard=1)
    w, _, _ = workloads.draw(cfg, 1, 6)
    c = oracle_mod.CoupledOracle(cfg, w, workloads.magnetic_potential(cfg, 6))
    A = c.csr().to_scipy(c.n).tocsr()
    nu, nup = c.nu, c.nu + c.np_
    Mup = A[:nup, :nup].tolil()
    for q in range(nu, nup):
        Mup[q, q] = 1e-10            # pressure constants: regularised (Q = L^2_0)
    Mlu, Slu, K = sla.splu(Mup.tocsc()), sla.splu(A[nup:, nup:].tocsc()), A[:nu, nup:]

    def P(r):
        yEB = Slu.solve(r[nup:])
        z = r[:nup].copy()
        z[:nu] -= K @ yEB
        return np.concatenate([Mlu.solve(z), yEB])

    b = np.random.default_rng(3).standard_normal(c.n)
    b[nu:nup] -= b[nu:nup].mean()
    its = _fgmres_np(lambda x: A @ x, P, b, 20, 1e-8)
    assert its is not None and its <= 4, its


def test_block_preconditioner_structure(oracle_mod):
    """P = [[I, -M~^-1 K], [0, I]] diag(M~^-1, S~^-1): the E-B output ignores
    r_up; r_EB = 0 gives y_EB = 0; with K = 0 (S = 0, B^n = 0) the (u,p) output ignores
    r_EB; and the (u,p) response to r_EB follows -M_up^-1 K y_EB (sign of K)."""
    import scipy.sparse.linalg as sla
    from paper_2104_14855_b200 import workloads
    cfg = _cfg("c3", 8, 2, Re=1.0, Rem=1.0, gamma=1.0, S=1.0)
    w, _, _ = workloads.draw(cfg, 1, 6)
    c = oracle_mod.CoupledOracle(cfg, w, workloads.magnetic_potential(cfg, 6))
    nu, nup = c.nu, c.nu + c.np_
    rng = np.random.default_rng(5)
    r = rng.standard_normal(c.n)
    r0up, r0eb = r.copy(), r.copy()
    r0up[:nup] = 0.0
    r0eb[nup:] = 0.0
    y, y_eb_only, y_up_only = c.precondition(r), c.precondition(r0up), c.precondition(r0eb)
    assert np.array_equal(y[nup:], y_eb_only[nup:])
    assert not np.any(y_up_only[nup:])
    # sign/presence of K: compare with the exact (u,p) solve of -K y_EB
    A = c.csr().to_scipy(c.n).tocsr()
    Mup = A[:nup, :nup].tolil()
    for q in range(nu, nup):
        Mup[q, q] = 1e-10
    ref = sla.splu(Mup.tocsc()).solve(np.concatenate([-(A[:nu, nup:] @ y_eb_only[nup:]), np.zeros(c.np_)]))
    got = y_eb_only[:nu]
    cos = got @ ref[:nu] / (np.linalg.norm(got) * np.linalg.norm(ref[:nu]))
    assert np.linalg.norm(got) > 0 and cos > 0.5, cos      # measured 0.78 (FGMRES(2) is inexact); -K gives < 0
    # K = 0: the (u,p) part is decoupled from r_EB
    cfg0 = _cfg("c3", 8, 2, Re=1.0, Rem=1.0, gamma=1.0, S=0.0)
    c0 = oracle_mod.CoupledOracle(cfg0, w, None)
    assert np.array_equal(c0.precondition(r)[:nup], c0.precondition(r0eb)[:nup])
