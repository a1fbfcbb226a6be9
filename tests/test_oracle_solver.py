"""Pins of the oracle's dense LU, sweep, transfer, V-cycle and GMRES against
special cases, closed forms, brute force and library routines.
"""
import dataclasses

import numpy as np
import pytest
import scipy.linalg as sla
import scipy.sparse.linalg as spla

import mms
from paper_2104_14855_b200.workloads import CONFIGS, draw, small


def make(oracle_mod, cfg, **kw):
    w, _, _ = draw(cfg, 0, 0)
    return oracle_mod.Oracle(cfg, w, **kw)


# ---------------- dense LU (R-lu) ----------------
def test_lu_random_matches_library(oracle_mod):
    rng = np.random.default_rng(0)
    for n in (1, 2, 7, 50, 108):
        a = rng.standard_normal((n, n)) + n * np.eye(n) * 0.1
        b = rng.standard_normal(n)
        x, lu, perm, st = oracle_mod.dense_lu_solve(a, b)
        assert st == 0
        ref = np.linalg.solve(a, b)
        assert np.linalg.norm(x - ref) <= 1e-11 * np.linalg.norm(ref)
        # P A = L U with the returned factors
        L = np.tril(lu, -1) + np.eye(n); U = np.triu(lu)
        assert np.abs(a[perm] - L @ U).max() <= 1e-13 * np.abs(a).max() * n
        # partial pivoting: |l_ij| <= 1
        assert np.abs(np.tril(lu, -1)).max(initial=0) <= 1.0


def test_lu_pivot_rule_and_permutation():
    from oracle import oracle as om
    # permutation matrix: exact solve, perm recovers the row order
    P = np.eye(5)[[3, 0, 4, 1, 2]]
    b = np.arange(1.0, 6.0)
    x, lu, perm, st = om.dense_lu_solve(P, b)
    assert st == 0 and np.array_equal(x, np.linalg.solve(P, b))
    # ties -> smallest row index: |a00| == |a10| keeps row 0 first
    a = np.array([[1.0, 2.0], [-1.0, 3.0]])
    x, lu, perm, st = om.dense_lu_solve(a, np.array([1.0, 1.0]))
    assert list(perm) == [0, 1]
    # Hilbert matrix (ill-conditioned): small backward error
    n = 8
    H = sla.hilbert(n)
    xh, _, _, st = om.dense_lu_solve(H, np.ones(n))
    assert st == 0 and np.linalg.norm(H @ xh - 1) <= 1e-12 * np.linalg.norm(H, 2) * np.linalg.norm(xh)
    # singular: zero column -> status k+1
    S = np.array([[1.0, 2.0, 3.0], [2.0, 4.0, 6.0], [0.0, 0.0, 0.0]])
    assert om.dense_lu_solve(S, np.ones(3))[3] == 2


# ---------------- sweep ----------------
def _brute_sweep(A, b, x, ptr, dofs, mult):
    """The subspace-correction step written with numpy.linalg.solve per patch."""
    r = b - A @ x
    c = np.zeros_like(x)
    for i in range(len(ptr) - 1):
        d = dofs[ptr[i]:ptr[i + 1]]
        c[d] += np.linalg.solve(A[np.ix_(d, d)], r[d])
    return x + c / mult


@pytest.mark.parametrize("name,N", [("c1", 8), ("c3", 4), ("c4", 2), ("c5", 2)])
def test_sweep_matches_brute_force(oracle_mod, name, N):
    cfg = small(name, N, 1)
    o = make(oracle_mod, cfg)
    n = o.n()
    _, b, x0 = draw(cfg, n, 1)
    A = o.csr().to_scipy().toarray()
    ptr, dofs, vert, mult = o.patches()
    for x in (np.zeros(n), x0):
        got = o.sweep(b, x, x_is_zero=not x.any())
        ref = _brute_sweep(A, b, x, ptr, dofs, mult)
        kap = max(np.linalg.cond(A[np.ix_(dofs[ptr[i]:ptr[i + 1]], dofs[ptr[i]:ptr[i + 1]])]) for i in range(len(ptr) - 1))
        assert np.linalg.norm(got - ref) <= max(1e-12, 50 * kap * 1.1e-16) * np.linalg.norm(ref)


@pytest.mark.parametrize("name,N,mode", [("c1", 8, 1), ("c1", 8, 2), ("c3", 4, 2), ("c5", 2, 2), ("c4", 2, 1)])
def test_sweep_weights_mode_matches_brute_force(oracle_mod, name, N, mode):
    """weights_mode ("damping parameters w_i"): 1 = per-DoF partition of
    unity 1/m_d, 2 = the uniform per-subspace weight 1/max_d m_d -- against the brute-force
    sweep written with that weight; mode 0 (by degree) is mode 1 at k = 1."""
    import dataclasses
    cfg = dataclasses.replace(small(name, N, 1), weights_mode=mode)
    o = make(oracle_mod, cfg)
    n = o.n()
    _, b, x0 = draw(cfg, n, 1)
    A = o.csr().to_scipy().toarray()
    ptr, dofs, vert, mult = o.patches()
    wdiv = mult if mode == 1 else np.full(n, mult.max())
    got = o.sweep(b, x0)
    ref = _brute_sweep(A, b, x0, ptr, dofs, wdiv)
    kap = max(np.linalg.cond(A[np.ix_(dofs[ptr[i]:ptr[i + 1]], dofs[ptr[i]:ptr[i + 1]])]) for i in range(len(ptr) - 1))
    assert np.linalg.norm(got - ref) <= max(1e-12, 50 * kap * 1.1e-16) * np.linalg.norm(ref)
    if mode == 2 and mult.min() != mult.max():          # the two modes really differ here
        o1 = make(oracle_mod, dataclasses.replace(cfg, weights_mode=1))
        assert not np.array_equal(o1.sweep(b, x0), got)
    d0 = make(oracle_mod, dataclasses.replace(cfg, weights_mode=0)).sweep(b, x0)
    d1 = make(oracle_mod, dataclasses.replace(cfg, weights_mode=1)).sweep(b, x0)
    assert np.array_equal(d0, d1)                        # k = 1: by degree = per-DoF


@pytest.mark.parametrize("name,N", [("c3", 4), ("c5", 2)])
def test_newton_reaction_vanishes_under_piecewise_constant_w(oracle_mod, name, N):
    """Reading R-newton: with the advecting field of R-w (curl / vcurl of a lowest-order
    interpolant: constant on every cell), grad u^n = 0 cellwise, so the Newton reaction
    (u . grad u^n, v) of Table 1 row F adds nothing: the flag is accepted and
    leaves the assembled operator unchanged (the zero of the term is a consequence of
    R-w, not something this test can pin independently)."""
    import dataclasses
    cfg = small(name, N, 1)
    o = make(oracle_mod, cfg)
    on = make(oracle_mod, dataclasses.replace(cfg, newton_reaction=1))
    A, An = o.csr(), on.csr()
    assert np.array_equal(A.rp, An.rp) and np.array_equal(A.v, An.v)


@pytest.mark.parametrize("name,N", [("c1", 4), ("c3", 3), ("c5", 1), ("c4", 2)])
def test_single_patch_is_direct_solve(oracle_mod, name, N):
    """One patch covering every free DoF (m_d = 1) => one sweep from zero is the
    exact solve (SURVEY §8c.12 "Patch solve"); two such patches with the partition
    of unity weights 1/2 give the same."""
    cfg = small(name, N, 1)
    o = make(oracle_mod, cfg)
    n = o.n()
    _, b, _ = draw(cfg, n, 2)
    A = o.csr().to_scipy().toarray()
    ref = np.linalg.solve(A, b)
    tol = max(1e-12, 10 * np.linalg.cond(A) * 1.1e-16)       # two LU codes differ by ~kappa u
    o.set_patches(np.array([0, n]), np.arange(n))
    x = o.sweep(b, None, x_is_zero=True)
    assert np.linalg.norm(x - ref) <= tol * np.linalg.norm(ref)
    o.set_patches(np.array([0, n, 2 * n]), np.concatenate([np.arange(n), np.arange(n)]))
    x2 = o.sweep(b, None, x_is_zero=True)
    assert np.linalg.norm(x2 - ref) <= tol * np.linalg.norm(ref)


def test_sweep_linear_and_zero_flag(oracle_mod):
    cfg = small("c3", 8, 1)
    o = make(oracle_mod, cfg)
    n = o.n()
    rng = np.random.default_rng(5)
    b1, b2 = rng.standard_normal(n), rng.standard_normal(n)
    s = lambda b: o.sweep(b, None, x_is_zero=True)
    lhs = s(2.5 * b1 + b2)
    # patches at gamma = Re = 1e4 have kappa ~ 1e5-1e7: rounding differences scale with kappa u
    assert np.linalg.norm(lhs - (2.5 * s(b1) + s(b2))) <= 1e-10 * np.linalg.norm(lhs)
    # x_is_zero is bit-identical to sweeping from an explicit +0 vector (b - A 0 = b)
    assert np.array_equal(s(b1), o.sweep(b1, np.zeros(n), x_is_zero=False))


# ---------------- transfer ----------------
def _affine_dofs(m, dim, block, n, rng):
    """DoF values (R-basis functionals) of the affine / lowest-order field that the
    space reproduces exactly, computed from the mesh geometry."""
    X = m["x"][:, :3]
    a = rng.standard_normal(3); Bm = rng.standard_normal((3, 3)); c = rng.standard_normal(3)
    if dim == 2:
        a[2] = 0; Bm[2, :] = 0; Bm[:, 2] = 0
    u = lambda p: a + Bm @ p
    out = np.zeros(n)
    for d in range(n):
        kind, ent, sub = m["dkind"][d], m["dent"][d], m["dsub"][d]
        if kind == 0:                                  # CG1: linear scalar c.x
            out[d] = c[:2] @ X[ent, :2]
        elif kind == 1:                                # NED1 contains a + b x x: use a + c x x
            p, q = X[m["ev"][ent]]
            mid = 0.5 * (p + q)
            out[d] = (a + np.cross(c, mid)) @ (q - p)
        else:
            if dim == 2:
                p, q = X[m["ev"][ent]]
                Av = np.array([q[1] - p[1], -(q[0] - p[0]), 0.0])
                verts = [p, q]
            else:
                p, q, r = X[m["fv"][ent]]
                Av = 0.5 * np.cross(q - p, r - p)
                verts = [p, q, r]
            if block == "vel":                         # BDM1 = full P1: |f| (u.n)(x_a)
                out[d] = u(verts[sub]) @ Av
            else:                                      # RT1 contains a + s x: constant a
                out[d] = a @ Av
    return out


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_prolongation_reproduces_affine_fields(oracle_mod, name):
    """P x_c = x_f for fields the coarse space contains (nested spaces),
    checked on fine DoFs whose entity lies strictly inside the interior coarse cells
    (there every coarse DoF is free, so no boundary constraint intervenes);
    entries are dyadic rationals (R-prol)."""
    cfg = small(name, 8, 2)
    o = make(oracle_mod, cfg)
    mf, mc = o.mesh(1), o.mesh(0)
    P = o.prolongation(1).to_scipy(o.n(0))
    hc = 1.0 / (cfg.N // 2)
    X = mf["x"][:, :cfg.dim]
    inner = np.all((X > hc + 1e-12) & (X < 1 - hc - 1e-12), axis=1)
    rows = []
    for d in range(o.n(1)):
        ent, kind = mf["dent"][d], mf["dkind"][d]
        vs = [ent] if kind == 0 else (mf["ev"][ent] if (kind == 1 or cfg.dim == 2) else mf["fv"][ent])
        if all(inner[v] for v in vs):
            rows.append(d)
    assert len(rows) > 10
    for seed in range(3):
        xc = _affine_dofs(mc, cfg.dim, cfg.block, o.n(0), np.random.default_rng(seed))
        xf = _affine_dofs(mf, cfg.dim, cfg.block, o.n(1), np.random.default_rng(seed))
        got = P @ xc
        assert np.abs(got - xf)[rows].max() <= 1e-12 * np.abs(xf).max()
    Pd = P.toarray()
    assert np.array_equal(Pd * 64, np.round(Pd * 64))


@pytest.mark.parametrize("name", ["c1", "c3", "c4", "c5"])
def test_prolongation_galerkin_identity(oracle_mod, name):
    """For conforming forms the coarse rediscretised operator equals P^T A_f P
    (nested spaces).  E-B is fully conforming (exact w: constant field);
    for the DG velocity form the identity holds for the volume terms: Re -> inf, w = 0."""
    base = small(name, 4, 2)
    wc = [1.0, 0.5] if base.dim == 2 else [1.0, 0.5, -0.3]
    if base.block == "eb":
        cfg = base
        pot = mms.constant_wind_potential(base.dim, base.N, wc)
    else:
        cfg = dataclasses.replace(base, Re=1e14, gamma=3.0)
        pot = draw(base, 0, 0)[0] * 0.0
    o = oracle_mod.Oracle(cfg, pot)
    Af = o.csr(1).to_scipy(); Ac = o.csr(0).to_scipy().toarray()
    P = o.prolongation(1).to_scipy(o.n(0))
    G = (P.T @ Af @ P).toarray()
    assert np.abs(G - Ac).max() <= 1e-11 * np.abs(Ac).max()


def test_restriction_is_transpose(oracle_mod):
    cfg = small("c5", 4, 2)
    o = make(oracle_mod, cfg)
    r = np.random.default_rng(0).standard_normal(o.n(1))
    P = o.prolongation(1).to_scipy(o.n(0))
    rc = o.restrict(r, 1)
    assert np.linalg.norm(rc - P.T @ r) <= 1e-14 * np.linalg.norm(rc)
    ec = np.random.default_rng(1).standard_normal(o.n(0))
    x = np.random.default_rng(2).standard_normal(o.n(1))
    assert np.linalg.norm(o.prolong_add(ec, x, 1) - (x + P @ ec)) <= 1e-14 * np.linalg.norm(x)


# ---------------- V-cycle and GMRES ----------------
def test_vcycle_special_cases(oracle_mod):
    cfg = small("c1", 8, 1)
    o = make(oracle_mod, cfg)
    n = o.n()
    _, b, _ = draw(cfg, n, 0)
    ref = np.linalg.solve(o.csr().to_scipy().toarray(), b)
    assert np.linalg.norm(o.vcycle(b) - ref) <= 1e-12 * np.linalg.norm(ref)    # L = 1: coarse solve
    o2 = make(oracle_mod, CONFIGS["c1"])
    assert np.array_equal(o2.vcycle(np.zeros(o2.n())), np.zeros(o2.n()))       # V(0) = 0
    rng = np.random.default_rng(0)
    b1, b2 = rng.standard_normal(o2.n()), rng.standard_normal(o2.n())
    v = o2.vcycle(3.0 * b1 - b2)
    assert np.linalg.norm(v - (3.0 * o2.vcycle(b1) - o2.vcycle(b2))) <= 1e-12 * np.linalg.norm(v)


def test_lu_exact_on_dyadic_factors():
    """R-lu on A = Q L U with dyadic L (|l_ij| <= 1/2, unit diagonal) and U (power-of-two
    diagonal, small dyadic entries): every elimination and substitution step is exact in
    binary, partial pivoting must pick the unit-l row at every step (so perm recovers Q),
    and the solve must return the integer x it was built from bit for bit.  A dropped
    term, a wrong index or a wrong pivot anywhere gives a different x."""
    from oracle import oracle as om
    rng = np.random.default_rng(11)
    for n in (1, 3, 17, 40):
        L = np.tril(rng.choice([-0.5, -0.25, 0.0, 0.25, 0.5], size=(n, n)), -1) + np.eye(n)
        U = np.triu(rng.choice([-2.0, -1.0, -0.5, 0.5, 1.0, 2.0], size=(n, n)), 1)
        U += np.diag(rng.choice([-4.0, -2.0, 2.0, 4.0, 8.0], size=n))
        Q = rng.permutation(n)
        A = np.empty((n, n))
        A[Q] = L @ U                      # row Q[k] of A is row k of L U
        xt = rng.integers(-9, 10, size=n).astype(float)
        b = A @ xt
        x, lu, perm, st = om.dense_lu_solve(A, b)
        assert st == 0
        assert list(perm) == list(Q)
        assert np.array_equal(np.tril(lu, -1), np.tril(L, -1)) and np.array_equal(np.triu(lu), U)
        assert np.array_equal(x, xt)


@pytest.mark.parametrize("name,N", [("c1", 8), ("c5", 2), ("c3", 8)])
def test_coarse_solve_is_lu_solve(oracle_mod, name, N):
    """SURVEY 8(c.8) "l = 0: return the coarse LU solve" (stand-in for MUMPS): the
    coarse solve is the R-lu solve of the coarse operator -- bit-identical to the dense
    R-lu routine pinned above on the exported operator -- and, against LAPACK's
    getrf/getrs (same method, another rounding order), a backward-stable solve:
    ||A x - b|| <= 4 n u ||A|| ||x|| and ||x - x_lapack|| <= 8 n u kappa(A) ||x||."""
    cfg = small(name, N, 1)
    o = make(oracle_mod, cfg)
    n = o.n()
    A = o.csr().to_scipy().toarray()
    rng = np.random.default_rng(4)
    u = 2.0 ** -53
    kap = np.linalg.cond(A, 2)
    for _ in range(3):
        b = rng.uniform(-1, 1, n)
        x = o.coarse_solve(b)
        assert np.array_equal(x, oracle_mod.dense_lu_solve(A, b)[0])
        nA = np.linalg.norm(A, 2)
        assert np.linalg.norm(A @ x - b) <= 4 * n * u * nA * np.linalg.norm(x)
        ref = sla.lu_solve(sla.lu_factor(A), b)
        assert np.linalg.norm(x - ref) <= 8 * n * u * kap * np.linalg.norm(x)
    e = np.zeros(n)
    assert np.array_equal(o.coarse_solve(e), e)            # A^-1 0 = 0 exactly


def test_vcycle_two_level_definition(oracle_mod):
    """V = S^nu2 (x + P A_c^-1 P^T (b - A S^nu1 0)) composed from the pinned parts."""
    cfg = CONFIGS["c1"]
    o = make(oracle_mod, cfg)
    n = o.n()
    _, b, _ = draw(cfg, n, 3)
    x = o.sweep(b, None, nsweeps=cfg.nu, x_is_zero=True)
    r = o.residual(b, x)
    ec = o.coarse_solve(o.restrict(r))
    x = o.prolong_add(ec, x)
    x = o.sweep(b, x, nsweeps=cfg.nu)
    assert np.array_equal(x, o.vcycle(b))
    Ac = o.csr(0).to_scipy().toarray()
    rc = o.restrict(r)
    assert np.linalg.norm(ec - np.linalg.solve(Ac, rc)) <= 1e-12 * np.linalg.norm(ec)


def test_gmres_exact_preconditioner_one_iteration(oracle_mod):
    """Preconditioner = exact A^-1 (single level => V = direct solve) => 1 iteration."""
    cfg = small("c3", 4, 1)
    o = make(oracle_mod, cfg)
    _, b, _ = draw(cfg, o.n(), 0)
    x, its, hist, conv = o.gmres(b)
    assert conv and its == 1
    A = o.csr().to_scipy().toarray()
    ref = np.linalg.solve(A, b)
    assert np.linalg.norm(x - ref) <= max(1e-10, 10 * np.linalg.cond(A) * 1.1e-16) * np.linalg.norm(ref)


def test_gmres_converges_c1(oracle_mod):
    cfg = CONFIGS["c1"]
    o = make(oracle_mod, cfg)
    _, b, _ = draw(cfg, o.n(), 0)
    x, its, hist, conv = o.gmres(b)
    assert conv and its < 30
    assert np.linalg.norm(b - o.spmv(x)) <= 1.0001e-7 * max(np.linalg.norm(b), 1.0)
    assert np.all(np.diff(hist) <= 1e-12 * hist[0])          # GMRES residual is monotone


# ---------------- kernel decomposition ----------------
@pytest.mark.parametrize("name,N", [("c3", 3), ("c5", 2), ("c2", 3), ("c4", 2)])
def test_kernel_decomposition(oracle_mod, name, N):
    """N = sum_i (V_i cap N) for the kernel N of the semi-definite AL term
    (gamma grad-div for velocity, (1/Rem) div-div C for E-B restricted to B):
    the local kernels of the star patches span the global kernel (dense rank)."""
    base = small(name, N, 1)
    if base.block == "vel":
        o1 = make(oracle_mod, dataclasses.replace(base, gamma=1.0))
        o2 = make(oracle_mod, dataclasses.replace(base, gamma=2.0))
        D = (o2.csr().to_scipy() - o1.csr().to_scipy()).toarray()     # = gamma-part (div, div)
        idx = np.arange(o1.n())
        ptr, dofs, _, _ = o1.patches()
    else:
        o1 = make(oracle_mod, base)
        A = o1.csr().to_scipy().toarray(); nE = o1.info()["nE"]
        D = A[nE:, nE:]
        idx = np.arange(nE, o1.n())
        ptr, dofs, _, _ = o1.patches()
    scale = np.abs(D).max()

    def null(M):
        if M.shape[0] == 0:
            return np.zeros((0, 0))
        u, s, vt = np.linalg.svd(M)
        k = int(np.sum(s > 1e-9 * scale))
        return vt[k:].T

    Ng = null(D)
    pos = {int(g): t for t, g in enumerate(idx)}
    cols = []
    for i in range(len(ptr) - 1):
        loc = [pos[int(d)] for d in dofs[ptr[i]:ptr[i + 1]] if int(d) in pos]
        if not loc:
            continue
        Z = null(D[np.ix_(loc, loc)])
        for z in Z.T:
            v = np.zeros(len(idx)); v[loc] = z
            cols.append(v)
    S = np.array(cols).T
    assert Ng.shape[1] > 0
    assert np.abs(D @ S).max() <= 1e-9 * scale                                  # local kernels lie in N
    assert np.linalg.matrix_rank(S, tol=1e-8) == Ng.shape[1]                    # and span it
