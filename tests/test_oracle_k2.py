"""Oracle pins for NEXT-2: element degree k = 2 for the 2D E-B block, E in CG2 and
B in RT2 (complex CG2 -> RT2 -> DG1), reading R-basis2 of DESIGN.md.

Pins (none re-types the oracle's formulas):
* DoF counts against closed forms; star patches against a brute-force support test
  (V_i = {v : supp v in K_i});
* DoF duality N_i(phi_j) = delta_ij with the global functionals of the fine-level
  prolongation code (written apart from the local-basis construction);
* manufactured solutions: L2 rates 3 (CG2 E) and 2 (RT2 B) -- k = 1 gives 2 and 1 --
  for the Newton, transient and Picard variants;
* the discrete complex: div(vcurl CG2) = 0, read off the assembled blocks alone;
* the Galerkin identity A_c = P^T A_f P for the conforming E-B forms (nested spaces);
* Picard antisymmetry of the E-B coupling, symmetric positive mass;
* Re_m-robust star multigrid for Picard.
"""
import dataclasses

import numpy as np
import pytest

import mms
from paper_2104_14855_b200.workloads import CONFIGS, draw, small


def _cfg(N, L, **kw):
    base = dict(degree=2)
    base.update(kw)
    return dataclasses.replace(small("c1", N, L), **base)


def _orc(oracle_mod, cfg, exact=False, wc=None):
    pot = draw(cfg, 1, 0)[0] if wc is None else mms.constant_wind_potential(2, cfg.N, wc)
    return oracle_mod.Oracle(cfg, pot, exact=exact)


@pytest.mark.parametrize("N", [2, 5, 8])
def test_k2_dof_counts_closed_form(oracle_mod, N):
    """Free E DoFs: interior vertices + interior edges = (N-1)^2 + 3N^2 - 2N; free B DoFs:
    2 per interior edge + 2 per cell = 10N^2 - 4N (E = 0, B.n = 0 on the boundary)."""
    o = _orc(oracle_mod, _cfg(N, 1))
    i = o.info()
    assert i["nE"] == (N - 1) ** 2 + 3 * N * N - 2 * N
    assert i["n"] - i["nE"] == 10 * N * N - 4 * N


def test_k2_patches_brute_force(oracle_mod):
    """A free DoF belongs to the star of vertex v iff every cell of its support contains v;
    the support of a DoF is the set of cells containing its entity.  Interior stars: 1
    vertex + 6 edge E DoFs, 6 x 2 edge + 6 x 2 cell B DoFs = 31."""
    o = _orc(oracle_mod, _cfg(6, 1))
    m = o.mesh()
    cv, ev = m["cv"], m["ev"]
    cells_of_vertex = [set() for _ in range(m["x"].shape[0])]
    for c, vs in enumerate(cv):
        for v in vs:
            cells_of_vertex[v].add(c)
    support = []
    for d in range(o.n()):
        k, e = m["dkind"][d], m["dent"][d]
        if k == 0:
            support.append(cells_of_vertex[e])
        elif k in (1, 2):
            support.append(cells_of_vertex[ev[e][0]] & cells_of_vertex[ev[e][1]])
        else:
            support.append({e})
    ptr, dofs, vert, _ = o.patches()
    got = {int(vert[i]): sorted(dofs[ptr[i]:ptr[i + 1]].tolist()) for i in range(len(vert))}
    want = {}
    for v in range(m["x"].shape[0]):
        s = sorted(d for d in range(o.n()) if support[d] <= cells_of_vertex[v])
        if s:
            want[v] = s
    assert got == want
    assert max(len(s) for s in want.values()) == 31


def test_k2_duality(oracle_mod):
    o = _orc(oracle_mod, _cfg(4, 2))
    assert o.duality_error() <= 1e-13 and o.duality_error(0) <= 1e-13
    oe = _orc(oracle_mod, _cfg(4, 2), exact=True)
    assert oe.duality_error() <= 1e-28


@pytest.mark.parametrize("kw", [dict(), dict(div_free_B=True), dict(dt=0.05), dict(picard=1)],
                         ids=["newton", "div-free-B", "transient", "picard"])
def test_k2_mms_rates(oracle_mod, kw):
    """L2 rates 3 (E in CG2) and 2 (B in RT2), Re_m = 1, constant w (measured 2.999 / 1.998)."""
    wc = [1.0, 0.5]
    dt, pic = kw.get("dt", 0.0), kw.get("picard", 0)
    base = dataclasses.replace(CONFIGS["c1"], Re=1.0, Rem=1.0, gamma=1.0, levels=1, dt=dt, picard=pic, degree=2)
    fs, ex = mms.eb_fields(2, 1.0, wc, **kw)
    errs = []
    for N in (16, 32):
        cfg = dataclasses.replace(base, N=N)
        errs.append(mms.solve_and_error(oracle_mod.Oracle(cfg, mms.constant_wind_potential(2, N, wc)), fs, ex))
    r = np.log(errs[0] / errs[1]) / np.log(2.0)
    assert r[0] >= 2.9 and min(r[1:]) >= 1.95, r


def test_k2_complex_div_vcurl_zero(oracle_mod):
    """vcurl CG2 lies in RT2 with zero divergence.  From the assembled blocks only:
    with BB(dt) = M_B / dt + C / Re_m, the B-E block is (vcurl E, C) = M_B D with D the RT2
    coefficients of vcurl E, so C M_B^-1 (B-E block) must vanish."""
    cfg = _cfg(4, 1, Rem=1.0, picard=1)
    A1 = _orc(oracle_mod, dataclasses.replace(cfg, dt=1.0)).csr().to_scipy().toarray()
    A2 = _orc(oracle_mod, dataclasses.replace(cfg, dt=0.5)).csr().to_scipy().toarray()
    nE = _orc(oracle_mod, cfg).info()["nE"]
    MB = A2[nE:, nE:] - A1[nE:, nE:]
    C = 2 * A1[nE:, nE:] - A2[nE:, nE:]
    BE = A1[nE:, :nE]
    D = np.linalg.solve(MB, BE)
    assert np.abs(C @ D).max() <= 1e-10 * np.abs(C).max() * np.abs(D).max()
    assert np.abs(C).max() > 1 and np.abs(D).max() > 0.1
    # the mass is symmetric positive definite
    assert np.allclose(MB, MB.T, rtol=0, atol=1e-13 * np.abs(MB).max())
    assert np.linalg.eigvalsh(0.5 * (MB + MB.T)).min() > 0


def test_k2_picard_coupling_antisymmetry(oracle_mod):
    """Picard: E-row coupling -(1/Re_m)(B, vcurl F) = -(1/Re_m) (B-E block)^T; the E-E block
    is the CG2 mass (symmetric positive definite)."""
    rem = 4.0
    o = _orc(oracle_mod, _cfg(4, 1, Rem=rem, picard=1))
    A = o.csr().to_scipy().toarray()
    nE = o.info()["nE"]
    EB, BE = A[:nE, nE:], A[nE:, :nE]
    assert np.abs(EB + BE.T / rem).max() <= 1e-13 * np.abs(BE).max()
    EE = A[:nE, :nE]
    assert np.allclose(EE, EE.T, rtol=0, atol=1e-14 * np.abs(EE).max())
    assert np.linalg.eigvalsh(EE).min() > 0


def test_k2_galerkin_identity(oracle_mod):
    """Conforming E-B forms with an exactly nested (constant) w: the rediscretised coarse
    operator equals P^T A_f P (R-prol), including the u^n x B Newton term."""
    o = _orc(oracle_mod, _cfg(4, 2, Rem=2.0), wc=[1.0, 0.5])
    Af = o.csr(1).to_scipy()
    Ac = o.csr(0).to_scipy().toarray()
    P = o.prolongation(1).to_scipy(o.n(0))
    G = (P.T @ Af @ P).toarray()
    assert np.abs(G - Ac).max() <= 1e-12 * np.abs(Ac).max()


def test_k2_prolongation_exact_build_agrees(oracle_mod):
    """The prolongation and operators of the fp64 and __float128 builds agree to rounding
    (the exact build is the parity reference)."""
    cfg = _cfg(4, 2)
    a, b = _orc(oracle_mod, cfg), _orc(oracle_mod, cfg, exact=True)
    Pa, Pb = a.prolongation(1), b.prolongation(1)
    assert np.array_equal(Pa.rp, Pb.rp) and np.array_equal(Pa.ci, Pb.ci)
    assert np.abs(Pa.v - Pb.v).max() <= 1e-14
    Aa, Ab = a.csr(), b.csr()
    assert np.abs(Aa.v - Ab.v).max() <= 1e-12 * np.abs(Ab.v).max()


def test_k2_picard_multigrid_rem_robust(oracle_mod):
    """Star multigrid on the k = 2 Picard E-B block: FGMRES(GMRES(6)-smoothed V) counts
    bounded for Re_m = 10 ... 1e4 (measured 4)."""
    its = []
    for rem in (10.0, 1e2, 1e3, 1e4):
        cfg = _cfg(32, 4, Re=rem, Rem=rem, picard=1)
        o = _orc(oracle_mod, cfg)
        o.set_smoother("gmres", 6)
        b = np.random.default_rng(3).standard_normal(o.n())
        _, k, _, conv = o.fgmres(b, maxit=40)
        its.append(k if conv else None)
    assert None not in its and max(its) <= 8, its


# ---------------- k = 2 AL velocity block: BDM2, sigma = 10 k^2 = 40 ----------------
def _vcfg(N, L, **kw):
    base = dict(degree=2, sigma=40.0)
    base.update(kw)
    return dataclasses.replace(small("c3", N, L), **base)


@pytest.mark.parametrize("N", [2, 5, 8])
def test_k2_velocity_counts(oracle_mod, N):
    """BDM2: 3 DoFs per interior edge + 3 per cell = 3(3N^2 - 2N) + 6N^2 = 15N^2 - 6N."""
    o = oracle_mod.Oracle(_vcfg(N, 1), draw(_vcfg(N, 1), 1, 0)[0])
    assert o.n() == 15 * N * N - 6 * N


def test_k2_velocity_patches_brute_force(oracle_mod):
    """Star of v = DoFs whose support (cells of the entity) lies in the cells around v;
    interior stars: 6 edges x 3 + 6 cells x 3 = 36 (the BDM2 star of P:575 Figure 2)."""
    cfg = _vcfg(6, 1)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    m = o.mesh()
    cv, ev = m["cv"], m["ev"]
    cells_of_vertex = [set() for _ in range(m["x"].shape[0])]
    for c, vs in enumerate(cv):
        for v in vs:
            cells_of_vertex[v].add(c)
    support = []
    for d in range(o.n()):
        k, e = m["dkind"][d], m["dent"][d]
        support.append(cells_of_vertex[ev[e][0]] & cells_of_vertex[ev[e][1]] if k == 2 else {e})
    ptr, dofs, vert, _ = o.patches()
    got = {int(vert[i]): sorted(dofs[ptr[i]:ptr[i + 1]].tolist()) for i in range(len(vert))}
    want = {v: sorted(d for d in range(o.n()) if support[d] <= cells_of_vertex[v]) for v in range(m["x"].shape[0])}
    want = {v: s for v, s in want.items() if s}
    assert got == want and max(len(s) for s in want.values()) == 36


def test_k2_velocity_duality(oracle_mod):
    cfg = _vcfg(4, 2)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    assert o.duality_error() <= 1e-12 and o.duality_error(0) <= 1e-12
    oe = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0], exact=True)
    assert oe.duality_error() <= 1e-28


@pytest.mark.parametrize("kw", [dict(), dict(dt=0.05)], ids=["steady", "transient"])
def test_k2_velocity_mms_rate(oracle_mod, kw):
    """BDM2 with SIPG (sigma = 40): L2 rate 3 for u (k = 1 gives 2); measured 3.05 / 3.03."""
    wc = [1.0, 0.5]
    base = dataclasses.replace(CONFIGS["c1"], block="vel", Re=1.0, Rem=1.0, gamma=1.0, levels=1, degree=2,
                               sigma=40.0, **kw)
    fs, ex = mms.vel_fields(2, 1.0, wc, **kw)
    errs = []
    for N in (16, 32):
        cfg = dataclasses.replace(base, N=N)
        errs.append(mms.solve_and_error(oracle_mod.Oracle(cfg, mms.constant_wind_potential(2, N, wc)), fs, ex))
    r = np.log(errs[0] / errs[1]) / np.log(2.0)
    assert r.min() >= 2.9, r


def test_k2_velocity_symmetry_and_advection_coercive(oracle_mod):
    """Without advection the BDM2 operator (2/Re eps:eps + SIPG + gamma div div) is
    symmetric; the upwind advection adds a positive semi-definite symmetric part."""
    cfg = _vcfg(4, 1, Re=3.0, gamma=7.0)
    w = draw(cfg, 1, 0)[0]
    A0 = oracle_mod.Oracle(cfg, w * 0.0).csr().to_scipy().toarray()
    A1 = oracle_mod.Oracle(cfg, w).csr().to_scipy().toarray()
    assert np.abs(A0 - A0.T).max() <= 1e-13 * np.abs(A0).max()
    assert np.linalg.eigvalsh(0.5 * (A0 + A0.T)).min() > 0
    D = A1 - A0
    assert np.abs(D).max() > 0
    assert np.linalg.eigvalsh(0.5 * (D + D.T)).min() >= -1e-10 * np.abs(D).max()


def test_k2_velocity_galerkin_identity_volume_terms(oracle_mod):
    """Nested BDM2 spaces: the conforming gamma (div u, div v) term satisfies
    A_c = P^T A_f P (Re -> inf removes the DG terms, w = 0)."""
    cfg = _vcfg(4, 2, Re=1e14, gamma=3.0)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0] * 0.0)
    Af = o.csr(1).to_scipy()
    Ac = o.csr(0).to_scipy().toarray()
    P = o.prolongation(1).to_scipy(o.n(0))
    assert np.abs((P.T @ Af @ P).toarray() - Ac).max() <= 1e-11 * np.abs(Ac).max()


def test_k2_velocity_multigrid_gamma_robust(oracle_mod):
    """Star patches capture the kernel of div at k = 2 (div-free BDM2 = vcurl CG3, every
    CG3 basis function lives in a star), and with the uniform weight of R-weights2 every
    local kernel correction stays in the kernel: FGMRES(GMRES(6)-smoothed V) counts flat
    for gamma = 1e2 ... 1e8 (measured 7-8); point-Jacobi patches break down."""
    its = []
    for g in (1e2, 1e4, 1e6, 1e8):
        cfg = _vcfg(16, 3, Re=1.0, gamma=g)
        o = oracle_mod.Oracle(cfg, draw(cfg, 1, 6)[0])
        o.set_smoother("gmres", 6)
        b = np.random.default_rng(3).standard_normal(o.n())
        _, k, _, conv = o.fgmres(b, maxit=60)
        its.append(k if conv else None)
    assert None not in its and max(its) <= 10 and max(its) - min(its) <= 1, its
    ctrl = []
    for g in (1e2, 1e6):
        cfg = _vcfg(16, 3, Re=1.0, gamma=g)
        o = oracle_mod.Oracle(cfg, draw(cfg, 1, 6)[0])
        o.set_smoother("gmres", 6)
        for lev in range(1, o.nlev):
            n = o.csr(lev).rp.size - 1
            o.set_patches(np.arange(n + 1), np.arange(n), lev)
        b = np.random.default_rng(3).standard_normal(o.n())
        _, k, _, conv = o.fgmres(b, maxit=60)
        ctrl.append(k if conv else None)
    assert ctrl[1] is None or (ctrl[0] is not None and ctrl[1] >= ctrl[0] + 10), ctrl


# ---------------- k = 2 in 3D, E-B block: NED1_2 x RT2 ----------------
def _c4k2(N, L, **kw):
    base = dict(degree=2)
    base.update(kw)
    return dataclasses.replace(small("c4", N, L), **base)


def test_k2_3d_counts_from_k1_entities(oracle_mod):
    """NED1_2: 2 DoFs per free edge + 2 per interior face; RT2: 3 per interior face + 3 per
    cell -- read against the k = 1 space on the same mesh (free edges, interior faces)."""
    N = 3
    cfg1 = dataclasses.replace(small("c4", N, 1))
    o1 = oracle_mod.Oracle(cfg1, draw(cfg1, 1, 0)[0])
    i1 = o1.info()
    ne_free, nf_int = i1["nE"], i1["n"] - i1["nE"]
    o2 = oracle_mod.Oracle(_c4k2(N, 1), draw(_c4k2(N, 1), 1, 0)[0])
    i2 = o2.info()
    assert i2["nE"] == 2 * ne_free + 2 * nf_int
    assert i2["n"] - i2["nE"] == 3 * nf_int + 3 * 6 * N ** 3


def test_k2_3d_duality_and_stars(oracle_mod):
    cfg = _c4k2(4, 2)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    assert o.duality_error() <= 1e-12 and o.duality_error(0) <= 1e-12
    ptr, _, _, _ = o.patches()
    assert np.diff(ptr).max() == 280       # 14 edges x 2 + 36 faces x (2 + 3) + 24 cells x 3


@pytest.mark.parametrize("pic", [0, 1], ids=["newton", "picard"])
def test_k2_3d_mms_rates(oracle_mod, pic):
    """NED1_2 E and RT2 B: L2 rate 2 (k = 1: rate 1); measured 1.86 / 1.92 at N = 2 -> 4,
    1.95 / 1.98 at 4 -> 8."""
    wc = [1.0, 0.5, -0.3]
    base = dataclasses.replace(CONFIGS["c4"], Re=1.0, Rem=1.0, gamma=1.0, levels=1, picard=pic, degree=2)
    fs, ex = mms.eb_fields(3, 1.0, wc, picard=pic)
    errs = []
    for N in (2, 4):
        cfg = dataclasses.replace(base, N=N)
        errs.append(mms.solve_and_error(oracle_mod.Oracle(cfg, mms.constant_wind_potential(3, N, wc)), fs, ex))
    r = np.log(errs[0] / errs[1]) / np.log(2.0)
    assert r.min() >= 1.8, r


def test_k2_3d_complex_div_curl_zero(oracle_mod):
    """curl NED1_2 lies in RT2 with zero divergence: C M_B^-1 (B-E block) = 0 from the
    assembled blocks (as the 2D pin)."""
    cfg = _c4k2(2, 1, Rem=1.0, picard=1)
    A1 = _orc(oracle_mod, dataclasses.replace(cfg, dt=1.0)).csr().to_scipy().toarray()
    A2 = _orc(oracle_mod, dataclasses.replace(cfg, dt=0.5)).csr().to_scipy().toarray()
    nE = _orc(oracle_mod, cfg).info()["nE"]
    MB = A2[nE:, nE:] - A1[nE:, nE:]
    C = 2 * A1[nE:, nE:] - A2[nE:, nE:]
    D = np.linalg.solve(MB, A1[nE:, :nE])
    assert np.abs(C @ D).max() <= 1e-10 * np.abs(C).max() * np.abs(D).max()
    assert np.abs(D).max() > 0.1


def test_k2_3d_galerkin_identity(oracle_mod):
    """Nested NED1_2 x RT2 spaces with a constant w: A_c = P^T A_f P (R-prol2)."""
    cfg = _c4k2(4, 2, Rem=2.0)
    o = oracle_mod.Oracle(cfg, mms.constant_wind_potential(3, 4, [1.0, 0.5, -0.3]))
    Af = o.csr(1).to_scipy()
    Ac = o.csr(0).to_scipy().toarray()
    P = o.prolongation(1).to_scipy(o.n(0))
    assert np.abs((P.T @ Af @ P).toarray() - Ac).max() <= 1e-11 * np.abs(Ac).max()


def test_k2_3d_picard_multigrid(oracle_mod):
    """Star multigrid on the 3D k = 2 Picard E-B block (280-DoF stars): FGMRES(GMRES(6)-
    smoothed V) converges in a handful of iterations for Re_m = 10 and 1e3."""
    its = []
    for rem in (10.0, 1e3):
        cfg = _c4k2(4, 2, Re=rem, Rem=rem, picard=1)
        o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
        o.set_smoother("gmres", 6)
        b = np.random.default_rng(3).standard_normal(o.n())
        _, k, _, conv = o.fgmres(b, maxit=40)
        its.append(k if conv else None)
    assert None not in its and max(its) <= 10, its


# ---------------- k = 2 in 3D, AL velocity block: BDM2, sigma = 40 ----------------
def _v3(N, L, **kw):
    base = dict(degree=2, sigma=40.0)
    base.update(kw)
    return dataclasses.replace(small("c5", N, L), **base)


@pytest.mark.parametrize("N", [2, 3])
def test_k2_3d_velocity_counts(oracle_mod, N):
    """BDM2 on tetrahedra: 6 DoFs per interior face (P2 normal traces) + 6 per cell;
    interior faces 12N^3 - 6N^2, cells 6N^3, so n = 108N^3 - 36N^2.  An interior star has
    36 faces x 6 + 24 cells x 6 = 360 DoFs ("3D BDM2 star ~ 360")."""
    cfg = _v3(N, 1)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    assert o.n() == 108 * N ** 3 - 36 * N ** 2
    assert np.diff(o.patches()[0]).max() == 360


def test_k2_3d_velocity_patches_brute_force(oracle_mod):
    """Star of v = DoFs whose support (the cells of the DoF's face or cell) lies in the
    cells around v, from the mesh alone."""
    cfg = _v3(3, 1)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    m = o.mesh()
    cells_of_vertex = [set() for _ in range(m["x"].shape[0])]
    for c, vs in enumerate(m["cv"]):
        for v in vs:
            cells_of_vertex[v].add(c)
    support = []
    for d in range(o.n()):
        k, e = m["dkind"][d], m["dent"][d]
        if k == 2:
            a, b, c = m["fv"][e]
            support.append(cells_of_vertex[a] & cells_of_vertex[b] & cells_of_vertex[c])
        else:
            support.append({e})
    ptr, dofs, vert, _ = o.patches()
    got = {int(vert[i]): sorted(dofs[ptr[i]:ptr[i + 1]].tolist()) for i in range(len(vert))}
    want = {v: sorted(d for d in range(o.n()) if support[d] <= cells_of_vertex[v]) for v in range(m["x"].shape[0])}
    assert got == {v: s for v, s in want.items() if s}


def test_k2_3d_velocity_duality(oracle_mod):
    cfg = _v3(4, 2)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
    assert o.duality_error() <= 1e-12 and o.duality_error(0) <= 1e-12
    cfg = _v3(2, 1)
    assert oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0], exact=True).duality_error() <= 1e-28


def test_k2_3d_velocity_mms_rate(oracle_mod):
    """BDM2 with SIPG (sigma = 40) in 3D: L2 rate 3 for u (k = 1: 2); measured 3.05 at
    N = 3 -> 6 (2.78 at 2 -> 4, pre-asymptotic)."""
    wc = [1.0, 0.5, -0.3]
    base = dataclasses.replace(CONFIGS["c5"], Re=1.0, Rem=1.0, S=1.0, gamma=1.0, levels=1, degree=2, sigma=40.0)
    fs, ex = mms.vel_fields(3, 1.0, wc)
    errs = [mms.solve_and_error(oracle_mod.Oracle(dataclasses.replace(base, N=N),
                                                  mms.constant_wind_potential(3, N, wc)), fs, ex) for N in (3, 6)]
    r = np.log(errs[0] / errs[1]) / np.log(2.0)
    assert r.min() >= 2.9, r


def test_k2_3d_velocity_symmetry_and_advection_coercive(oracle_mod):
    """Without advection the 3D BDM2 operator is symmetric positive definite; the upwind
    advection adds a positive semi-definite symmetric part."""
    cfg = _v3(2, 1, Re=3.0, gamma=7.0)
    w = draw(cfg, 1, 0)[0]
    A0 = oracle_mod.Oracle(cfg, w * 0.0).csr().to_scipy().toarray()
    A1 = oracle_mod.Oracle(cfg, w).csr().to_scipy().toarray()
    assert np.abs(A0 - A0.T).max() <= 1e-13 * np.abs(A0).max()
    assert np.linalg.eigvalsh(0.5 * (A0 + A0.T)).min() > 0
    D = A1 - A0
    assert np.abs(D).max() > 0
    assert np.linalg.eigvalsh(0.5 * (D + D.T)).min() >= -1e-10 * np.abs(D).max()


def test_k2_3d_velocity_galerkin_identity_volume_terms(oracle_mod):
    """Nested 3D BDM2 spaces: the conforming gamma (div u, div v) term satisfies
    A_c = P^T A_f P (Re -> inf removes the DG terms, w = 0); measured 8e-13."""
    cfg = _v3(4, 2, Re=1e14, gamma=3.0)
    o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0] * 0.0)
    Af = o.csr(1).to_scipy()
    Ac = o.csr(0).to_scipy().toarray()
    P = o.prolongation(1).to_scipy(o.n(0))
    assert np.abs((P.T @ Af @ P).toarray() - Ac).max() <= 1e-11 * np.abs(Ac).max()


def test_k2_3d_velocity_multigrid_gamma_robust(oracle_mod):
    """3D BDM2 star multigrid (360-DoF stars): FGMRES(GMRES(6)-smoothed V) counts do not
    grow with gamma; point-Jacobi patches do not converge."""
    its, ctrl = [], []
    for g in (1e2, 1e6):
        cfg = _v3(4, 2, Re=1.0, gamma=g)
        o = oracle_mod.Oracle(cfg, draw(cfg, 1, 0)[0])
        o.set_smoother("gmres", 6)
        b = np.random.default_rng(0).uniform(-1, 1, o.n())
        _, k, _, conv = o.fgmres(b, maxit=40)
        its.append(k if conv else None)
        o.set_patches(np.arange(o.n(1) + 1, dtype=np.int64), np.arange(o.n(1), dtype=np.int32), 1)
        _, k, _, conv = o.fgmres(b, maxit=40)
        ctrl.append(k if conv else None)
    assert None not in its and max(its) - min(its) <= 1 and max(its) <= 15, its
    assert ctrl == [None, None], ctrl
