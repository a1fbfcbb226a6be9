"""Parity tier P-A (CPU, no GPU): the library's own host setup vs the oracle.

The library (paper_2104_14855_b200/csrc/fe_setup.cpp: closed-form barycentric moments in
double-double, gather-form assembly) and the oracle (oracle/*.c: Gauss quadrature,
scatter-form assembly) build the hierarchy independently.  Bit-exact: free-DoF numbering
(through the CSR pattern), vertex-star patch lists, the prolongation (dyadic rationals,
reading R-prol) and -- against the oracle's exact build (__float128, reading R-exact) --
every operator value.  Against the oracle's fp64 build the values agree to
<= 1e-13 max|row|.
"""
import numpy as np
import pytest

CASES = [("c1", 8, 2), ("c2", 128, 5), ("c3", 32, 4), ("c4", 8, 3), ("c5", 12, 3), ("c5", 6, 2)]


@pytest.fixture(scope="module")
def mh():
    from paper_2104_14855_b200 import build_lib, mhdp
    build_lib.build()
    return mhdp


@pytest.mark.parametrize("name,N,L", CASES, ids=[f"{c}-N{n}L{l}" for c, n, l in CASES])
def test_host_setup_matches_oracle(mh, oracle_mod, name, N, L):
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small(name, N, L)
    w, _, _ = workloads.draw(cfg, 1, seed=2)
    orc = oracle_mod.Oracle(cfg, w)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w)
    assert ctx.num_levels() == L
    for l in range(L):
        A = orc.csr(l)
        rp, ci, v = ctx.csr(l)
        assert np.array_equal(A.rp, rp), f"level {l}: row pointer"
        assert np.array_equal(A.ci, ci), f"level {l}: column pattern"
        rowmax = np.maximum.reduceat(np.abs(A.v), A.rp[:-1])
        scale = np.repeat(rowmax, np.diff(A.rp))
        assert np.max(np.abs(A.v - v) / scale) <= 1e-13, f"level {l}: values"
        if l == 0:
            continue
        ptr_o, dofs_o, verts_o, _ = orc.patches(l)
        ptr_l, dofs_l = ctx.patches(l)
        assert np.array_equal(ptr_o, ptr_l) and np.array_equal(dofs_o, dofs_l), f"level {l}: patches"
        # the vertex of each star (what ESINGULAR reports)
        assert np.array_equal(ctx.patch_vertices(l), verts_o), f"level {l}: patch vertices"
        P = orc.prolongation(l)
        prp, pci, pv = ctx.prolongation(l)
        assert np.array_equal(P.rp, prp) and np.array_equal(P.ci, pci), f"level {l}: prolongation pattern"
        assert np.array_equal(P.v.view(np.uint64), pv.view(np.uint64)), f"level {l}: prolongation values"
        info = ctx.info(l)
        assert info["npatch"] == len(ptr_o) - 1 and info["sum_n"] == len(dofs_o)


EXACT_CASES = [("c1", 8, 2), ("c2", 32, 3), ("c3", 16, 3), ("c4", 4, 2), ("c5", 4, 2)]


@pytest.mark.parametrize("name,N,L", EXACT_CASES, ids=[f"{c}-N{n}L{l}" for c, n, l in EXACT_CASES])
def test_operator_bitexact_vs_exact_oracle(mh, oracle_mod, name, N, L):
    """R-exact: both implementations return, for every entry, the fp64 rounding (through
    the row grid) of the exact discrete bilinear form -- so the operators are identical."""
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small(name, N, L)
    w, _, _ = workloads.draw(cfg, 1, seed=5)
    orc = oracle_mod.Oracle(cfg, w, exact=True)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w)
    for l in range(L):
        A = orc.csr(l)
        rp, ci, v = ctx.csr(l)
        assert np.array_equal(A.rp, rp) and np.array_equal(A.ci, ci)
        diff = np.flatnonzero(A.v.view(np.uint64) != v.view(np.uint64))
        assert diff.size == 0, f"level {l}: {diff.size} entries differ, e.g. {A.v[diff[:3]]} vs {v[diff[:3]]}"


VARIANTS = [("c1", dict(dt=0.01)), ("c3", dict(dt=0.01)), ("c4", dict(picard=1)), ("c5", dict(dt=0.5)),
            ("c4", dict(dt=0.05, picard=1)),
            ("c3", dict(mu=5e-3)), ("c5", dict(mu=5e-3)), ("c5", dict(mu=0.25, dt=0.5))]   # Burman, R-mu


@pytest.mark.parametrize("name,kw", VARIANTS, ids=[f"{c}-{'-'.join(f'{k}{v}' for k, v in kw.items())}" for c, kw in VARIANTS])
def test_next4_variants_bitexact(mh, oracle_mod, name, kw):
    """NEXT-4: transient (eta = 1, (1/dt) mass terms) and Picard (delta = 0) operators
    assembled by the library equal the exact oracle's bit for bit."""
    import dataclasses
    from paper_2104_14855_b200 import workloads
    cfg = dataclasses.replace(workloads.small(name, 4, 2), **kw)
    w, _, _ = workloads.draw(cfg, 1, seed=8)
    orc = oracle_mod.Oracle(cfg, w, exact=True)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w)
    for l in range(2):
        A = orc.csr(l)
        rp, ci, v = ctx.csr(l)
        assert np.array_equal(A.rp, rp) and np.array_equal(A.ci, ci)
        assert np.array_equal(A.v.view(np.uint64), v.view(np.uint64))


@pytest.mark.parametrize("name", ["c3", "c5"])
def test_lorentz_variant_bitexact(mh, oracle_mod, name):
    """NEXT-4 Lorentz term S(u x B^n, v x B^n), transient, S = 1e3: bit-exact."""
    import dataclasses
    from paper_2104_14855_b200 import workloads
    cfg = dataclasses.replace(workloads.small(name, 4, 2), S=1e3, dt=0.1)
    w, _, _ = workloads.draw(cfg, 1, seed=4)
    bn = workloads.magnetic_potential(cfg, 4)
    orc = oracle_mod.Oracle(cfg, w, exact=True, bn=bn)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w, bn=bn)
    for l in range(2):
        A = orc.csr(l)
        assert np.array_equal(A.v.view(np.uint64), ctx.csr(l)[2].view(np.uint64))


def test_gamma_and_curl_entries_bitwise(mh, oracle_mod):
    """The div-div blocks follow the exact single-rounded form of reading R-gamma on both
    sides: on the E-B block the B-B entries (C only) agree bit for bit."""
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c4", 4, 1)
    w, _, _ = workloads.draw(cfg, 1, seed=0)
    orc = oracle_mod.Oracle(cfg, w)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w)
    A = orc.csr()
    rp, ci, v = ctx.csr()
    nE = orc.info()["nE"]
    rows = np.repeat(np.arange(len(rp) - 1), np.diff(rp))
    bb = (rows >= nE) & (ci >= nE)
    assert bb.sum() > 0
    assert np.array_equal(A.v[bb].view(np.uint64), v[bb].view(np.uint64))


def test_appendix_a_counts_full_c5_finest(mh):
    """Counts of the full c5 finest level (tests/golden) from the
    library's own setup: n, nnz, patches, sum n_i, sum n_i^2."""
    import json
    import os
    from paper_2104_14855_b200 import workloads
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a_counts.json")))
    cfg = workloads.small("c5", 24, 1)
    w, _, _ = workloads.draw(cfg, 1, seed=0)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w)
    i = ctx.info(0)
    row = [r for r in gold["c5"] if r[0] == 24][0]
    assert (i["n"], i["nnz"]) == (row[1], row[2])


COUPLED = [(2, 8, 2, dict()), (3, 4, 2, dict()), (2, 4, 2, dict(picard=1, dt=0.1)), (3, 2, 1, dict(dt=0.05))]


@pytest.mark.parametrize("dim,N,L,kw", COUPLED, ids=[f"{d}D-N{n}-{k}" for d, n, l, k in COUPLED])
def test_coupled_operator_bitexact(mh, oracle_mod, dim, N, L, kw):
    """NEXT-3: the coupled 4x4 Newton operator over [u | p | E | B] (Table 1) assembled by
    the library (double-double closed forms) equals the exact oracle's (quadrature in
    __float128), bit for bit, including every coupling block."""
    import dataclasses
    from paper_2104_14855_b200 import workloads
    cfg = dataclasses.replace(workloads.small("c3" if dim == 2 else "c5", N, L), Re=10.0, Rem=5.0, gamma=100.0,
                              S=3.0, **kw)
    w, _, _ = workloads.draw(cfg, 1, 6)
    bn = workloads.magnetic_potential(cfg, 6)
    orc = oracle_mod.CoupledOracle(cfg, w, bn, exact=True)
    lib = mh.Coupled(cfg, w, bn, device=-1)
    assert (lib.nu, lib.np_, lib.nE, lib.nB) == (orc.nu, orc.np_, orc.nE, orc.nB)
    A = orc.csr()
    rp, ci, v = lib.csr()
    assert np.array_equal(A.rp, rp) and np.array_equal(A.ci, ci)
    diff = np.flatnonzero(A.v.view(np.uint64) != v.view(np.uint64))
    assert diff.size == 0, f"{diff.size} entries differ"


K2_CASES = [("c1", 8, 2, dict()), ("c2", 32, 3, dict()), ("c2", 16, 3, dict(picard=1, dt=0.05)),
            ("c2", 64, 4, dict(Rem=7.0)),
            ("c3", 8, 2, dict(sigma=40.0)), ("c3", 32, 4, dict(sigma=40.0, Re=100.0, gamma=1e4)),
            ("c3", 16, 3, dict(sigma=40.0, dt=0.05)), ("c3-lorentz", 16, 2, dict(sigma=40.0, S=30.0)),
            ("c4", 4, 2, dict()),                                   # 3D NED1_2 x RT2, 280-DoF stars
            ("c5", 2, 1, dict(sigma=40.0, dt=0.05, gamma=1e4))]     # 3D BDM2, 360-DoF stars


@pytest.mark.parametrize("name,N,L,kw", K2_CASES, ids=[f"{c}-N{n}L{l}-{k}" for c, n, l, k in K2_CASES])
def test_k2_host_setup_bitexact_vs_exact_oracle(mh, oracle_mod, name, N, L, kw):
    """NEXT-2 (k = 2): 2D CG2 x RT2 E-B and BDM2 velocity blocks, 3D NED1_2 x RT2 and BDM2.
    Numbering, patches, prolongation (R-prol2) and operator values of the library
    (closed-form barycentric, facet and edge integrals in double-double; {lam_a psi_q} /
    {lam_a lam_b e_r} / Arnold-Falk-Winther primal bases) equal the oracle's exact build
    (quadrature in __float128, monomial primal bases) bit for bit on every level."""
    import dataclasses
    from paper_2104_14855_b200 import workloads
    lorentz = name.endswith("-lorentz")
    cfg = dataclasses.replace(workloads.small(name.replace("-lorentz", ""), N, L), degree=2, **kw)
    w, _, _ = workloads.draw(cfg, 1, seed=2)
    bn = workloads.magnetic_potential(cfg, 2) if lorentz else None
    orc = oracle_mod.Oracle(cfg, w, exact=True, bn=bn)
    ctx = mh.Context(-1)
    ctx.assemble(cfg, w, bn=bn)
    for l in range(L):
        A = orc.csr(l)
        rp, ci, v = ctx.csr(l)
        assert np.array_equal(A.rp, rp) and np.array_equal(A.ci, ci), f"level {l}: pattern"
        diff = np.flatnonzero(A.v.view(np.uint64) != v.view(np.uint64))
        assert diff.size == 0, f"level {l}: {diff.size} values differ"
        if l == 0:
            continue
        ptr_o, dofs_o, verts_o, _ = orc.patches(l)
        ptr_l, dofs_l = ctx.patches(l)
        assert np.array_equal(ptr_o, ptr_l) and np.array_equal(dofs_o, dofs_l), f"level {l}: patches"
        # the vertex of each star (what ESINGULAR reports)
        assert np.array_equal(ctx.patch_vertices(l), verts_o), f"level {l}: patch vertices"
        P = orc.prolongation(l)
        prp, pci, pv = ctx.prolongation(l)
        assert np.array_equal(P.rp, prp) and np.array_equal(P.ci, pci), f"level {l}: prolongation pattern"
        assert np.array_equal(P.v.view(np.uint64), pv.view(np.uint64)), f"level {l}: prolongation values"


def test_coupled_rejects_degree_2(mh):
    """NEXT-3 is built at k = 1 only: a k = 2 coupled system is refused (include/mhdp.h)."""
    import dataclasses
    from paper_2104_14855_b200 import workloads
    cfg = dataclasses.replace(workloads.small("c3", 4, 1), degree=2, sigma=40.0)
    w, _, _ = workloads.draw(cfg, 1, 0)
    with pytest.raises(mh.MhdpError):
        mh.Coupled(cfg, w, None, device=-1)
