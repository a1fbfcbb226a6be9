"""Pins of the oracle's meshes, numbering and patches (SURVEY §8c.12 "Mesh / numbering").

Every expected value here is a closed form, a brute-force recount from the
exported mesh, or the independent enumeration of SURVEY Appendix A
(tests/golden/appendix_a_counts.json) -- never the oracle's own output.
"""
import json
import os

import numpy as np
import pytest

from paper_2104_14855_b200.workloads import CONFIGS, draw, small

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "appendix_a_counts.json")))


def make(oracle_mod, cfg, nlev=None):
    w, _, _ = draw(cfg, 0, 0)
    return oracle_mod.Oracle(cfg, w, nlev=nlev)


@pytest.mark.parametrize("dim,N", [(2, 1), (2, 2), (2, 7), (3, 1), (3, 2), (3, 5)])
def test_entity_counts_closed_form_and_euler(oracle_mod, dim, N):
    cfg = small("c1" if dim == 2 else "c4", N, 1)
    i = make(oracle_mod, cfg).info()
    if dim == 2:
        assert (i["nv"], i["ne"], i["nc"]) == ((N + 1) ** 2, 3 * N * N + 2 * N, 2 * N * N)
        assert i["nv"] - i["ne"] + i["nc"] == 1                       # Euler characteristic of the disc
        assert i["n"] == (2 * N - 1) ** 2                              # free E-B DoFs
    else:
        assert i["nv"] == (N + 1) ** 3
        assert i["ne"] == 3 * N * (N + 1) ** 2 + 3 * N * N * (N + 1) + N ** 3
        assert i["nf"] == 6 * N * N * (N + 1) + 6 * N ** 3
        assert i["nc"] == 6 * N ** 3
        assert i["nv"] - i["ne"] + i["nf"] - i["nc"] == 1              # Euler characteristic of the ball
        # free E-B DoFs: interior edges (edges not on a boundary face) + interior faces
        ne_b, nf_b = 18 * N * N, 12 * N * N                              # boundary edges / faces (App. A)
        assert i["n"] == (i["ne"] - ne_b) + (i["nf"] - nf_b)


@pytest.mark.parametrize("name,nlev", [("c2", 5), ("c3", 5), ("c4", 4), ("c5", 3)])
def test_appendix_a_counts(oracle_mod, name, nlev):
    rows = GOLDEN[name]
    rows = rows[len(rows) - nlev:]          # finest first; drop levels finer than tested
    N = rows[0][0]
    cfg = small(name, N, nlev)
    o = make(oracle_mod, cfg)
    for lev in range(nlev):
        row = rows[nlev - 1 - lev]
        i = o.info(lev)
        assert row[0] == N >> (nlev - 1 - lev)
        assert (i["n"], i["nnz"]) == (row[1], row[2])
        if row[3] is not None:
            assert (i["npatch"], i["sum_n"], i["sum_n2"]) == (row[3], row[4], row[5])


def _entity_vertices(m, dim, kind, ent):
    if kind == 0:
        return {int(ent)}
    if kind == 1 or dim == 2:
        return set(int(v) for v in m["ev"][ent])
    return set(int(v) for v in m["fv"][ent])


@pytest.mark.parametrize("name,N", [("c1", 3), ("c3", 3), ("c4", 2), ("c5", 2)])
def test_patches_brute_force(oracle_mod, name, N):
    """V_i = {v : supp v in K_i}: brute force over cells.  A free DoF's
    support is the set of cells containing its entity; it lies in star(v) iff
    every such cell contains v."""
    cfg = small(name, N, 1)
    o = make(oracle_mod, cfg)
    m = o.mesh()
    dim = cfg.dim
    ptr, dofs, vert, mult = o.patches()
    cells = [set(int(v) for v in c) for c in m["cv"]]
    n = o.n()
    supp = []
    for d in range(n):
        ev = _entity_vertices(m, dim, m["dkind"][d], m["dent"][d])
        supp.append([c for c, cs in enumerate(cells) if ev <= cs])
    expect = {}
    nv = m["x"].shape[0]
    for v in range(nv):
        ds = [d for d in range(n) if all(v in cells[c] for c in supp[d])]
        if ds:
            expect[v] = ds
    assert list(vert) == sorted(expect)
    for i, v in enumerate(vert):
        assert list(dofs[ptr[i]:ptr[i + 1]]) == expect[int(v)]
    # multiplicities: vertex DoF 1, edge DoF 2, face DoF 3 (R-weights)
    for d in range(n):
        ev = _entity_vertices(m, dim, m["dkind"][d], m["dent"][d])
        assert mult[d] == len(ev)
    # every cell lies in the d+1 stars of its vertices
    cnt = np.zeros(len(cells), int)
    for v in range(nv):
        for c, cs in enumerate(cells):
            cnt[c] += v in cs
    assert np.all(cnt == dim + 1)


@pytest.mark.parametrize("name,size", [("c1", 7), ("c3", 12), ("c4", 50), ("c5", 108)])
def test_interior_star_sizes(oracle_mod, name, size):
    """Interior vertex stars: 2D 6 triangles (7 E-B / 12 BDM DoFs); 3D Kuhn 24 tets,
    14 edges + 36 faces (50 E-B) / 36 faces x 3 (108 BDM)."""
    cfg = small(name, 4, 1)
    ptr, dofs, vert, mult = make(oracle_mod, cfg).patches()
    sizes = np.diff(ptr)
    assert sizes.max() == size
    nint = (cfg.N - 1) ** cfg.dim
    assert np.sum(sizes == size) == nint


def test_vertex_and_cell_numbering(oracle_mod):
    """Vertex (i,j[,k]) has id i + (N+1)(j + (N+1)k) and coordinate lattice/N; 2D
    cells T[2s], T[2s+1] of square s follow the bottom-left -> top-right diagonal;
    3D Kuhn tet p of cube c has the axis-permutation p (lexicographic) walk."""
    N = 3
    o = make(oracle_mod, small("c1", N, 1))
    m = o.mesh()
    for v in range(16):
        i, j = v % (N + 1), v // (N + 1)
        assert np.array_equal(m["x"][v, :2], [i / N, j / N])
    s = 1 + N * 2          # square (1,2)
    vid = lambda i, j: i + (N + 1) * j
    assert list(m["cv"][2 * s]) == sorted([vid(1, 2), vid(2, 2), vid(2, 3)])
    assert list(m["cv"][2 * s + 1]) == sorted([vid(1, 2), vid(2, 3), vid(1, 3)])
    o3 = make(oracle_mod, small("c4", 2, 1))
    m3 = o3.mesh()
    vid3 = lambda i, j, k: i + 3 * (j + 3 * k)
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    c = 1 + 2 * (0 + 2 * 1)  # cube (1,0,1)
    for p, sig in enumerate(perms):
        cur = [1, 0, 1]
        walk = [vid3(*cur)]
        for a in sig:
            cur[a] += 1
            walk.append(vid3(*cur))
        assert list(m3["cv"][6 * c + p]) == sorted(walk)
    # edges and faces: lexicographic order of sorted tuples, each appearing in a cell
    ev = m3["ev"]
    assert np.all(ev[:, 0] < ev[:, 1])
    assert all(tuple(ev[t]) < tuple(ev[t + 1]) for t in range(len(ev) - 1))
    fv = m3["fv"]
    assert all(tuple(fv[t]) < tuple(fv[t + 1]) for t in range(len(fv) - 1))
