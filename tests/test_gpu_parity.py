"""GPU parity, tier P-B (the north-star criterion): the LIBRARY's own setup + CUDA path
against the ORACLE's own setup + CPU path, on the same seeded inputs.

The oracle runs its exact build (reading R-exact), whose operators are bit-identical to
the library's (test_library_host.py); every later step is order-defined (R-order), so
the expected result is BIT-EXACT.  The north-star criterion -- relative l2 <= 1e-10
after one Schwarz sweep (x0 = 0, which skips K1, and x0 = U(-1,1)) and after one
V-cycle, GMRES(V) counts within +-1 -- is asserted as well.  Full sizes for c1 and c2,
reduced hierarchies of c3-c5; the full-size c3, c4 and c5 sweeps (the launch
configuration bench.py times for c5) are checked on sampled DoFs that the oracle
recomputes one by one from a masked assembly.
"""
import numpy as np
import pytest

from gpu_helpers import cuda_vec, host, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10
CASES = [("c1", None, None, 0), ("c1", None, None, 1), ("c1", None, None, 2), ("c2", None, None, 0),
         ("c3", 64, 4, 0), ("c4", 16, 3, 0), ("c5", 6, 2, 0), ("c5", 8, 2, 1),
         ("c4-transient-picard", 8, 2, 0), ("c5-transient", 6, 2, 2), ("c5-lorentz", 6, 2, 3),
         ("c1-k2", None, None, 0), ("c2-k2", 64, 4, 1), ("c2-k2-transient-picard", 32, 3, 2),   # NEXT-2
         ("c3-k2", 32, 4, 0), ("c3-k2-transient", 16, 3, 1), ("c3-k2-lorentz", 16, 3, 2),
         ("c4-k2", 4, 2, 0), ("c4-k2-transient-picard", 4, 2, 1), ("c5-k2", 4, 2, 0),      # 3D k = 2
         ("c3-burman", 32, 4, 0), ("c5-burman", 6, 2, 1)]                                   # R-mu


def _setup(oracle_mod, name, N, L, seed):
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    import dataclasses
    variant = {}
    if "-k2" in name:                                                    # NEXT-2: k = 2
        name = name.replace("-k2", "")
        variant["degree"] = 2
        if name.startswith("c3") or name.startswith("c5"):
            variant["sigma"] = 40.0                                      # 10 k^2
    if name.endswith("-burman"):                                          # P:190-194, R-mu
        name = name.split("-")[0]
        variant["mu"] = 5e-3
    lorentz = name.endswith("-lorentz")
    if name.endswith("-transient-picard"):
        name = name.split("-")[0]
        variant.update(dt=0.05, picard=1)                                # NEXT-4
    elif name.endswith("-transient"):
        name = name.split("-")[0]
        variant.update(dt=0.01)
    elif lorentz:
        name = name.split("-")[0]
        variant.update(S=1e3, dt=0.1)
    cfg = workloads.CONFIGS[name] if N is None else workloads.small(name, N, L)
    cfg = dataclasses.replace(cfg, **variant)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w0, _, _ = workloads.draw(cfg, 1, seed)
    bn = workloads.magnetic_potential(cfg, seed) if lorentz else None
    ctx.assemble(cfg, w0, bn=bn)
    n = ctx.n()
    w, b, x0 = workloads.draw(cfg, n, seed)
    assert np.array_equal(w, w0)
    ctx.setup()
    orc = oracle_mod.Oracle(cfg, w, exact=True, bn=bn)
    assert orc.n() == n
    return cfg, ctx, orc, b, x0


def _same(got, ref):
    assert rel_l2(got, ref) <= TOL
    assert np.array_equal(np.asarray(got).view(np.uint64), np.asarray(ref).view(np.uint64)), \
        f"not bit-exact: rel l2 {rel_l2(got, ref):.3e}"


@pytest.fixture(scope="module", params=CASES, ids=[f"{c}-{n or 'full'}-s{s}" for c, n, l, s in CASES])
def pb(request, oracle_mod):
    name, N, L, seed = request.param
    return _setup(oracle_mod, name, N, L, seed)


def test_sweep_from_zero(pb):
    cfg, ctx, orc, b, x0 = pb
    xo = orc.sweep(b, np.zeros_like(b), x_is_zero=True)
    xg = cuda_vec(np.zeros_like(b))
    ctx.smooth(cuda_vec(b), xg, nsweeps=1, x_is_zero=True)
    _same(host(xg), xo)


def test_sweep_from_random(pb):
    cfg, ctx, orc, b, x0 = pb
    xo = orc.sweep(b, x0, nsweeps=1)
    xg = cuda_vec(x0)
    ctx.smooth(cuda_vec(b), xg, nsweeps=1)
    _same(host(xg), xo)


def test_vcycle(pb):
    import torch
    cfg, ctx, orc, b, x0 = pb
    xo = orc.vcycle(b)
    xg = torch.empty(len(b), dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(b), xg)
    _same(host(xg), xo)


# GMRES(V) maxit per case: 200 where the oracle converges only after 80 (c3 N64 L4: 154,
# c5 N8 L2: 136 iterations), else 80
MAXIT = {("c3", 64): 200, ("c5", 8): 200}


def test_gmres_iteration_count(pb, request):
    """a8 (c.9): GMRES(V) counts within +-1 where either side converges, and
    convergence exactly where the oracle converges; where either side stops at maxit, the
    residual histories are compared instead (<= 1e-6 relative per iteration
    over the first 20 iterations).  Both sides run the same order-defined iteration, so
    the histories are also expected bit for bit."""
    import torch
    cfg, ctx, orc, b, x0 = pb
    if len(b) > 100_000:
        pytest.skip("oracle GMRES too slow at this size; counts checked on the smaller cases")
    name, N = request.node.callspec.params["pb"][:2]
    maxit = MAXIT.get((name, N), 80)
    _, its_o, hist_o, conv_o = orc.gmres(b, maxit=maxit)
    xg = torch.empty(len(b), dtype=torch.float64, device="cuda:0")
    its_g, _, conv_g = ctx.gmres(cuda_vec(b), xg, maxit=maxit)
    hist_g = ctx.last_history
    assert conv_g == conv_o
    if conv_o and conv_g:
        assert abs(its_o - its_g) <= 1, (its_o, its_g)
    else:
        k = min(20, len(hist_o), len(hist_g))
        rel = np.abs(hist_g[:k] - hist_o[:k]) / np.abs(hist_o[:k])
        assert rel.max() <= 1e-6, rel.max()
    assert its_g == its_o and np.array_equal(hist_g, hist_o)


def _mask_around(cfg, verts, radius=3):
    """finest-level cells whose vertices all lie within lattice distance `radius` of one
    of `verts` (enough for every row of every patch containing the sampled DoFs)"""
    N, d = cfg.N, cfg.dim
    near = np.zeros((N + 1,) * d, bool)
    for v in verts:
        c = [v % (N + 1), (v // (N + 1)) % (N + 1), v // (N + 1) ** 2][:d][::-1]   # (k,)j,i
        near[tuple(slice(max(0, x - radius), x + radius + 1) for x in c)] = True
    if d == 2:
        sq = near[:-1, :-1] & near[1:, :-1] & near[:-1, 1:] & near[1:, 1:]
        return np.repeat(sq.ravel(), 2).astype(np.uint8)
    cube = near[:-1, :-1, :-1] & near[1:, :-1, :-1] & near[:-1, 1:, :-1] & near[:-1, :-1, 1:] \
        & near[1:, 1:, :-1] & near[1:, :-1, 1:] & near[:-1, 1:, 1:] & near[1:, 1:, 1:]
    return np.repeat(cube.ravel(), 6).astype(np.uint8)


def _patch_vertices(cfg):
    """vertex id of each library patch (R-patch: non-empty stars in vertex order).  Empty
    stars: 2D BDM1 -- the corners (N,0), (0,N) (only boundary edges); none for 3D."""
    N = cfg.N
    nv = (N + 1) ** cfg.dim
    if cfg.dim == 2 and cfg.block == "vel":
        return np.setdiff1d(np.arange(nv), [N, N * (N + 1)])
    return np.arange(nv)


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c3", "c4"])
def test_full_size_sweep_sampled(oracle_mod, name):
    """Full-size c3 / c4 (c5, the configuration bench.py times, is checked whole against
    the oracle's golden sweep and V-cycle in test_gpu_golden.py, which replaced its ~300 s
    sampled case here; c3 / c4 are checked both ways): one
    sweep from x0 = U(-1,1) on the GPU; the DoFs of the patches of ~40 sampled vertices
    (interior, wall, edge, corner) recomputed one by one by the exact oracle from a
    masked assembly; bit-exact, and relative l2 over the sample <= 1e-10."""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.CONFIGS[name]
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w0, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w0)
    n = ctx.n()
    w, b, x0 = workloads.draw(cfg, n, 0)
    ctx.setup()
    xg = cuda_vec(x0)
    ctx.smooth(cuda_vec(b), xg, nsweeps=1)
    xg = host(xg)
    N, d = cfg.N, cfg.dim
    pverts = _patch_vertices(cfg)
    ptr, dofs = ctx.patches()
    assert len(ptr) - 1 == len(pverts)
    rng = np.random.default_rng(11)
    corners = [0, N, (N + 1) ** d - 1]
    pick = np.unique(np.concatenate([rng.integers(0, (N + 1) ** d, 36), corners, [(N + 1) ** d // 2]]))
    pidx = np.flatnonzero(np.isin(pverts, pick))
    sample = np.unique(np.concatenate([dofs[ptr[i]:ptr[i + 1]] for i in pidx]))
    sample = np.sort(rng.choice(sample, size=min(200, sample.size), replace=False))
    mask = _mask_around(cfg, pverts[pidx])
    orc = oracle_mod.Oracle(cfg, w, nlev=1, cmask=mask, exact=True)
    xo = orc.sweep_sample(b, x0, sample.astype(np.int32))
    _same(xg[sample], xo)
