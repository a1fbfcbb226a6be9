"""GPU parity, tier P-C: the library's CUDA kernels on the ORACLE's operator.

The oracle's CSR, patches and prolongations are installed through the C-ABI's
algebraic entry; the oracle and the GPU then run the same method on the same
operator.  Every reduction follows the order of reading R-order, so the
expected result is BIT-EXACT: patch LU factors and pivots, residual, one sweep (x0 = 0
and x0 = U(-1,1)), two sweeps, restriction, prolongation, coarse solve and V-cycle.
GMRES(V) runs the oracle's iteration step for step (R-dot inner products): equal
counts and bit-identical residual histories.  Sizes span several tiles with ragged tails (patch sizes
of every boundary class, levels whose n is not a multiple of 32).
"""
import numpy as np
import pytest

from gpu_helpers import bits, cuda_vec, host, load_oracle_levels, rel_l2

pytestmark = pytest.mark.gpu

CASES = [("c1", 8, 2), ("c2", 32, 3), ("c3", 16, 3), ("c4", 8, 2), ("c5", 6, 2), ("c2-k2", 32, 3), ("c3-k2", 16, 3),
         ("c4-k2", 4, 2), ("c5-k2", 4, 2)]


@pytest.fixture(scope="module", params=CASES, ids=[f"{c}-N{n}L{l}" for c, n, l in CASES])
def pair(request, oracle_mod):
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    name, N, L = request.param
    import dataclasses
    k2 = name.endswith("-k2")                       # NEXT-2: CG2 x RT2 (31-DoF stars), BDM2, 3D
    cfg = workloads.small(name.replace("-k2", ""), N, L)   # NED1_2 x RT2 (280) and BDM2 (360 DoFs)
    if k2:
        cfg = dataclasses.replace(cfg, degree=2, sigma=40.0 if cfg.block == "vel" else cfg.sigma)
        if cfg.dim == 3:                            # Newton at Rem = S = 1e3 needs the GMRES(6)
            cfg = dataclasses.replace(cfg, picard=1)   # smoother; Picard: GMRES(V) in 8
    # draw with the finest n of this hierarchy
    probe = oracle_mod.Oracle(cfg, workloads.advecting_potential(cfg, np.array([0.3, -1.1, 0.7])))
    n = probe.n()
    w, b, x0 = workloads.draw(cfg, n, seed=1)
    orc = oracle_mod.Oracle(cfg, w)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    load_oracle_levels(ctx, orc, cfg)
    return cfg, orc, ctx, b, x0


def test_patch_lu_bitexact(pair):
    cfg, orc, ctx, b, x0 = pair
    top = orc.nlev - 1
    npatch = orc.info(top)["npatch"]
    ptr = orc.patches(top)[0]
    sizes = np.diff(ptr)
    # every size class plus a spread of indices
    pick = sorted(set([int(np.flatnonzero(sizes == s)[0]) for s in np.unique(sizes)] +
                      list(np.linspace(0, npatch - 1, 7).astype(int))))
    for i in pick:
        lu_o, perm_o, st = orc.patch_lu(i, top)
        assert st == 0
        lu_g, perm_g = ctx.patch_lu(i, top)
        assert np.array_equal(perm_o, perm_g), f"patch {i}: pivot order differs"
        assert np.array_equal(bits(lu_o), bits(lu_g)), f"patch {i}: factors differ"


def test_residual_and_spmv_bitexact(pair):
    import torch
    cfg, orc, ctx, b, x0 = pair
    for l in range(orc.nlev):
        n = orc.n(l)
        rng = np.random.default_rng(l)
        bb, xx = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        r = torch.empty(n, dtype=torch.float64, device="cuda:0")
        ctx.residual(cuda_vec(bb), cuda_vec(xx), r, level=l)
        assert np.array_equal(bits(host(r)), bits(orc.residual(bb, xx, l)))
        ctx.spmv(cuda_vec(xx), r, level=l)
        assert np.array_equal(bits(host(r)), bits(orc.spmv(xx, l)))


@pytest.mark.parametrize("zero", [True, False])
@pytest.mark.parametrize("nsweeps", [1, 2])
def test_sweep_bitexact(pair, zero, nsweeps):
    cfg, orc, ctx, b, x0 = pair
    x_in = np.zeros_like(x0) if zero else x0
    xo = orc.sweep(b, x_in, nsweeps=nsweeps, x_is_zero=zero)
    xg = cuda_vec(x_in)
    ctx.smooth(cuda_vec(b), xg, nsweeps=nsweeps, x_is_zero=zero)
    xg = host(xg)
    assert rel_l2(xg, xo) <= 1e-10
    assert np.array_equal(bits(xg), bits(xo))


def test_transfer_bitexact(pair):
    import torch
    cfg, orc, ctx, b, x0 = pair
    for l in range(1, orc.nlev):
        rng = np.random.default_rng(10 + l)
        r = rng.uniform(-1, 1, orc.n(l)); ec = rng.uniform(-1, 1, orc.n(l - 1)); x = rng.uniform(-1, 1, orc.n(l))
        rc = torch.empty(orc.n(l - 1), dtype=torch.float64, device="cuda:0")
        ctx.restrict(cuda_vec(r), rc, level=l)
        assert np.array_equal(bits(host(rc)), bits(orc.restrict(r, l)))
        xg = cuda_vec(x)
        ctx.prolong_add(cuda_vec(ec), xg, level=l)
        assert np.array_equal(bits(host(xg)), bits(orc.prolong_add(ec, x, l)))


def test_coarse_solve_bitexact(pair):
    import torch
    cfg, orc, ctx, b, x0 = pair
    rng = np.random.default_rng(5)
    bc = rng.uniform(-1, 1, orc.n(0))
    xg = torch.empty(orc.n(0), dtype=torch.float64, device="cuda:0")
    ctx.coarse_solve(cuda_vec(bc), xg)
    assert np.array_equal(bits(host(xg)), bits(orc.coarse_solve(bc)))


def test_vcycle_bitexact(pair):
    import torch
    cfg, orc, ctx, b, x0 = pair
    xo = orc.vcycle(b)
    xg = torch.empty(len(b), dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(b), xg)
    xg = host(xg)
    assert rel_l2(xg, xo) <= 1e-10
    assert np.array_equal(bits(xg), bits(xo))
    # host-buffer entry point gives the same bits
    xh = np.zeros_like(b)
    ctx.vcycle_host(np.ascontiguousarray(b), xh)
    assert np.array_equal(bits(xh), bits(xo))


def test_gmres_iterations(pair):
    """a8 under P-C: GMRES(V) on the shared operator is the oracle's iteration step for
    step (R-dot inner products, the same Givens arithmetic): equal counts, the residual
    histories bit for bit whether or not it converges, and a true residual
    within the stopping tolerance when it does."""
    import torch
    cfg, orc, ctx, b, x0 = pair
    _, its_o, hist_o, conv_o = orc.gmres(b, maxit=60)
    xg = torch.empty(len(b), dtype=torch.float64, device="cuda:0")
    its_g, rel_g, conv_g = ctx.gmres(cuda_vec(b), xg, maxit=60)
    assert conv_o == conv_g and its_o == its_g
    assert np.array_equal(bits(ctx.last_history), bits(hist_o))
    if conv_g:
        A = orc.csr().to_scipy()
        r = b - A @ host(xg)
        assert np.linalg.norm(r) <= 1.01 * max(1e-7 * np.linalg.norm(b), 1e-7)


def _union_patches(orc, N, level, block):
    """unions of the vertex stars of level `level` over blocks of lattice vertices"""
    ptr, dofs, verts, _ = orc.patches(level)
    lat = np.stack([verts % (N + 1), (verts // (N + 1)) % (N + 1), verts // (N + 1) ** 2], axis=1)
    key = (lat[:, 0] // block[0]) + 1000 * (lat[:, 1] // block[1]) + 1000000 * (lat[:, 2] // block[2])
    out = [np.unique(np.concatenate([dofs[ptr[i]:ptr[i + 1]] for i in np.flatnonzero(key == k)]))
           for k in np.unique(key)]
    nptr = np.concatenate([[0], np.cumsum([len(p) for p in out])]).astype(np.int64)
    return nptr, np.concatenate(out).astype(np.int32)


@pytest.mark.parametrize("block", [(2, 1, 1), (2, 2, 1)], ids=["to198", "to354"])
def test_large_patches_bitexact(oracle_mod, block):
    """Stars beyond 160 DoFs, up to the 3D k = 2 sizes: unions of neighbouring
    c5 vertex stars (up to 198 / 354 DoFs) installed on both sides.  K6 keeps such patch
    matrices in a global-memory scratch, K2 streams them through 4 KB-chunk rings; factors,
    sweeps and the V-cycle are bit-exact against the oracle."""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c5", 6, 2)
    w, _, _ = workloads.draw(cfg, 1, 4)
    orc = oracle_mod.Oracle(cfg, w)
    ptr, dofs = _union_patches(orc, cfg.N, 1, block)
    assert np.diff(ptr).max() > 160
    orc.set_patches(ptr, dofs, 1)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    load_oracle_levels(ctx, orc, cfg)
    n = orc.n()
    rng = np.random.default_rng(2)
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    big = int(np.argmax(np.diff(ptr)))
    lu_g, perm_g = ctx.patch_lu(big)
    lu_o, perm_o, st = orc.patch_lu(big)
    assert st == 0 and np.array_equal(perm_g, perm_o) and np.array_equal(bits(lu_g), bits(lu_o))
    xg = cuda_vec(x0)
    ctx.smooth(cuda_vec(b), xg, nsweeps=1)
    assert np.array_equal(bits(host(xg)), bits(orc.sweep(b, x0, nsweeps=1)))
    xv = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(b), xv)
    assert np.array_equal(bits(host(xv)), bits(orc.vcycle(b)))


def test_coarse_solve_large_bitexact(oracle_mod):
    """K8 on a coarse operator of 2016 DoFs (c5 family, N = 4, one level: 63 row blocks, so
    the far warps of k8_coarse.cu hand partial sums to the chain CTA) is bit-identical to
    the oracle's R-lu solve -- for several right-hand sides in a row
    (the kernel's epoch / progress words carry over between calls), through the V-cycle
    entry (one level: V = coarse solve) and with b and x aliased."""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c5", 4, 1)
    w, _, _ = workloads.draw(cfg, 1, 2)
    orc = oracle_mod.Oracle(cfg, w)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    load_oracle_levels(ctx, orc, cfg)
    n = orc.n(0)
    assert n == 2016
    rng = np.random.default_rng(9)
    for k in range(4):
        bc = rng.uniform(-1, 1, n)
        xg = torch.empty(n, dtype=torch.float64, device="cuda:0")
        ctx.coarse_solve(cuda_vec(bc), xg)
        ref = orc.coarse_solve(bc)
        assert np.array_equal(bits(host(xg)), bits(ref)), k
    xv = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(bc), xv)
    assert np.array_equal(bits(host(xv)), bits(ref))
    xa = cuda_vec(bc)
    ctx.coarse_solve(xa, xa)
    assert np.array_equal(bits(host(xa)), bits(ref))


def test_patch_lu_every_size_33_to_128(oracle_mod):
    """k_patch_lu_cm (k6_patch_lu.cu: panels of 4, four-warp panel group) on one patch of EVERY
    size 33..128 -- every ragged last panel (n mod 4), every count of 32-row chunks, last chunks
    of 1..32 rows -- next to the c5 vertex stars: random sorted subsets of unions of neighbouring
    stars, installed on both sides.  Principal submatrices of the (coercive) velocity operator
    are nonsingular; on the uniform mesh they are full of exact zeros and exactly tied pivot
    candidates.  Factors and pivots bit for bit against the oracle's od_lu, then one sweep."""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c5", 6, 2)
    w, _, _ = workloads.draw(cfg, 1, 4)
    orc = oracle_mod.Oracle(cfg, w)
    ptr0, dofs0 = orc.patches(1)[:2]
    uptr, udofs = _union_patches(orc, cfg.N, 1, (2, 1, 1))
    big = [udofs[uptr[i]:uptr[i + 1]] for i in range(len(uptr) - 1) if uptr[i + 1] - uptr[i] >= 128]
    assert big
    rng = np.random.default_rng(5)
    extra = [np.sort(rng.choice(big[m % len(big)], size=m, replace=False)).astype(np.int32) for m in range(33, 129)]
    stars = [dofs0[ptr0[i]:ptr0[i + 1]] for i in range(len(ptr0) - 1)]
    allp = stars + extra
    ptr = np.concatenate([[0], np.cumsum([len(p) for p in allp])]).astype(np.int64)
    dofs = np.concatenate(allp).astype(np.int32)
    assert np.diff(ptr).max() == 128
    orc.set_patches(ptr, dofs, 1)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    load_oracle_levels(ctx, orc, cfg)
    for i in range(len(stars), len(allp)):
        lu_o, perm_o, st = orc.patch_lu(i)
        assert st == 0
        lu_g, perm_g = ctx.patch_lu(i)
        assert np.array_equal(perm_o, perm_g), f"size {len(allp[i])}: pivot order differs"
        assert np.array_equal(bits(lu_o), bits(lu_g)), f"size {len(allp[i])}: factors differ"
    n = orc.n()
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    xg = cuda_vec(x0)
    ctx.smooth(cuda_vec(b), xg, nsweeps=1)
    assert np.array_equal(bits(host(xg)), bits(orc.sweep(b, x0, nsweeps=1)))
