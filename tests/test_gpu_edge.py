"""GPU edge cases of the C-ABI: error paths, degenerate decompositions, determinism.

* ESINGULAR names the singular star (mhdp_last_error `where`: its mesh vertex on the
  mesh path, the patch index for operators installed by mhdp_load_level; the message
  names the level), and a singular coarse operator is reported as -1 (include/mhdp.h).
* ESTATE for device calls before mhdp_setup; EINVAL for patches above 160 DoFs.
* One patch covering every DoF: a sweep from 0 is the dense LU solve (P:536 with
  V_1 = V; the oracle pins this against numpy, test_oracle_solver.py) -- on the GPU it
  exercises the largest patch kernels (T = 3..5 rows per lane) and is compared bit for
  bit with the oracle using the same decomposition.
* Patches of size 1 (a diagonal, Jacobi-like decomposition) and a mixed ragged set.
* Determinism: repeated sweeps / V-cycles are bit-identical.
"""
import numpy as np
import pytest

from gpu_helpers import bits, cuda_vec, host, load_oracle_levels

pytestmark = pytest.mark.gpu


def _ctx():
    import torch
    from paper_2104_14855_b200 import mhdp
    return mhdp.Context(0, torch.cuda.current_stream().cuda_stream)


def test_state_errors():
    import torch
    from paper_2104_14855_b200 import mhdp
    ctx = _ctx()
    x = torch.zeros(4, dtype=torch.float64, device="cuda:0")
    assert ctx._L.mhdp_smooth(ctx.h, 1, 1, 0, x.data_ptr(), x.data_ptr()) == 5      # ESTATE: no setup
    assert ctx._L.mhdp_vcycle(ctx.h, 0, x.data_ptr(), x.data_ptr()) == 5


def test_singular_patch_reported(oracle_mod):
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c1", 4, 2)
    w, _, _ = workloads.draw(cfg, 1, 0)
    orc = oracle_mod.Oracle(cfg, w)
    ctx = _ctx()
    ctx.begin_levels(2, cfg)
    A0 = orc.csr(0)
    ctx.load_level(0, A0.rp, A0.ci, A0.v)
    A = orc.csr(1)
    v = A.v.copy()
    ptr, dofs, _, _ = orc.patches(1)
    bad = 3
    for d in dofs[ptr[bad]:ptr[bad + 1]]:          # zero the rows of one patch's DoFs
        v[A.rp[d]:A.rp[d + 1]] = 0.0
    P = orc.prolongation(1)
    ctx.load_level(1, A.rp, A.ci, v, ptr, dofs, P.rp, P.ci, P.v)
    with pytest.raises(mhdp.MhdpError) as e:
        ctx.setup()
    assert e.value.status == 4
    patch = e.value.where
    assert "level 1" in str(e.value)
    first = min(i for i in range(len(ptr) - 1) if np.isin(dofs[ptr[i]:ptr[i + 1]], dofs[ptr[bad]:ptr[bad + 1]]).any())
    assert patch == first      # the first singular patch in patch order


def test_singular_coarse_reported(oracle_mod):
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c1", 4, 1)
    ctx = _ctx()
    ctx.begin_levels(1, cfg)
    n = 5
    rp = np.arange(n + 1, dtype=np.int64)
    ci = np.arange(n, dtype=np.int32)
    ctx.load_level(0, rp, ci, np.array([1.0, 2.0, 0.0, 1.0, 1.0]))
    with pytest.raises(mhdp.MhdpError) as e:
        ctx.setup()
    assert e.value.status == 4 and e.value.where == -1


def test_patch_too_large_rejected():
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = workloads.small("c1", 4, 2)
    ctx = _ctx()
    ctx.begin_levels(2, cfg)
    n0, n = 3, 400                              # one star above K2_MAX_N = 384
    ctx.load_level(0, np.arange(n0 + 1), np.arange(n0, dtype=np.int32), np.ones(n0))
    rp = np.arange(n + 1)
    P_rp = np.arange(n + 1)
    P_ci = (np.arange(n) % n0).astype(np.int32)
    ctx.load_level(1, rp, np.arange(n, dtype=np.int32), np.ones(n), np.array([0, n]), np.arange(n, dtype=np.int32),
                   P_rp, P_ci, np.ones(n))
    with pytest.raises(mhdp.MhdpError) as e:
        ctx.setup()
    assert e.value.status == 1


def _single_patch_case(oracle_mod, name, N, decomposition):
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small(name, N, 2)
    w, _, _ = workloads.draw(cfg, 1, 3)
    orc = oracle_mod.Oracle(cfg, w)
    n = orc.n()
    if decomposition == "single" and n > 160:
        pytest.skip("above the 160-DoF patch limit")
    if decomposition == "single":
        ptr, dofs = np.array([0, n], np.int64), np.arange(n, dtype=np.int32)
    elif decomposition == "diagonal":
        ptr, dofs = np.arange(n + 1, dtype=np.int64), np.arange(n, dtype=np.int32)
    else:   # ragged: blocks of sizes 1, 2, 3, ... cycling, overlapping by one DoF
        ptr, dofs, start, k = [0], [], 0, 1
        while start < n:
            blk = list(range(max(0, start - 1), min(n, start + k)))
            dofs += blk
            ptr.append(len(dofs))
            start += k
            k = k % 7 + 1
        ptr, dofs = np.array(ptr, np.int64), np.array(dofs, np.int32)
    orc.set_patches(ptr, dofs)
    ctx = _ctx()
    ctx.begin_levels(2, cfg)
    A0 = orc.csr(0)
    ctx.load_level(0, A0.rp, A0.ci, A0.v)
    A = orc.csr(1)
    P = orc.prolongation(1)
    ctx.load_level(1, A.rp, A.ci, A.v, ptr, dofs, P.rp, P.ci, P.v)
    ctx.setup()
    return cfg, orc, ctx, n


@pytest.mark.parametrize("name,N", [("c1", 4), ("c1", 6), ("c3", 4), ("c4", 2)])
def test_single_patch_is_direct_solve(oracle_mod, name, N):
    cfg, orc, ctx, n = _single_patch_case(oracle_mod, name, N, "single")
    rng = np.random.default_rng(1)
    b = rng.uniform(-1, 1, n)
    xo = orc.sweep(b, np.zeros(n), x_is_zero=True)
    xg = cuda_vec(np.zeros(n))
    ctx.smooth(cuda_vec(b), xg, nsweeps=1, x_is_zero=True)
    assert np.array_equal(bits(host(xg)), bits(xo))
    A = orc.csr().to_scipy().toarray()
    assert np.linalg.norm(A @ host(xg) - b) <= 1e-9 * np.linalg.norm(b) * np.linalg.cond(A)


@pytest.mark.parametrize("decomposition", ["diagonal", "ragged"])
def test_degenerate_decompositions(oracle_mod, decomposition):
    cfg, orc, ctx, n = _single_patch_case(oracle_mod, "c3", 8, decomposition)
    rng = np.random.default_rng(2)
    b, x0 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
    xo = orc.sweep(b, x0, nsweeps=2)
    xg = cuda_vec(x0)
    ctx.smooth(cuda_vec(b), xg, nsweeps=2)
    assert np.array_equal(bits(host(xg)), bits(xo))


def test_determinism_repeated_runs(oracle_mod):
    import torch
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c5", 8, 2)
    w, _, _ = workloads.draw(cfg, 1, 4)
    ctx = _ctx()
    ctx.assemble(cfg, w)
    ctx.setup()
    n = ctx.n()
    _, b, x0 = workloads.draw(cfg, n, 4)
    outs = []
    for _ in range(3):
        xg = torch.empty(n, dtype=torch.float64, device="cuda:0")
        ctx.vcycle(cuda_vec(b), xg)
        xs = cuda_vec(x0)
        ctx.smooth(cuda_vec(b), xs, nsweeps=2)
        outs.append((bits(host(xg)), bits(host(xs))))
    for o in outs[1:]:
        assert np.array_equal(o[0], outs[0][0]) and np.array_equal(o[1], outs[0][1])


@pytest.mark.parametrize("smoother", ["richardson", "gmres"])
def test_vcycle_graph_replay_bitexact(oracle_mod, smoother):
    """mhdp_vcycle replays a captured CUDA graph from the second call with the same
    (level, b, x); the replayed cycle is bit-identical to the direct one and to the
    oracle."""
    import torch
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c5", 6, 2)
    w, _, _ = workloads.draw(cfg, 1, 9)
    ctx = _ctx()
    ctx.assemble(cfg, w, smoother=smoother)
    ctx.setup()
    n = ctx.n()
    _, b, _ = workloads.draw(cfg, n, 9)
    orc = oracle_mod.Oracle(cfg, w, exact=True)
    orc.set_smoother(smoother, 6)
    ref = bits(orc.vcycle(b))
    bd = cuda_vec(b)
    xg = torch.empty(n, dtype=torch.float64, device="cuda:0")
    for call in range(4):
        xg.fill_(3.0)
        ctx.vcycle(bd, xg)
        assert np.array_equal(bits(host(xg)), ref), f"call {call}"
    assert ctx.graphs_active() >= 1


@pytest.mark.parametrize("name,N", [("c1", 4), ("c3", 4), ("c4", 2), ("c5", 2)])
def test_k2_single_level_vcycle_is_coarse_solve(oracle_mod, name, N):
    """NEXT-2 degenerate hierarchy: one level at k = 2 -- the V-cycle is the coarse solve
    (explicit inverse, R-coarse), bit-exact against the oracle's exact build."""
    import dataclasses
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = dataclasses.replace(workloads.small(name, N, 1), degree=2,
                              sigma=40.0 if name in ("c3", "c5") else 10.0)
    w, _, _ = workloads.draw(cfg, 1, 3)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    ctx.assemble(cfg, w)
    ctx.setup()
    n = ctx.n()
    b = np.random.default_rng(3).uniform(-1, 1, n)
    orc = oracle_mod.Oracle(cfg, w, exact=True)
    x = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(torch.from_numpy(b).cuda(), x)
    assert np.array_equal(x.cpu().numpy().view(np.uint64), orc.vcycle(b).view(np.uint64))


def test_vcycle_host_batch_matches_serial():
    """mhdp_vcycle_host_batch (copies overlapped on two device slots) returns, for every
    right-hand side, the bits of mhdp_vcycle_host; nrhs = 0 is a no-op, odd counts and
    repeated calls reuse the slots' captured graphs."""
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c5", 6, 2)
    ctx = _ctx()
    w, _, _ = workloads.draw(cfg, 1, 2)
    ctx.assemble(cfg, w)
    ctx.setup()
    n = ctx.n()
    rng = np.random.default_rng(8)
    B = np.ascontiguousarray(rng.uniform(-1, 1, (5, n)))
    ref = np.zeros_like(B)
    for k in range(5):
        ctx.vcycle_host(np.ascontiguousarray(B[k]), ref[k])
    for count in (5, 3, 1):
        X = np.full((count, n), 7.0)
        ctx.vcycle_host_batch(np.ascontiguousarray(B[:count]), X)
        assert np.array_equal(X.view(np.uint64), ref[:count].view(np.uint64)), count
    ctx.vcycle_host_batch(np.zeros((0, n)), np.zeros((0, n)))


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 63, 65, 257, 300])
def test_coarse_lu_solve_ragged_sizes(oracle_mod, n):
    """K7 + K8 on dense coarse operators whose order is not a multiple of the 32-row
    blocks / 32-column panels (ragged tails, one-block and few-block chains, with and
    without far warps): the solve equals the oracle's pinned R-lu routine bit for bit,
    and row pivoting is exercised (a permuted diagonally weighted random matrix)."""
    import torch
    from paper_2104_14855_b200 import workloads
    rng = np.random.default_rng(n)
    A = rng.uniform(-1, 1, (n, n)) + np.diag(rng.uniform(1, 2, n)) * n ** 0.5
    A = A[rng.permutation(n)]                       # pivots away from the diagonal
    b = rng.uniform(-1, 1, n)
    ref = oracle_mod.dense_lu_solve(A, b)[0]
    cfg = workloads.small("c1", 4, 1)
    ctx = _ctx()
    ctx.begin_levels(1, cfg)
    rp = np.arange(0, n * n + 1, n, dtype=np.int64)
    ci = np.tile(np.arange(n, dtype=np.int32), n)
    ctx.load_level(0, rp, ci, A.ravel())
    ctx.setup()
    x = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.coarse_solve(cuda_vec(b), x)
    assert np.array_equal(bits(host(x)), bits(ref))


def test_pivot_div_is_the_ieee_quotient():
    """PivotDiv (k2_common.cuh) forms the LU multipliers l = a_ik / a_kk of K6 / K7 from one
    reciprocal per pivot (the instruction sequence of the inline fast path of '/').  R-lu
    asks for the IEEE quotient: compared bit for bit with numpy's division (IEEE RN) on
    numerators over the whole exponent range, exact and signed zeros, subnormals, operands
    outside the guarded range (IEEE fallback), infinities and NaN, and on pivots that are
    random, powers of two, of both signs, with an all-ones significand, tiny and huge."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    import probe
    rng = np.random.Generator(np.random.PCG64(20260421))
    mant = rng.uniform(1.0, 2.0, 200000)
    x = np.concatenate([
        mant[:100000] * np.exp2(rng.integers(-30, 30, 100000)) * rng.choice([-1.0, 1.0], 100000),
        mant[100000:] * np.exp2(rng.integers(-1000, 1000, 100000)) * rng.choice([-1.0, 1.0], 100000),
        [0.0, -0.0, 5e-324, -5e-324, 2.2250738585072014e-308, 1.7976931348623157e308, -1.7976931348623157e308,
         np.inf, -np.inf, np.nan, 1.0, -1.0, 3.0, 1.0 / 3.0, 2.0 ** -400, 2.0 ** 400, 2.0 ** -401, 2.0 ** 401],
        np.nextafter(np.exp2(np.arange(-60.0, 60.0)), 0.0), np.nextafter(np.exp2(np.arange(-60.0, 60.0)), np.inf)])
    allones = np.array([0x3FFFFFFFFFFFFFFF, 0xBFEFFFFFFFFFFFFF, 0x40AFFFFFFFFFFFFF], dtype=np.uint64).view(np.float64)
    piv = np.concatenate([
        rng.uniform(1.0, 2.0, 40) * np.exp2(rng.integers(-40, 40, 40)) * rng.choice([-1.0, 1.0], 40),
        [1.0, -1.0, 2.0, 0.5, 3.0, -7.0, 1e4, -1e-4, 1.0 / 3.0, 2.0 ** -399, 2.0 ** 399, 2.0 ** -420, 2.0 ** 420,
         5e-324, 1.7976931348623157e308],
        allones, np.nextafter(np.exp2(np.arange(-8.0, 8.0)), 0.0)])
    got = probe.pivot_div(x, piv)
    with np.errstate(all="ignore"):
        want = x[None, :] / piv[:, None]
    nan = np.isnan(want)
    assert np.array_equal(np.isnan(got), nan)
    assert np.array_equal(bits(got[~nan]), bits(want[~nan]))
