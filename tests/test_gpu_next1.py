"""GPU parity for NEXT-1: the paper's relaxation -- GMRES(6)
preconditioned by the vertex-star Schwarz operator on every level -- and flexible
GMRES as the outermost solver (tolerances P:654).

Inner products use the pinned order of reading R-dot on both sides and the scalar
Givens / back-substitution steps round every operation separately, so the V-cycle and
the FGMRES iterates are expected BIT-EXACT against the oracle: on the oracle's operator
(tier P-C) and with the library's own setup against the oracle's exact build (P-B).
"""
import numpy as np
import pytest

from gpu_helpers import bits, cuda_vec, host, load_oracle_levels

pytestmark = pytest.mark.gpu


def _ctx():
    import torch
    from paper_2104_14855_b200 import mhdp
    return mhdp.Context(0, torch.cuda.current_stream().cuda_stream)


@pytest.mark.parametrize("n", [0, 1, 255, 256, 257, 4097, 100003, 3939840])
def test_pinned_dot_bitexact(oracle_mod, n):
    rng = np.random.default_rng(n)
    a, b = rng.standard_normal(n), rng.standard_normal(n)
    ctx = _ctx()
    got = ctx.dot(cuda_vec(a), cuda_vec(b))
    assert np.float64(got).view(np.uint64) == np.float64(oracle_mod.dot(a, b)).view(np.uint64)


CASES_PC = [("c1", 8, 2), ("c3", 16, 3), ("c4", 8, 2), ("c5", 6, 2)]


@pytest.mark.parametrize("name,N,L", CASES_PC, ids=[f"{c}-N{n}L{l}" for c, n, l in CASES_PC])
def test_gmres_smoothed_vcycle_and_fgmres_on_oracle_operator(oracle_mod, name, N, L):
    import torch
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small(name, N, L)
    w0, _, _ = workloads.draw(cfg, 1, 6)
    probe = oracle_mod.Oracle(cfg, w0)
    w, b, _ = workloads.draw(cfg, probe.n(), 6)
    orc = oracle_mod.Oracle(cfg, w)
    orc.set_smoother("gmres", 6)
    ctx = _ctx()
    load_oracle_levels(ctx, orc, cfg, smoother="gmres", smoother_its=6)
    xo = orc.vcycle(b)
    xg = torch.empty(len(b), dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(b), xg)
    assert np.array_equal(bits(host(xg)), bits(xo))
    xo, its_o, _, conv_o = orc.fgmres(b, maxit=40)
    its_g, _, conv_g = ctx.fgmres(cuda_vec(b), xg, maxit=40)
    assert (its_g, conv_g) == (its_o, conv_o)
    assert np.array_equal(bits(host(xg)), bits(xo))


CASES_PB = [("c1", None, None), ("c3", 32, 4), ("c5", 6, 2), ("c2-k2", 64, 4), ("c3-k2", 32, 4), ("c4-k2", 4, 2), ("c5-k2", 4, 2)]


@pytest.mark.parametrize("name,N,L", CASES_PB, ids=[f"{c}-{n or 'full'}" for c, n, l in CASES_PB])
def test_gmres_smoothed_end_to_end(oracle_mod, name, N, L):
    import torch
    from paper_2104_14855_b200 import workloads
    import dataclasses
    k2 = name.endswith("-k2")                       # NEXT-2
    name = name.replace("-k2", "")
    cfg = workloads.CONFIGS[name] if N is None else workloads.small(name, N, L)
    if k2:
        cfg = dataclasses.replace(cfg, degree=2, sigma=40.0 if cfg.block == "vel" else cfg.sigma)
    ctx = _ctx()
    w0, _, _ = workloads.draw(cfg, 1, 7)
    ctx.assemble(cfg, w0, smoother="gmres", smoother_its=6)
    n = ctx.n()
    w, b, _ = workloads.draw(cfg, n, 7)
    ctx.setup()
    orc = oracle_mod.Oracle(cfg, w, exact=True)
    orc.set_smoother("gmres", 6)
    xo = orc.vcycle(b)
    xg = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(cuda_vec(b), xg)
    assert np.array_equal(bits(host(xg)), bits(xo))
    xo, its_o, _, conv_o = orc.fgmres(b, maxit=40)
    its_g, rel, conv_g = ctx.fgmres(cuda_vec(b), xg, maxit=40)
    assert (its_g, conv_g) == (its_o, conv_o)
    assert np.array_equal(bits(host(xg)), bits(xo))


def test_gmres_smoother_zero_rhs_breakdown(oracle_mod):
    """b = 0: the smoother's Krylov space is empty (beta = 0, R-gmres6 breakdown), the
    V-cycle returns exactly 0 (no NaN from the 0/0 of the first basis vector)."""
    import torch
    from paper_2104_14855_b200 import workloads
    cfg = workloads.small("c5", 4, 2)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx = _ctx()
    ctx.assemble(cfg, w, smoother="gmres", smoother_its=6)
    ctx.setup()
    n = ctx.n()
    xg = torch.full((n,), 7.0, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(torch.zeros(n, dtype=torch.float64, device="cuda:0"), xg)
    assert torch.count_nonzero(xg).item() == 0
