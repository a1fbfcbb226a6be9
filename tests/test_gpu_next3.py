"""GPU parity for NEXT-3: the coupled Newton system over [u | p | E | B]
(Table 1) and the paper's outer solver -- flexible GMRES preconditioned by the
block upper-triangular preconditioner with inner FGMRES(2) solves on the E-B block and
on the (u, p) block.

The library assembles everything itself (double-double host setup, reading R-cgrid for
the coupling rows) and the oracle is its exact build: the operators agree bit for bit
(tests/test_library_host.py), every reduction is pinned (R-dot) and the scalar Krylov
steps round each operation separately, so apply, precondition and the outer FGMRES
iterates are expected BIT-EXACT (tier P-B).
"""
import dataclasses

import numpy as np
import pytest

from gpu_helpers import bits, cuda_vec, host

pytestmark = pytest.mark.gpu

CASES = [
    ("2D-N8L2", "c3", 8, 2, dict(), "richardson"),
    ("2D-N8L2-gmres", "c3", 8, 2, dict(), "gmres"),
    ("2D-N8L3-picard-transient", "c3", 8, 3, dict(picard=1, dt=0.1), "richardson"),
    ("3D-N4L2", "c5", 4, 2, dict(), "richardson"),
    ("3D-N4L2-transient", "c5", 4, 2, dict(dt=0.05), "gmres"),
]


def _pair(oracle_mod, name, N, L, kw, smoother, seed=6):
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    cfg = dataclasses.replace(workloads.small(name, N, L), Re=10.0, Rem=5.0, gamma=100.0, S=3.0, **kw)
    w, _, _ = workloads.draw(cfg, 1, seed)
    bn = workloads.magnetic_potential(cfg, seed)
    orc = oracle_mod.CoupledOracle(cfg, w, bn, exact=True, smoother=smoother, smoother_its=6)
    lib = mhdp.Coupled(cfg, w, bn, device=0, stream=torch.cuda.current_stream().cuda_stream,
                       smoother=smoother, smoother_its=6)
    assert lib.n == orc.n
    return orc, lib


def _rhs(n, seed):
    return np.random.default_rng(seed).standard_normal(n)


@pytest.mark.parametrize("case,name,N,L,kw,smoother", CASES, ids=[c[0] for c in CASES])
def test_coupled_apply_bitexact(oracle_mod, case, name, N, L, kw, smoother):
    import torch
    orc, lib = _pair(oracle_mod, name, N, L, kw, smoother)
    x = _rhs(orc.n, 1)
    y = torch.empty(orc.n, dtype=torch.float64, device="cuda:0")
    lib.apply(cuda_vec(x), y)
    assert np.array_equal(bits(host(y)), bits(orc.apply(x)))


@pytest.mark.parametrize("case,name,N,L,kw,smoother", CASES, ids=[c[0] for c in CASES])
def test_coupled_precondition_bitexact(oracle_mod, case, name, N, L, kw, smoother):
    import torch
    orc, lib = _pair(oracle_mod, name, N, L, kw, smoother)
    r = _rhs(orc.n, 2)
    y = torch.empty(orc.n, dtype=torch.float64, device="cuda:0")
    lib.precondition(cuda_vec(r), y)
    assert np.array_equal(bits(host(y)), bits(orc.precondition(r)))


@pytest.mark.parametrize("case,name,N,L,kw,smoother", CASES, ids=[c[0] for c in CASES])
def test_coupled_outer_fgmres_bitexact(oracle_mod, case, name, N, L, kw, smoother):
    import torch
    orc, lib = _pair(oracle_mod, name, N, L, kw, smoother)
    b = _rhs(orc.n, 3)
    xo, its_o, hist, conv_o = orc.fgmres(b, rtol=1e-8, atol=1e-12, maxit=30)
    x = torch.empty(orc.n, dtype=torch.float64, device="cuda:0")
    its_g, rel_g, conv_g = lib.fgmres(cuda_vec(b), x, rtol=1e-8, atol=1e-12, maxit=30)
    assert (its_g, conv_g) == (its_o, conv_o)
    assert np.array_equal(bits(host(x)), bits(xo))
    # the true residual of the returned iterate (the paper's stopping test)
    res = np.linalg.norm(b - orc.apply(host(x))) / np.linalg.norm(b)
    if conv_g:
        assert res <= 1e-7


def test_coupled_repeatable_and_stream_ordered(oracle_mod):
    """Two solves on the same object give identical bits (workspaces are reset)."""
    import torch
    _, lib = _pair(oracle_mod, "c3", 8, 2, dict(), "richardson")
    b = cuda_vec(_rhs(lib.n, 4))
    x1 = torch.empty(lib.n, dtype=torch.float64, device="cuda:0")
    x2 = torch.empty_like(x1)
    lib.fgmres(b, x1, maxit=10)
    lib.fgmres(b, x2, maxit=10)
    assert torch.equal(x1, x2)
