"""Shared helpers of the GPU parity tests (test infrastructure).

`load_oracle_levels` feeds the ORACLE's assembled hierarchy into the library through
its algebraic entry (mhdp_begin_levels / mhdp_load_level): both sides then run their
smoother / V-cycle on the very same operator (parity tier P-C of DESIGN.md), so the
comparison isolates the CUDA kernels.  Data flows oracle -> library only.
"""
import numpy as np


def bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def rel_l2(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def load_oracle_levels(ctx, orc, cfg, smoother="richardson", smoother_its=6):
    ctx.begin_levels(orc.nlev, cfg, smoother, smoother_its)
    for l in range(orc.nlev):
        A = orc.csr(l)
        if l == 0:
            ctx.load_level(0, A.rp, A.ci, A.v)
        else:
            ptr, dofs, _, _ = orc.patches(l)
            P = orc.prolongation(l)
            ctx.load_level(l, A.rp, A.ci, A.v, ptr, dofs, P.rp, P.ci, P.v)
    ctx.setup()


def cuda_vec(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, np.float64)).to("cuda:0")


def host(t):
    return t.detach().cpu().numpy()
