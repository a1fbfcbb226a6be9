"""Patch conditioning (max kappa(A_i) per level; the full report is
tools/kappa_report.py -> profiles/kappa_report.json).  Pin: every vertex star of the AL
velocity block contains local divergence-free fields (the kernel of gamma (div, div);
P:549-571), so the smallest singular value of A_i stays O(1/Re) while the largest grows
with gamma -- kappa(A_i) is linear in gamma.  A star that lost its kernel functions (a
wrong patch definition) would instead saturate."""
import dataclasses

import numpy as np


def test_star_patch_kappa_linear_in_gamma(oracle_mod):
    import sys, os
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools"))
    from kappa_report import patch_kappas
    from paper_2104_14855_b200 import workloads
    kap = {}
    for g in (1e2, 1e4, 1e6):
        cfg = dataclasses.replace(workloads.small("c3", 8, 1), Re=1.0, gamma=g)
        w, _, _ = workloads.draw(cfg, 1, 0)
        o = oracle_mod.Oracle(cfg, w, nlev=1)
        ptr, dofs, _, _ = o.patches()
        kap[g] = max(k for _, k in patch_kappas(o.csr().to_scipy(), ptr, dofs))
    r1, r2 = kap[1e4] / kap[1e2], kap[1e6] / kap[1e4]
    assert 30 < r1 < 300 and 30 < r2 < 300, kap
