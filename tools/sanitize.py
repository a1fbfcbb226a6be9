"""Small end-to-end exercise of every device kernel for compute-sanitizer (SURVEY §4 layer
4 / §5 "race detection"): c1 and c2 (2D E-B) and a reduced c5 (3D velocity, 3D k = 1
stars, far warps of K8 active), each: setup (K6, K7, K8 pack), one sweep from x0, one
V-cycle, a coarse solve, three GMRES(V) iterations and one GMRES(6)-smoothed V-cycle.

    compute-sanitizer --tool memcheck   python tools/sanitize.py
    compute-sanitizer --tool racecheck  python tools/sanitize.py
    compute-sanitizer --tool synccheck  python tools/sanitize.py
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402

CASES = [("c1", None, None), ("c2", 32, 3), ("c5", 8, 2)]


def run(name, N, L):
    cfg = workloads.CONFIGS[name] if N is None else workloads.small(name, N, L)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w)
    n = ctx.n()
    _, b, x0 = workloads.draw(cfg, n, 0)
    ctx.setup()
    bd = torch.from_numpy(b).cuda()
    x = torch.from_numpy(x0.copy()).cuda()
    ctx.smooth(bd, x, nsweeps=1)
    v = torch.empty_like(bd)
    ctx.vcycle(bd, v)
    n0 = ctx.n(0)
    bc = torch.from_numpy(np.random.default_rng(1).uniform(-1, 1, n0)).cuda()
    xc = torch.empty_like(bc)
    ctx.coarse_solve(bc, xc)
    ctx.gmres(bd, v, maxit=3)
    ctx.set_smoother("gmres", 6)
    ctx.vcycle(bd, v)
    torch.cuda.synchronize()
    print(f"{cfg.name}: n = {n}, n0 = {n0}, |V b| = {float(v.norm()):.6e}", flush=True)
    ctx.close()


if __name__ == "__main__":
    for c in CASES:
        run(*c)
    print("sanitize run complete")
