"""Does the Burman stabilisation (reading R-mu) restore GMRES(V) convergence on
c5 at Re = gamma = 1e4?  Full c5 (48^3 x 6, 4 levels, V(2,2)), seed-0
right-hand side, GMRES(V) to max(1e-7 |b|, 1e-7) for several mu, with the
Richardson and the GMRES(6) smoother.   python tools/mu_study.py [maxit]"""
import dataclasses
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402

maxit = int(sys.argv[1]) if len(sys.argv) > 1 else 300
out = []
for mu in (0.0, 5e-3, 5e-2, 5e-1):
    cfg = dataclasses.replace(workloads.CONFIGS["c5"], mu=mu)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w)
    n = ctx.n()
    _, b, _ = workloads.draw(cfg, n, 0)
    ctx.setup()
    bd = torch.from_numpy(b).cuda()
    x = torch.empty_like(bd)
    rec = {"mu": mu}
    t = time.perf_counter()
    its, rel, conv = ctx.gmres(bd, x, maxit=maxit)
    rec["gmres_richardson"] = {"its": its, "relres": rel, "converged": conv, "s": time.perf_counter() - t,
                               "hist_every_50": ctx.last_history[::50].tolist()}
    ctx.set_smoother("gmres", 6)
    t = time.perf_counter()
    its, rel, conv = ctx.fgmres(bd, x, maxit=min(maxit, 100))
    rec["fgmres_gmres6"] = {"its": its, "relres": rel, "converged": conv, "s": time.perf_counter() - t}
    out.append(rec)
    print(json.dumps(rec), flush=True)
    ctx.close()
