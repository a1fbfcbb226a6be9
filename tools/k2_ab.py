import sys, os, time, json, dataclasses
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
from paper_2104_14855_b200 import mhdp, workloads
cfg2 = dataclasses.replace(workloads.CONFIGS["c2"], N=512, levels=7, degree=2)
ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
w, _, _ = workloads.draw(cfg2, 1, 0)
ctx.assemble(cfg2, w)
w, b, x = workloads.draw(cfg2, ctx.n(), 0)
ctx.setup()
bd = torch.from_numpy(b).cuda(); xd = torch.from_numpy(x).cuda(); rd = torch.empty_like(bd)
ctx.residual(bd, xd, rd)
out = {"env": os.environ.get("MHDP_K2", "tma")}
for lvl in range(ctx.num_levels() - 1, 0, -1):
    bl = torch.from_numpy(np.random.default_rng(lvl).uniform(-1, 1, ctx.info(lvl)["n"])).cuda()
    ctx.patch_apply(bl, level=lvl) if 'level' in ctx.patch_apply.__code__.co_varnames else None
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        ctx.patch_apply(bl, level=lvl)
    e1.record(); torch.cuda.synchronize()
    i = ctx.info(lvl)
    ms = e0.elapsed_time(e1) / 20
    out[f"L{lvl}"] = {"ms": ms, "gbs": (8 * i["sum_n2"] + 16 * i["sum_n"]) / (ms * 1e-3) / 1e9, "np": i["npatch"]}
xs = xd.clone()
ctx.vcycle(bd, xs); torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.vcycle(bd, xs)
e1.record(); torch.cuda.synchronize()
out["vcycle_ms"] = e0.elapsed_time(e1) / 10
print(json.dumps(out))
