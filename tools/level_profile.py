"""Per-level, per-kernel timing of one configuration inside ONE process (CUDA events on
the launching stream, warm caches), so that kernel changes can be compared without the
box-to-box variance of separate bench runs.  Not part of the product or the tests.

    python tools/level_profile.py [c5|c4|c3|c2k2|c3k2|c4k2|c5k2] [reps]
"""
import dataclasses
import json
import os
import sys

sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402


def timed(fn, reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
    if name == "c2k2":
        cfg = dataclasses.replace(workloads.CONFIGS["c2"], N=512, levels=7, degree=2)
    elif name == "c3k2":
        cfg = dataclasses.replace(workloads.CONFIGS["c3"], N=256, levels=6, degree=2, sigma=40.0)
    elif name == "c5k2":
        cfg = dataclasses.replace(workloads.CONFIGS["c5"], N=24, levels=4, degree=2, sigma=40.0)
    elif name == "c4k2":
        cfg = dataclasses.replace(workloads.CONFIGS["c4"], degree=2)
    else:
        cfg = workloads.CONFIGS[name]
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w)
    w, b, x0 = workloads.draw(cfg, ctx.n(), 0)
    ctx.setup()
    L = ctx.num_levels()
    out = {"config": name, "env": {k: v for k, v in os.environ.items() if k.startswith("MHDP_")}, "levels": []}
    for lvl in range(L - 1, 0, -1):
        i = ctx.info(lvl)
        rng = np.random.default_rng(lvl)
        bl = torch.from_numpy(rng.uniform(-1, 1, i["n"])).cuda()
        xl = torch.from_numpy(rng.uniform(-1, 1, i["n"])).cuda()
        rl = torch.empty_like(bl)
        nc = ctx.info(lvl - 1)["n"]
        rc = torch.empty(nc, dtype=torch.float64, device="cuda")
        row = {"level": lvl, "n": i["n"], "npatch": i["npatch"], "max_n": i["max_n"]}
        row["K1_ms"] = timed(lambda: ctx.residual(bl, xl, rl, level=lvl), reps)
        row["K2_ms"] = timed(lambda: ctx.patch_apply(rl, level=lvl), reps)
        row["K3_ms"] = timed(lambda: ctx.patch_update(xl, level=lvl), reps)
        row["sweep_ms"] = timed(lambda: ctx.smooth(bl, xl, level=lvl, nsweeps=1), reps)
        row["restrict_ms"] = timed(lambda: ctx.restrict(rl, rc, level=lvl), reps)
        row["prolong_ms"] = timed(lambda: ctx.prolong_add(rc, xl, level=lvl), reps)
        row["K2_gbs"] = (8 * i["sum_n2"] + 16 * i["sum_n"]) / (row["K2_ms"] * 1e-3) / 1e9
        row["K1_gbs"] = (8 * i["nnz"] + 24 * i["n"]) / (row["K1_ms"] * 1e-3) / 1e9
        out["levels"].append(row)
    n0 = ctx.info(0)["n"]
    bc = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n0)).cuda()
    xc = torch.empty_like(bc)
    out["coarse_ms"] = timed(lambda: ctx.coarse_solve(bc, xc), reps)
    bd = torch.from_numpy(b).cuda()
    xd = torch.empty_like(bd)
    out["vcycle_ms"] = timed(lambda: ctx.vcycle(bd, xd), reps)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
