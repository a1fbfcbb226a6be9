"""Device setup timings (mhdp_setup_timings) of a configuration: K6 per level, K7, K8 pack,
wall time, with flop rates against the measured FP64 peak.   python tools/setup_profile.py [c5]"""
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402
import probe  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c5"
cfg = workloads.CONFIGS[name]
ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
w, _, _ = workloads.draw(cfg, 1, 0)
ctx.assemble(cfg, w)
ctx.setup()
t = ctx.setup_timings()
peak = probe.fp64_peak(0)
L = ctx.num_levels()
out = {"config": name, "fp64_peak_tflops": peak / 1e12, "K7_ms": t["K7_ms"], "K8_pack_ms": t["K8_pack_ms"],
       "wall_s": t["wall_s"], "host_stage_s": t["host_stage_s"], "K6": []}
n0 = ctx.n(0)
out["K7_tflops"] = (2 / 3) * n0 ** 3 / (t["K7_ms"] * 1e-3) / 1e12
for l in range(1, L):
    ptr, _ = ctx.patches(l)
    sz = np.diff(ptr).astype(np.float64)
    fl = (2 / 3) * float(np.sum(sz ** 3))
    out["K6"].append({"level": l, "ms": t["K6_ms"][l], "tflops": fl / (t["K6_ms"][l] * 1e-3) / 1e12})
print(json.dumps(out))
