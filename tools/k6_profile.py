"""K6 (batched patch LU, setup) timing: assemble a config with the library's host setup and
run mhdp_setup once (K6 on every level), for ncu:

  ncu --kernel-name regex:k_patch_lu --clock-control none --metrics \
      gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
      sm__inst_executed_pipe_fp64.sum --csv python tools/k6_profile.py c5

Without ncu it prints the wall time of mhdp_setup (host->device copies included).
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402


def main():
    name = sys.argv[1] if len(sys.argv) > 1 else "c5"
    cfg = workloads.CONFIGS[name]
    torch.cuda.set_device(0)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w = workloads.advecting_potential(cfg, None if cfg.dim == 2 else np.array([0.3, -1.1, 0.7]))
    ctx.assemble(cfg, w)
    t = time.perf_counter()
    ctx.setup()
    torch.cuda.synchronize()
    print(f"{name}: setup {time.perf_counter() - t:.3f} s, n = {ctx.n()}", flush=True)


if __name__ == "__main__":
    main()
