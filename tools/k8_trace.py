"""K8 (coarse LU solve) timing and per-block trace on a c5-sized coarse operator.

python tools/k8_trace.py [N]   (c5 family, one level of N^3 x 6 tets; N = 6 -> n0 = 7128,
the coarse level of the full c5 hierarchy).  Prints the CUDA-event time per solve and,
from mhdp_coarse_solve_trace, per pass: total span, mean chain time per block, mean
stall of the chain between blocks, claim waits and far-warp hand-off slack.
"""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])
from paper_2104_14855_b200 import mhdp, workloads  # noqa: E402


def main():
    N = int(sys.argv[1]) if len(sys.argv) > 1 else 6
    cfg = workloads.small("c5", N, 1)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w)
    ctx.setup()
    n = ctx.n(0)
    b = torch.from_numpy(np.random.default_rng(0).uniform(-1, 1, n)).cuda()
    x = torch.empty_like(b)
    for _ in range(3):
        ctx.coarse_solve(b, x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        ctx.coarse_solve(b, x)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    tr = ctx.coarse_solve_trace(b, x).astype(np.float64)
    t0 = tr[0, 0, 0]
    LFs = 7   # k8_lf() in k8_coarse.cu
    out = {"n0": n, "ms_per_solve": ms}
    for p, name in ((0, "forward"), (1, "back")):
        T = tr[p] - t0
        nb = T.shape[0]
        chain = T[:, 3] - T[:, 2]
        gap = T[1:, 2] - T[:-1, 3]
        claim = T[:, 1] - T[:, 0]
        far = T[:, 4]
        slack = np.where(far > 0, T[:, 0] - far, np.nan)   # > 0: far hand-off arrived before the claim started
        out[name] = {"span_us": (T[:, 3].max() - T[:, 2].min()) / 1e3, "blocks": nb,
                     "chain_ns_mean": float(chain.mean()), "gap_ns_mean": float(gap.mean()),
                     "gap_ns_p90": float(np.percentile(gap, 90)), "claim_ns_mean": float(claim.mean()),
                     "claim_ns_max": float(claim.max()),
                     "far_slack_ns_min": float(np.nanmin(slack)) if np.isfinite(slack).any() else None,
                     "far_slack_ns_median": float(np.nanmedian(slack)) if np.isfinite(slack).any() else None}
        catch_done = T[1:, 13] - T[:-1, 3]   # > 0: block r+1's catch-up ended after block r finished
        out[name]["catchup_end_minus_prev_chain_end_ns_median"] = float(np.median(catch_done))
        out[name]["catchup_ns_median"] = float(np.median(T[:, 13] - T[:, 1]))
        out[name]["claim_start_minus_prev_chain_end_ns_median"] = float(np.median(T[1:, 0] - T[:-1, 3]))
        out[name]["catchup_wait_cycles_median"] = float(np.median(tr[p][LFs:, 14]))
        out[name]["catchup_total_cycles_median"] = float(np.median(tr[p][LFs:, 15]))
        ref = np.concatenate([[np.nan], T[:-1, 3]])            # chain end of block r-1
        rel = lambda k: float(np.nanmedian((T[LFs + 1:, k] - ref[LFs + 1:]) / 1e3))
        out[name]["rel_to_prev_chain_end_us"] = {"claim_start": rel(0), "far_handoff": rel(4), "claim_done": rel(1),
                                                  "catchup_done": rel(13), "chain_start": rel(2), "chain_end": rel(3)}
        mbc = tr[p][:, 5:13]
        out[name]["minib_cycles_cum_median"] = [float(v) for v in np.median(mbc, axis=0)]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
