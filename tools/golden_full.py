"""Golden values of the FULL c5 configuration (BASELINE.json configs[4]: 3D AL velocity
block, 48^3 x 6 tets, 4 levels, Re = gamma = 1e4) computed by the ORACLE alone.

Writes tests/golden/c5_full_seed0.json (SURVEY 8(c.14) "P-B one V-cycle" at c5; north
star "on the largest 3D config"):
  * per level: sha256 of the operator (rowptr int64 | col int32 | val float64, little
    endian) of the oracle's exact build (reading R-exact) -- P-A at full size;
  * one Schwarz sweep from x = 0 and one V-cycle V(2,2) on the seed-0 right-hand side:
    sha256 of the float64 result, its l2 norm and 4096 sampled entries (index, bits).
Only oracle/ and the seeded input module (paper_2104_14855_b200.workloads, which holds
no method arithmetic) are called.  Single-threaded exact assembly: about two hours.

    python tools/golden_full.py [--out tests/golden/c5_full_seed0.json]
"""
import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import oracle as om  # noqa: E402
from paper_2104_14855_b200 import workloads  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "tests", "golden", "c5_full_seed0.json"))
    ap.add_argument("--config", default="c5")
    ap.add_argument("--N", type=int, default=None)
    ap.add_argument("--levels", type=int, default=None)
    args = ap.parse_args()
    cfg = workloads.CONFIGS[args.config]
    if args.N is not None:
        cfg = workloads.small(args.config, args.N, args.levels or cfg.levels)
    seed = 0
    log = lambda *m: print(f"[{time.strftime('%H:%M:%S')}]", *m, flush=True)
    w, _, _ = workloads.draw(cfg, 1, seed)
    t0 = time.time()
    log("oracle exact build of", cfg)
    orc = om.Oracle(cfg, w, exact=True)
    n = orc.n()
    w2, b, _ = workloads.draw(cfg, n, seed)
    assert np.array_equal(w, w2)
    out = {"config": cfg.name, "N": cfg.N, "levels": cfg.levels, "seed": seed, "n": n,
           "block": cfg.block, "dim": cfg.dim, "oracle": "exact build (reading R-exact)",
           "levels_info": []}
    for l in range(orc.nlev):
        A = orc.csr(l)
        out["levels_info"].append({"level": l, "n": int(A.n), "nnz": int(len(A.v)),
                                   "sha256": sha(A.rp.astype("<i8"), A.ci.astype("<i4"), A.v.astype("<f8"))})
        log("level", l, "n", A.n, "nnz", len(A.v))
    out["setup_s"] = time.time() - t0
    rng = np.random.default_rng(123)
    idx = np.sort(rng.choice(n, size=min(4096, n), replace=False))
    out["sample_idx"] = idx.tolist()
    t1 = time.time()
    xs = orc.sweep(b, np.zeros(n), nsweeps=1, x_is_zero=True)
    out["sweep_s"] = time.time() - t1
    out["sweep"] = {"sha256": sha(xs.astype("<f8")), "norm": float(np.linalg.norm(xs)),
                    "sample_bits": [format(int(v), "016x") for v in xs[idx].view(np.uint64)]}
    log("sweep done")
    t2 = time.time()
    xv = orc.vcycle(b)
    out["vcycle_s"] = time.time() - t2
    out["vcycle"] = {"sha256": sha(xv.astype("<f8")), "norm": float(np.linalg.norm(xv)),
                     "sample_bits": [format(int(v), "016x") for v in xv[idx].view(np.uint64)]}
    log("vcycle done")
    out["b_sha256"] = sha(b.astype("<f8"))
    with open(args.out, "w") as f:
        json.dump(out, f, indent=1)
    log("wrote", args.out, "total", time.time() - t0, "s")


if __name__ == "__main__":
    main()
