"""Report max kappa_2(A_i) of the vertex-star patch matrices per level (SURVEY §8(c) test
plan: "max kappa(A_i) per level reported (dense SVD in the oracle; c5 via a sample of
>= 1000 patches incl. all boundary size classes)").  Operators and patches come from the
oracle (fp64 build); A_i = R_i A R_i^T is formed from the CSR and its 2-norm
condition number computed by a dense SVD.  The finest c5 level is sampled: >= 1000
patches, every size class included, assembled by the oracle's masked assembly around the
sampled vertices (rows of the patch DoFs are then exact).  Not part of the product.

    python tools/kappa_report.py [out.json]      (CPU, a few minutes)
"""
import dataclasses
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

from oracle import oracle as om  # noqa: E402
from paper_2104_14855_b200 import workloads  # noqa: E402

U = 2.0 ** -53


def patch_kappas(A, ptr, dofs, idx=None):
    A = A.tocsr()
    idx = range(len(ptr) - 1) if idx is None else idx
    out = []
    for i in idx:
        d = dofs[ptr[i]:ptr[i + 1]]
        s = np.linalg.svd(A[d][:, d].toarray(), compute_uv=False)
        out.append((len(d), float(s[0] / s[-1])))
    return out


def summarize(ks):
    by = {}
    for n, k in ks:
        by.setdefault(n, []).append(k)
    return {"patches": len(ks), "max_kappa": max(k for _, k in ks), "max_kappa_times_u": max(k for _, k in ks) * U,
            "median_kappa": float(np.median([k for _, k in ks])),
            "by_size": {str(n): {"count": len(v), "max": max(v)} for n, v in sorted(by.items())}}


def level_report(cfg):
    w, _, _ = workloads.draw(cfg, 1, 0)
    o = om.Oracle(cfg, w)
    rep = []
    for lev in range(1, o.nlev):
        ptr, dofs, _, _ = o.patches(lev)
        rep.append(dict(level=lev, N=cfg.N >> (o.nlev - 1 - lev), n=o.n(lev),
                        **summarize(patch_kappas(o.csr(lev).to_scipy(), ptr, dofs))))
    return rep


def c5_finest_sample(nsample=1000, seed=5):
    from test_gpu_parity import _mask_around, _patch_vertices
    cfg = workloads.CONFIGS["c5"]
    w, _, _ = workloads.draw(cfg, 1, 0)
    pverts = _patch_vertices(cfg)
    N = cfg.N
    lat = np.stack([pverts % (N + 1), (pverts // (N + 1)) % (N + 1), pverts // (N + 1) ** 2], axis=1)
    cls = ((lat == 0) | (lat == N)).sum(axis=1)          # 0 interior, 1 face, 2 edge, 3 corner
    rng = np.random.default_rng(seed)
    pick = []
    for c in range(4):                                      # every boundary class, then fill
        ids = np.flatnonzero(cls == c)
        pick.extend(rng.choice(ids, size=min(len(ids), 60), replace=False).tolist())
    rest = np.setdiff1d(np.arange(len(pverts)), pick)
    pick = np.unique(np.concatenate([pick, rng.choice(rest, size=nsample - len(pick), replace=False)]))
    mask = _mask_around(cfg, pverts[pick])
    o = om.Oracle(cfg, w, nlev=1, cmask=mask)
    ptr, dofs, verts, _ = o.patches()
    pos = {int(v): i for i, v in enumerate(verts)}
    idx = [pos[int(v)] for v in pverts[pick]]
    return dict(level=3, N=N, n=o.n(), sampled=True, **summarize(patch_kappas(o.csr().to_scipy(), ptr, dofs, idx)))


def main():
    out = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "profiles", "kappa_report.json")
    t0 = time.time()
    rep = {"note": "max kappa_2(A_i) of the star patch matrices per level (oracle operators, dense SVD); "
                   "kappa u bounds the relative perturbation a patch solve amplifies (SURVEY c.13)"}
    for name in ("c1", "c2", "c3", "c4"):
        rep[name] = level_report(workloads.CONFIGS[name])
        print(name, [(r["level"], f'{r["max_kappa"]:.2e}') for r in rep[name]], flush=True)
    rep["c5"] = level_report(workloads.small("c5", 24, 3))      # levels 1 (12^3) and 2 (24^3) of c5
    rep["c5"].append(c5_finest_sample())
    print("c5", [(r["level"], f'{r["max_kappa"]:.2e}') for r in rep["c5"]], flush=True)
    # NEXT-2 (k = 2): 2D CG2 x RT2 / BDM2, 3D NED1_2 x RT2 (280-DoF stars) / BDM2 (360)
    k2 = {"c2k2": dataclasses.replace(workloads.small("c2", 64, 3), degree=2),
          "c3k2": dataclasses.replace(workloads.small("c3", 64, 3), degree=2, sigma=40.0),
          "c4k2": dataclasses.replace(workloads.small("c4", 8, 3), degree=2),
          "c5k2": dataclasses.replace(workloads.small("c5", 8, 3), degree=2, sigma=40.0)}
    for name, cfg in k2.items():
        rep[name] = level_report(cfg)
        print(name, [(r["level"], f'{r["max_kappa"]:.2e}') for r in rep[name]], flush=True)
    rep["seconds"] = time.time() - t0
    json.dump(rep, open(out, "w"), indent=1)


if __name__ == "__main__":
    main()
