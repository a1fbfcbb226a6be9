"""Full-size parity, tier P-B, on the BASELINE.json configurations themselves (SURVEY
8(c.14); north star "on the largest 3D config"): the LIBRARY's own host setup and
CUDA path at full size (c3: 256^2 velocity, c4: 32^3 x 6 E-B, c5: 48^3 x 6 velocity, the
launch configuration bench.py times) against golden values that tools/golden_full.py
computed from the ORACLE alone (exact build, reading R-exact) and stored under
tests/golden/<cfg>_full_seed0.json:

  * every level's operator (P-A): sha256 of rowptr | col | val;
  * one Schwarz sweep from x = 0 and one V-cycle V(2,2) on the seed-0 right-hand side:
    sha256 of the whole float64 result (bit-exact, so relative l2 = 0 <= 1e-10), the
    l2 norm, and 4096 sampled entries -- which give the sampled relative difference
    should the hashes ever disagree.
"""
import hashlib
import json
import os

import numpy as np
import pytest

from gpu_helpers import cuda_vec, host

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def _sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def _check(got, ref, idx, what):
    got = np.asarray(got, dtype="<f8")
    ref_bits = np.array([int(s, 16) for s in ref["sample_bits"]], dtype=np.uint64)
    ref_vals = ref_bits.view(np.float64)
    samp = got[idx]
    rel = np.linalg.norm(samp - ref_vals) / np.linalg.norm(ref_vals)
    assert rel <= 1e-10, f"{what}: sampled relative l2 {rel:.3e}"
    assert abs(np.linalg.norm(got) - ref["norm"]) <= 1e-12 * ref["norm"], what
    assert np.array_equal(samp.view(np.uint64), ref_bits), f"{what}: sampled entries not bit-exact"
    assert _sha(got) == ref["sha256"], f"{what}: not bit-exact (sampled rel l2 {rel:.3e})"


@pytest.mark.parametrize("name", ["c3", "c4", "c5"])
def test_full_size_against_oracle_golden(name):
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    path = os.path.join(GOLDEN, f"{name}_full_seed0.json")
    if not os.path.exists(path):
        pytest.skip(f"{path} not generated (python tools/golden_full.py --config {name})")
    with open(path) as f:
        g = json.load(f)
    cfg = workloads.CONFIGS[name]
    assert (g["N"], g["levels"], g["seed"]) == (cfg.N, cfg.levels, 0)
    ctx = mhdp.Context(0, torch.cuda.current_stream().cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, 0)
    ctx.assemble(cfg, w)
    n = ctx.n()
    assert n == g["n"]
    _, b, _ = workloads.draw(cfg, n, 0)
    assert _sha(b.astype("<f8")) == g["b_sha256"]
    for li in g["levels_info"]:                       # P-A: the level operators
        rp, ci, v = ctx.csr(li["level"])
        assert (len(rp) - 1, len(v)) == (li["n"], li["nnz"])
        assert _sha(rp.astype("<i8"), ci.astype("<i4"), v.astype("<f8")) == li["sha256"], li["level"]
    ctx.setup()
    idx = np.asarray(g["sample_idx"], dtype=np.int64)
    bd = cuda_vec(b)
    xs = cuda_vec(np.zeros(n))
    ctx.smooth(bd, xs, nsweeps=1, x_is_zero=True)
    _check(host(xs), g["sweep"], idx, "sweep")
    xv = torch.empty(n, dtype=torch.float64, device="cuda:0")
    ctx.vcycle(bd, xv)
    _check(host(xv), g["vcycle"], idx, "V-cycle")
