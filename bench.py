"""Benchmark of the vertex-star Schwarz smoother / V-cycle (arXiv 2104.14855) on B200.

Workload (BASELINE.json configs[4], the largest 3D configuration, which fits one GPU):
  c5 = 3D augmented-Lagrangian velocity block, 48^3 cubes x 6 Kuhn tets, BDM1,
  Re = gamma = 1e4, 4 levels, V(2,2), vertex-star patches (108 DoFs interior).
A step is one V-cycle(2,2) of the whole hot path (residual SpMV,
patch gather + LU apply, weighted gather-update on every level, restriction,
prolongation, dense coarse solve).  Setup (a0-a2: host assembly, batched patch LU,
coarse LU) runs once before the timed region.

metric: smoothed DoFs/s in SURVEY A26's sense -- free DoFs of the finest level per sweep,
(nu_pre + nu_post) n_finest per V-cycle -- plus the V-cycle ms, a finest-level single
sweep's DoFs/s and its achieved HBM GB/s (SURVEY §8(d) algorithmic bytes) against
MEASURED_PEAKS.json.  `value_all_levels` counts every level's sweeps (sum_l (nu_pre +
nu_post) n_l), the round-1 definition.

Multi-GPU: the method runs on one GPU (BASELINE north star); --gpus N runs N independent
replicas (one process per GPU, each its own seeded right-hand side), "replicas only" in
DESIGN.md, weak scaling with no data-path collective; the step time is the max over ranks.

--impl reference: the reference arm is the ORACLE (plain single-threaded C) as it stands,
timed on the host on a bounded sample of the same workload family (c5 at N = 12, 3
levels, V(2,2); setup excluded), same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

REF_SAMPLE = ("c5", 12, 3)


def k2_traffic():
    """DRAM bytes per K2 launch from the committed `ncu --set full` capture (profiles/), or None."""
    p = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "k2_traffic.json")
    try:
        with open(p) as f:
            return json.load(f)
    except (OSError, ValueError):
        return None


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return None


def fp64_peak_flops(device=0):
    """FP64 FMA throughput of the GPU measured by tools/probe.cu ("FP64 peak
    is not in MP. Measure it"), or None when the probe library is missing."""
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import probe
        v = probe.fp64_peak(device)
        return v if v > 0 else None
    except Exception:
        return None


def host_info():
    """CPU model, logical cores and a single-thread STREAM-copy figure of the host the
    oracle baseline runs on."""
    model = "unknown"
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    a = np.ones(1 << 25)            # 256 MB
    b = np.empty_like(a)
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        np.copyto(b, a)
        best = min(best, time.perf_counter() - t)
    return {"cpu_model": model, "nproc": os.cpu_count(),
            "stream_copy_gbs_1thread": 2 * a.nbytes / best / 1e9}


def oracle_full_size_record():
    """Full-size oracle timings recorded by tools/golden_full.py (the exact build, one
    core, on the build container -- not this host), when the golden file exists."""
    p = os.path.join(ROOT, "tests", "golden", "c5_full_seed0.json")
    try:
        g = json.load(open(p))
    except (OSError, ValueError):
        return None
    return {"config": "c5 full (48^3 x 6, 4 levels)", "setup_s": g.get("setup_s"), "sweep_s": g.get("sweep_s"),
            "vcycle_s": g.get("vcycle_s"), "cores": 1, "where": "build container (tools/golden_full.py), exact build",
            "vcycle_dofs_per_s": (4 * g["n"] / g["vcycle_s"]) if g.get("vcycle_s") else None}


_SAMPLER_SRC = r"""
import sys, time, json
idx, out = int(sys.argv[1]), sys.argv[2]
names = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
         0x80: "hw_power_brake_slowdown"}
rows = []
try:
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(idx)
    mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
    src = "nvml"
    def sample():
        bits = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        return [nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), mx, [v for k, v in names.items() if bits & k]]
except Exception:
    import subprocess
    src = "nvidia-smi"
    q = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
        "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"
    nm = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    def sample():
        p = subprocess.run(["nvidia-smi", "-i", str(idx), "--query-gpu=" + q, "--format=csv,noheader,nounits"],
                           capture_output=True, text=True, timeout=5).stdout.strip().split(",")
        p = [x.strip() for x in p]
        return [float(p[0]), float(p[1]), [nm[i] for i in range(4) if p[2 + i] == "Active"]]
sys.stdout.write("ready\n"); sys.stdout.flush()
while True:
    try:
        rows.append(sample())
    except Exception:
        pass
    if sys.stdin in __import__("select").select([sys.stdin], [], [], 0.005 if src == "nvml" else 0.2)[0]:
        break
json.dump({"source": src, "rows": rows}, open(out, "w"))
"""


class ClockSampler:
    """SM clocks and clock-event (throttle) reasons sampled during the timed region by a
    separate process (no GIL contention with the timed loop): NVML every 5 ms, else
    nvidia-smi every 200 ms."""

    def __init__(self, index=0):
        self.index = index
        self.samples = []
        self.source = None
        self._p = None
        self._out = None

    def __enter__(self):
        import tempfile
        fd, self._out = tempfile.mkstemp(suffix=".json")
        os.close(fd)
        try:
            self._p = subprocess.Popen([sys.executable, "-c", _SAMPLER_SRC, str(self.index), self._out],
                                       stdin=subprocess.PIPE, stdout=subprocess.PIPE, text=True)
            self._p.stdout.readline()          # sampler initialised
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        try:
            self._p.stdin.write("stop\n")
            self._p.stdin.flush()
            self._p.wait(timeout=20)
            with open(self._out) as f:
                d = json.load(f)
            self.samples, self.source = d["rows"], d["source"]
        except Exception:
            pass
        finally:
            try:
                os.unlink(self._out)
            except OSError:
                pass

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"], "samples": 0}
        sm = [float(x[0]) for x in self.samples]
        return {"sm_mhz": float(np.median(sm)), "sm_min_mhz": min(sm), "sm_max_mhz": max(float(x[1]) for x in self.samples),
                "reasons": sorted({r for x in self.samples for r in x[2]}), "samples": len(self.samples),
                "source": self.source}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def max_over_ranks(x: float, device=None) -> float:
    """Max of a per-rank time over all ranks (identity without a process group).  Each
    rank runs an independent replica (replicas only), so the whole-job step
    time is the slowest replica's."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def replica_seed(base: int, rank: int) -> int:
    """Seed of the right-hand side of rank `rank`'s replica."""
    return base + rank


# ----------------------------------------------------------------------------------------
# reference arm: the oracle
# ----------------------------------------------------------------------------------------
def oracle_vcycle_sample(steps, warmup, seed=0):
    from oracle import oracle
    from paper_2104_14855_b200 import workloads
    name, N, L = REF_SAMPLE
    cfg = workloads.small(name, N, L)
    w0, _, _ = workloads.draw(cfg, 1, seed)
    orc = oracle.Oracle(cfg, w0)
    w, b, _ = workloads.draw(cfg, orc.n(), seed)
    ts = time.perf_counter()
    orc = oracle.Oracle(cfg, w)
    orc.vcycle(b)                       # factors every level (lazy) -- setup, not timed
    setup_s = time.perf_counter() - ts
    for _ in range(max(0, warmup - 1)):
        orc.vcycle(b)
    smoothed = 2 * cfg.nu * orc.n()              # A26: finest-level DoFs per sweep
    t0 = time.perf_counter()
    for _ in range(steps):
        orc.vcycle(b)
    dt = (time.perf_counter() - t0) / steps
    return {"value": smoothed / dt, "ms_per_step": dt * 1e3, "smoothed_per_step": smoothed,
            "setup_s": setup_s,
            "sample": f"oracle V(2,2) on {name} at N={N}, {L} levels ({orc.n()} finest DoFs; same element, "
                      f"patch and operator structure as the full c5), setup excluded, {steps} cycles"}


METRIC = "smoothed DoFs/s (V(2,2) cycle); achieved HBM GB/s vs peak; V-cycle ms"


def workload_config(cfg, L=None, fin=None, ws=1):
    """The `config` object of both arms (BASELINE.json's metric is quoted on c5)."""
    c = {"workload": f"{cfg.name}: 3D AL velocity block, BDM1, {cfg.N}^3 x 6 tets, {L or cfg.levels} levels, "
                     f"V({cfg.nu},{cfg.nu}), Re=gamma=1e4",
         "parallelism": f"replicas x{ws}" if ws > 1 else "single GPU",
         "l2": "working set per step >> L2 (9.9 GB of patch factors streamed per sweep)"}
    if fin is not None:
        c.update({"finest_dofs": fin["n"], "nnz": fin["nnz"], "patches": fin["npatch"], "sum_n2": fin["sum_n2"]})
    return c


def run_reference(args):
    ws, rank, _ = dist_init()
    if rank != 0:
        return
    from paper_2104_14855_b200 import workloads
    r = oracle_vcycle_sample(args.steps, args.warmup)
    cfg = dict(workload_config(workloads.CONFIGS[args.config]), sample=r["sample"])
    line = {"impl": "reference", "metric": METRIC, "value": r["value"],
            "unit": "DoF/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": r["ms_per_step"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": cfg,
            "cpu_baseline": {"value": r["value"], "unit": "DoF/s", "cores": 1, "kind": "oracle", "sample": r["sample"]},
            "e2e": {"value": r["value"], "unit": "DoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------------------
def _timed(stream, fn, reps=1):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        out = fn()
    e1.record(stream)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


def _k2_variant(cfg, seed, dev, stream, desc):
    """one NEXT-2 (k = 2) hierarchy: host assembly, V-cycle, K2, sweep, GMRES(6)-smoothed FGMRES"""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    ctx = mhdp.Context(dev.index, stream.cuda_stream)
    w, _, _ = workloads.draw(cfg, 1, seed)
    t0 = time.perf_counter()
    ctx.assemble(cfg, w)
    t_asm = time.perf_counter() - t0
    w, b, x = workloads.draw(cfg, ctx.n(), seed)
    t0 = time.perf_counter()
    ctx.setup()
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    L = ctx.num_levels()
    fin = ctx.info(L - 1)
    bd = torch.from_numpy(b).to(dev)
    xd = torch.from_numpy(x).to(dev)
    ctx.vcycle(bd, xd)
    ms_v, _ = _timed(stream, lambda: ctx.vcycle(bd, xd), reps=10)
    rd = torch.empty_like(bd)
    ctx.residual(bd, xd, rd)
    ctx.patch_apply(rd)
    ms_k2, _ = _timed(stream, lambda: ctx.patch_apply(rd), reps=10)
    ms_sw, _ = _timed(stream, lambda: ctx.smooth(bd, xd, nsweeps=1), reps=10)
    k2_bytes = 8 * fin["sum_n2"] + 16 * fin["sum_n"]
    sweep_bytes = 8 * fin["sum_n2"] + 8 * fin["nnz"] + 24 * fin["n"]
    ctx.set_smoother("gmres", 6)
    ms_f, (its, rel, conv) = _timed(stream, lambda: ctx.fgmres(bd, xd, maxit=60))
    smoothed = 2 * cfg.nu * fin["n"]             # A26: finest-level DoFs per sweep
    ctx.close()
    return {"config": desc, "finest_dofs": fin["n"], "nnz": fin["nnz"], "patches": fin["npatch"],
            "max_patch": fin["max_n"], "sum_n2": fin["sum_n2"], "factor_gb": 8e-9 * fin["sum_n2"],
            "host_assembly_s": t_asm, "device_setup_s": t_setup,
            "vcycle_ms": ms_v, "smoothed_dofs_per_s": smoothed / (ms_v * 1e-3),
            "sweep_ms": ms_sw, "sweep_gbs": sweep_bytes / (ms_sw * 1e-3) / 1e9,
            "K2_ms": ms_k2, "K2_gbs": k2_bytes / (ms_k2 * 1e-3) / 1e9,
            "fgmres_gmres6_vcycle": {"its": its, "converged": conv, "relres": rel, "ms": ms_f}}


def run_configs(seed, dev, stream):
    """SURVEY 8(d) "per config": the other BASELINE.json configurations (c1-c4) on the same
    kernels -- V-cycle ms (median of 20 after 3 warm-ups), finest sweep ms, finest K2
    algorithmic GB/s and fraction of the measured HBM peak, A26 DoFs/s.  Setup excluded."""
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    out = {}
    for name in ("c1", "c2", "c3", "c4"):
        cfg = workloads.CONFIGS[name]
        ctx = mhdp.Context(dev.index, stream.cuda_stream)
        w, _, _ = workloads.draw(cfg, 1, seed)
        ctx.assemble(cfg, w)
        n = ctx.n()
        _, b, x0 = workloads.draw(cfg, n, seed)
        ctx.setup()
        fin = ctx.info(ctx.num_levels() - 1)
        bd = torch.from_numpy(b).to(dev)
        xd = torch.empty_like(bd)
        for _ in range(3):
            ctx.vcycle(bd, xd)
        ts = []
        for _ in range(20):
            t, _ = _timed(stream, lambda: ctx.vcycle(bd, xd))
            ts.append(t)
        ms_v = float(np.median(ts))
        xs = torch.from_numpy(x0).to(dev)
        ms_s, _ = _timed(stream, lambda: ctx.smooth(bd, xs, nsweeps=1), reps=20)
        rd = torch.empty_like(bd)
        ctx.residual(bd, xs, rd)
        ms_k2, _ = _timed(stream, lambda: ctx.patch_apply(rd), reps=20)
        k2_bytes = 8 * fin["sum_n2"] + 16 * fin["sum_n"]
        out[name] = {"finest_dofs": n, "levels": ctx.num_levels(), "vcycle_ms": ms_v, "sweep_ms": ms_s,
                     "K2_ms": ms_k2, "K2_gbs": k2_bytes / (ms_k2 * 1e-3) / 1e9,
                     "K2_frac": k2_bytes / (ms_k2 * 1e-3) / 1e9 / peak,
                     "dofs_per_s": 2 * cfg.nu * n / (ms_v * 1e-3)}
        ctx.close()
    return out


def run_variants(cfg, seed, dev, stream):
    """NEXT-2: the k = 2 (CG2 x RT2) 2D E-B block at 512^2 (V-cycle, sweep, K2, FGMRES).
    NEXT-4: the c5 operator in the transient (implicit Euler, dt = 0.01 as P:656) Newton
    variant with the Lorentz term of a seeded B^n (S = 1): V-cycle time and the paper's
    FGMRES(GMRES(6)-smoothed V) solve.  NEXT-3: the coupled 4x4 Newton system (3D, 24^3,
    3 levels, Picard, Re = Re_m = 10, S = 1, gamma = 100) solved by outer FGMRES with the
    block upper-triangular preconditioner (inner FGMRES(2) solves).  Setup excluded."""
    import dataclasses
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    out = {}
    cfg4 = dataclasses.replace(cfg, dt=0.01, S=1.0)
    ctx = mhdp.Context(dev.index, stream.cuda_stream)
    w, b, _ = workloads.draw(cfg4, 1, seed)
    ctx.assemble(cfg4, w, bn=workloads.magnetic_potential(cfg4, seed))
    w, b, _ = workloads.draw(cfg4, ctx.n(), seed)
    ctx.setup()
    bd = torch.from_numpy(b).to(dev)
    xd = torch.empty_like(bd)
    ctx.vcycle(bd, xd)
    ms_v, _ = _timed(stream, lambda: ctx.vcycle(bd, xd), reps=5)
    ctx.set_smoother("gmres", 6)
    ms_f, (its, rel, conv) = _timed(stream, lambda: ctx.fgmres(bd, xd, maxit=60))
    out["next4_c5_transient_lorentz"] = {
        "config": "c5 operator + (1/dt)(u,v), dt = 0.01, + S(u x B^n, v x B^n), S = 1", "vcycle_ms": ms_v,
        "fgmres_gmres6_vcycle": {"its": its, "converged": conv, "relres": rel, "ms": ms_f}}
    ctx.close()
    del ctx
    cfg3 = dataclasses.replace(workloads.small("c5", 24, 3), Re=10.0, Rem=10.0, S=1.0, gamma=100.0, picard=1)
    w3, _, _ = workloads.draw(cfg3, 1, seed)
    co = mhdp.Coupled(cfg3, w3, workloads.magnetic_potential(cfg3, seed), device=dev.index,
                      stream=stream.cuda_stream, smoother="gmres", smoother_its=6)
    r = np.random.default_rng(seed).standard_normal(co.n)
    r[co.nu:co.nu + co.np_] -= r[co.nu:co.nu + co.np_].mean()     # consistent: Q = L^2_0
    rd = torch.from_numpy(r).to(dev)
    yd = torch.empty_like(rd)
    co.precondition(rd, yd)
    ms_p, _ = _timed(stream, lambda: co.precondition(rd, yd), reps=3)
    ms_o, (its3, rel3, conv3) = _timed(stream, lambda: co.fgmres(rd, yd, maxit=40))
    out["next3_coupled_outer"] = {
        "config": "3D 24^3 x 6 tets, 3 levels, Picard, Re = Re_m = 10, S = 1, gamma = 100",
        "dofs": {"u": co.nu, "p": co.np_, "E": co.nE, "B": co.nB}, "precondition_ms": ms_p,
        "fgmres": {"its": its3, "converged": conv3, "relres": rel3, "ms": ms_o}}
    co.close()
    # NEXT-2: k = 2, the paper's element degree, on both blocks (2D) and the 3D E-B block
    out["next2_k2_eb2d"] = _k2_variant(
        dataclasses.replace(workloads.CONFIGS["c2"], N=512, levels=7, degree=2), seed, dev, stream,
        "2D E-B block, CG2 x RT2 (k = 2), 512^2 x 2 cells, 7 levels, V(2,2), Re_m = S = 1e3")
    out["next2_k2_vel2d"] = _k2_variant(
        dataclasses.replace(workloads.CONFIGS["c3"], N=256, levels=6, degree=2, sigma=40.0), seed, dev, stream,
        "2D AL velocity block, BDM2 (k = 2), 256^2 x 2 cells, 6 levels, V(2,2), Re = gamma = 1e4, sigma = 40")
    out["next2_k2_eb3d"] = _k2_variant(
        dataclasses.replace(workloads.CONFIGS["c4"], degree=2, picard=1), seed, dev, stream,
        "3D E-B block, NED1_2 x RT2 (k = 2), 32^3 x 6 cells, 4 levels, V(2,2), Re_m = S = 1e3, Picard "
        "(280-DoF stars; the Newton block at Re_m >= 100 is not solved by the star V-cycle, DESIGN 9d)")
    out["next2_k2_vel3d"] = _k2_variant(
        dataclasses.replace(workloads.CONFIGS["c5"], N=24, levels=4, degree=2, sigma=40.0), seed, dev, stream,
        "3D AL velocity block, BDM2 (k = 2), 24^3 x 6 cells, 4 levels, V(2,2), Re = gamma = 1e4, sigma = 40 "
        "(360-DoF stars; 24^3 bounds the double-double host assembly time)")
    return out


def run_ours(args):
    import torch
    from paper_2104_14855_b200 import mhdp, workloads
    ws, rank, local = dist_init()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if torch.cuda.is_available() else "gloo")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = workloads.CONFIGS[args.config]
    stream = torch.cuda.current_stream(dev)
    ctx = mhdp.Context(local, stream.cuda_stream)
    seed = replica_seed(args.seed, rank)
    t0 = time.perf_counter()
    w0, _, _ = workloads.draw(cfg, 1, seed)
    ctx.assemble(cfg, w0)
    t_asm = time.perf_counter() - t0
    n = ctx.n()
    w, b, x0 = workloads.draw(cfg, n, seed)
    t0 = time.perf_counter()
    ctx.setup()
    t_setup = time.perf_counter() - t0
    L = ctx.num_levels()
    infos = [ctx.info(l) for l in range(L)]
    fin = infos[-1]
    smoothed = (cfg.nu + cfg.nu) * fin["n"]                                    # A26
    smoothed_all = sum((cfg.nu + cfg.nu) * infos[l]["n"] for l in range(1, L))  # every level
    # setup kernels against the FP64 FMA peak: K6 (2/3) sum_i n_i^3 per level,
    # K7 (2/3) n0^3
    stt = ctx.setup_timings()
    fp64 = fp64_peak_flops(dev.index)
    k6 = []
    for l in range(1, L):
        ptr, _ = ctx.patches(l)
        sz = np.diff(ptr).astype(np.float64)
        fl = float((2.0 / 3.0) * np.sum(sz ** 3))
        ms6 = stt["K6_ms"][l]
        k6.append({"level": l, "ms": ms6, "flop": fl, "tflops": fl / (ms6 * 1e-3) / 1e12 if ms6 > 0 else None})
    n0c = infos[0]["n"]
    fl7 = (2.0 / 3.0) * float(n0c) ** 3
    setup_kernels = {
        "fp64_peak_tflops": fp64 / 1e12 if fp64 else None,
        "fp64_peak_source": "tools/probe.cu: DFMA chains on every SM (measured in this run)",
        "K6_patch_lu": k6,
        "K6_finest_frac_fp64_peak": (k6[-1]["tflops"] * 1e12 / fp64) if (fp64 and k6 and k6[-1]["tflops"]) else None,
        "K6_all_levels_ms": float(sum(k["ms"] for k in k6)),
        "K7_coarse_lu": {"n0": n0c, "ms": stt["K7_ms"], "flop": fl7,
                         "tflops": fl7 / (stt["K7_ms"] * 1e-3) / 1e12 if stt["K7_ms"] > 0 else None,
                         "frac_fp64_peak": (fl7 / (stt["K7_ms"] * 1e-3) / fp64) if (fp64 and stt["K7_ms"] > 0) else None},
        "K8_pack_ms": stt["K8_pack_ms"], "device_setup_wall_s": stt["wall_s"]}

    bd = torch.from_numpy(b).to(dev)
    xd = torch.empty_like(bd)
    x0d = torch.from_numpy(x0).to(dev)

    def barrier():
        if ws > 1:
            import torch.distributed as dist
            dist.barrier()

    # ---- V-cycle (the step) ----
    for _ in range(args.warmup):
        ctx.vcycle(bd, xd)
    torch.cuda.synchronize(dev)
    barrier()
    torch.cuda.synchronize(dev)
    l0 = ctx.launch_count()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            ctx.vcycle(bd, xd)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    launches = ctx.launch_count() - l0
    ms = ev0.elapsed_time(ev1) / args.steps
    barrier()
    ms = max_over_ranks(ms, dev)

    # ---- finest single sweep (K1+K2+K3) and the dominant kernel K2 alone ----
    reps = max(3, args.steps)
    xs = x0d.clone()
    ctx.smooth(bd, xs, nsweeps=1)
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(reps):
        ctx.smooth(bd, xs, nsweeps=1)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_sweep = e0.elapsed_time(e1) / reps
    rd = torch.empty_like(bd)
    ctx.residual(bd, x0d, rd)
    ctx.patch_apply(rd)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(reps):
        ctx.patch_apply(rd)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_k2 = e0.elapsed_time(e1) / reps
    e0.record(stream)
    for _ in range(reps):
        ctx.residual(bd, x0d, rd)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_k1 = e0.elapsed_time(e1) / reps
    # one sweep on every level (where the V-cycle's time goes besides the finest level)
    level_sweep_ms = []
    for l in range(1, L):
        nl = infos[l]["n"]
        bl = torch.from_numpy(np.random.default_rng(l).uniform(-1, 1, nl)).to(dev)
        xl = torch.zeros_like(bl)
        ctx.smooth(bl, xl, level=l, nsweeps=1)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(reps):
            ctx.smooth(bl, xl, level=l, nsweeps=1)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        level_sweep_ms.append(e0.elapsed_time(e1) / reps)
    # coarse solve (K8) alone
    n0 = infos[0]["n"]
    bc = torch.from_numpy(np.random.default_rng(seed).uniform(-1, 1, n0)).to(dev)
    xc = torch.empty_like(bc)
    ctx.coarse_solve(bc, xc)
    torch.cuda.synchronize(dev)
    e0.record(stream)
    for _ in range(reps):
        ctx.coarse_solve(bc, xc)
    e1.record(stream)
    torch.cuda.synchronize(dev)
    ms_k8 = e0.elapsed_time(e1) / reps

    # ---- Krylov solves: GMRES(V-cycle) with the Richardson smoother (iteration counts of the
    # north star), and NEXT-1: the paper's GMRES(6)-smoothed V-cycle inside flexible GMRES
    # (rtol = atol = 1e-7) ----
    solves = None
    if not args.no_solves and ws == 1:          # single-GPU line only (not the scaling runs)
        xk = torch.empty_like(bd)
        e0.record(stream)
        its_r, rel_r, conv_r = ctx.gmres(bd, xk, maxit=600)   # basis of 2 x 601 x 31.5 MB
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_gr = e0.elapsed_time(e1)
        ctx.set_smoother("gmres", 6)
        ctx.vcycle(bd, xk)
        torch.cuda.synchronize(dev)
        e0.record(stream)
        for _ in range(3):
            ctx.vcycle(bd, xk)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_vg = e0.elapsed_time(e1) / 3
        e0.record(stream)
        its_f, rel_f, conv_f = ctx.fgmres(bd, xk, maxit=60)
        e1.record(stream)
        torch.cuda.synchronize(dev)
        ms_f = e0.elapsed_time(e1)
        ctx.set_smoother("richardson", 6)
        solves = {"gmres_richardson_vcycle": {"its": its_r, "converged": conv_r, "relres": rel_r, "ms": ms_gr},
                  "next1_gmres6_smoothed_vcycle_ms": ms_vg,
                  "next1_fgmres": {"its": its_f, "converged": conv_f, "relres": rel_f, "ms": ms_f},
                  "tolerance": "max(1e-7 |b|, 1e-7), Euclidean (P:654)"}

    # ---- NEXT-4 / NEXT-3 measured on the same kernels (skipped with --no-variants) ----
    variants = None
    configs = None
    if not args.no_variants and ws == 1:
        variants = run_variants(cfg, seed, dev, stream)
        configs = run_configs(seed, dev, stream)

    # algorithmic bytes: K2 per patch i: 8 n_i^2 factor + 8 n_i gathered r
    # + 8 n_i written y; sweep: 8 sum n_i^2 + 8 nnz + 24 n
    k2_bytes = 8 * fin["sum_n2"] + 16 * fin["sum_n"]
    sweep_bytes = 8 * fin["sum_n2"] + 8 * fin["nnz"] + 24 * fin["n"]
    k1_bytes = 8 * fin["nnz"] + 24 * fin["n"]
    pk = peaks()
    peak = pk["hbm_gbs"] if pk else 6650.0
    k2_gbs = k2_bytes / (ms_k2 * 1e-3) / 1e9
    tr = k2_traffic()

    # ---- e2e: host buffers through the C-ABI, pinned memory.  Every step uploads its own
    # right-hand side and downloads its x.  Serial: mhdp_vcycle_host per step.  Batched
    # (the headline): mhdp_vcycle_host_batch over the K steps, whose copies overlap the
    # neighbouring V-cycles ----
    bh = torch.from_numpy(b).pin_memory()
    xh = torch.empty(n, dtype=torch.float64).pin_memory()
    bnp, xnp = bh.numpy(), xh.numpy()
    ctx.vcycle_host(bnp, xnp)
    barrier()
    te = time.perf_counter()
    for _ in range(args.steps):
        ctx.vcycle_host(bnp, xnp)
    e2e_serial_ms = max_over_ranks((time.perf_counter() - te) * 1e3 / args.steps, dev)
    Bh = torch.empty((args.steps, n), dtype=torch.float64).pin_memory()
    Xh = torch.empty((args.steps, n), dtype=torch.float64).pin_memory()
    for k in range(args.steps):
        Bh[k] = torch.from_numpy(b) * (1.0 + k / 64.0)       # K distinct right-hand sides
    Bnp, Xnp = Bh.numpy(), Xh.numpy()
    ctx.vcycle_host_batch(Bnp[:2], Xnp[:2])                    # warm: both slots' graphs
    ctx.vcycle_host_batch(Bnp[:2], Xnp[:2])
    barrier()
    te = time.perf_counter()
    ctx.vcycle_host_batch(Bnp, Xnp)
    e2e_ms = max_over_ranks((time.perf_counter() - te) * 1e3 / args.steps, dev)

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        r = oracle_vcycle_sample(steps=2, warmup=1)
        cpu = {"value": r["value"], "unit": "DoF/s", "cores": 1, "kind": "oracle", "sample": r["sample"],
               "oracle_setup_s_of_sample": r["setup_s"], "host": host_info(),
               "full_size_record": oracle_full_size_record()}

    if rank == 0:
        value = ws * smoothed / (ms * 1e-3)
        line = {
            "metric": METRIC,
            "value": value, "unit": "DoF/s", "n_gpus": ws, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, L, fin, ws),
            "vcycle_ms": ms,
            "value_all_levels": ws * smoothed_all / (ms * 1e-3),
            "value_definition": "A26: (nu_pre + nu_post) x finest-level free DoFs per V-cycle; "
                                "value_all_levels: every level's sweeps",
            "sweep": {"ms": ms_sweep, "dofs_per_s": fin["n"] / (ms_sweep * 1e-3),
                      "gbs": sweep_bytes / (ms_sweep * 1e-3) / 1e9,
                      "frac": sweep_bytes / (ms_sweep * 1e-3) / 1e9 / peak, "bytes": sweep_bytes},
            "kernels": {"K2_patch_apply_ms": ms_k2, "K1_residual_ms": ms_k1,
                        "K1_gbs": k1_bytes / (ms_k1 * 1e-3) / 1e9, "K8_coarse_solve_ms": ms_k8,
                        "coarse_n": n0, "sweep_ms_per_level": level_sweep_ms},
            "roofline": {"bound": "hbm", "kernel": "K2 patch gather + LU apply (finest level)",
                         "achieved": k2_gbs, "peak": peak, "unit": "GB/s", "frac": k2_gbs / peak,
                         "traffic": (tr["traffic_bytes_per_launch"] if tr else None),
                         "traffic_source": (tr["source"] if tr else None),
                         "algorithmic_bytes": k2_bytes,
                         "peak_source": "MEASURED_PEAKS.json hbm_gbs" if pk else "fallback"},
            "e2e": {"value": ws * smoothed / (e2e_ms * 1e-3), "unit": "DoF/s", "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                    "api": "mhdp_vcycle_host_batch (K right-hand sides, copies overlapped)",
                    "serial_ms_per_step": e2e_serial_ms,
                    "serial_value": ws * smoothed / (e2e_serial_ms * 1e-3)},
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "setup_s": {"host_assembly": t_asm, "device_setup": t_setup},
            "setup_kernels": setup_kernels,
            "cpu_baseline": cpu,
            "solves": solves,
            "variants": variants,
            "other_configs": configs,
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c5")
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solves", action="store_true", help="skip the GMRES / FGMRES solves")
    ap.add_argument("--no-variants", action="store_true", help="skip the NEXT-4 / NEXT-3 measurements")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
