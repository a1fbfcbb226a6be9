"""Thin ctypes binding of libmhdp.so (include/mhdp.h) -- argument marshalling only.

Every step of the hot path runs in the library's CUDA kernels; this module converts
Python/numpy/torch arguments into plain pointers and sizes and raises on a non-zero
status.  There is no fallback: if libmhdp.so is missing or fails to load, importing
a Context raises.  Device vectors may be passed as torch CUDA tensors (fp64,
contiguous) or raw integer device pointers.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .build_lib import LIB

STATUS = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ESINGULAR", 5: "ESTATE", 6: "ENOCONV"}
BLOCK = {"eb": 0, "vel": 1}


class MhdpError(RuntimeError):
    def __init__(self, status, msg, where):
        super().__init__(f"mhdp {STATUS.get(status, status)}: {msg} (where={where})")
        self.status, self.msg, self.where = status, msg, where


class Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("n_fine", C.c_int), ("n_levels", C.c_int)]


class Params(C.Structure):
    _fields_ = [("Re", C.c_double), ("Rem", C.c_double), ("S", C.c_double), ("gamma", C.c_double),
                ("sigma", C.c_double), ("mu_stab", C.c_double), ("theta", C.c_double),
                ("nu_pre", C.c_int), ("nu_post", C.c_int), ("smoother", C.c_int), ("smoother_its", C.c_int),
                ("dt", C.c_double), ("picard", C.c_int), ("degree", C.c_int),
                ("weights_mode", C.c_int), ("newton_reaction", C.c_int)]


class LevelInfo(C.Structure):
    _fields_ = [(k, C.c_longlong) for k in ("n", "nnz", "npatch", "sum_n", "sum_n2", "max_n", "p_nnz",
                                            "bytes_operator", "bytes_factors", "bytes_transfer")]


_lib = None

# every symbol declared in include/mhdp.h
SYMBOLS = ["mhdp_create", "mhdp_destroy", "mhdp_assemble", "mhdp_begin_levels", "mhdp_load_level", "mhdp_setup",
           "mhdp_get_level_info", "mhdp_num_levels", "mhdp_spmv", "mhdp_residual", "mhdp_patch_apply",
           "mhdp_patch_update", "mhdp_smooth", "mhdp_restrict", "mhdp_prolong_add", "mhdp_coarse_solve",
           "mhdp_vcycle", "mhdp_vcycle_host", "mhdp_vcycle_host_batch", "mhdp_smooth_host", "mhdp_gmres", "mhdp_export_csr",
           "mhdp_export_patches", "mhdp_export_patch_vertices", "mhdp_export_prolongation", "mhdp_export_patch_lu", "mhdp_export_slots",
           "mhdp_synchronize", "mhdp_last_error", "mhdp_launch_count", "mhdp_fgmres", "mhdp_dot", "mhdp_set_smoother", "mhdp_vcycle_graphs_active", "mhdp_assemble_lorentz",
           "mhdp_coupled_create", "mhdp_coupled_destroy", "mhdp_coupled_sizes", "mhdp_coupled_export_csr",
           "mhdp_coupled_apply", "mhdp_coupled_precondition", "mhdp_coupled_fgmres", "mhdp_coupled_set_smoother",
           "mhdp_coupled_last_error", "mhdp_coarse_solve_trace", "mhdp_setup_timings", "mhdp_set_graphs"]


def lib():
    """Load libmhdp.so (raises OSError if it was not built: no fallback path exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise OSError(f"{LIB} not built: run paper_2104_14855_b200.build_lib.build()")
        L = C.CDLL(LIB)
        vp, i64, i64p, ip, dp = C.c_void_p, C.c_longlong, C.POINTER(C.c_longlong), C.POINTER(C.c_int), C.POINTER(C.c_double)
        sig = {
            "mhdp_create": [C.POINTER(vp), C.c_int, vp],
            "mhdp_assemble": [vp, C.c_int, C.POINTER(Mesh), C.POINTER(Params), dp],
            "mhdp_assemble_lorentz": [vp, C.c_int, C.POINTER(Mesh), C.POINTER(Params), dp, C.c_void_p],
            "mhdp_begin_levels": [vp, C.c_int, C.POINTER(Params)],
            "mhdp_load_level": [vp, C.c_int, i64, i64p, ip, dp, i64, i64p, ip, i64p, ip, dp],
            "mhdp_setup": [vp],
            "mhdp_get_level_info": [vp, C.c_int, C.POINTER(LevelInfo)],
            "mhdp_spmv": [vp, C.c_int, vp, vp],
            "mhdp_residual": [vp, C.c_int, vp, vp, vp],
            "mhdp_patch_apply": [vp, C.c_int, vp],
            "mhdp_patch_update": [vp, C.c_int, vp],
            "mhdp_smooth": [vp, C.c_int, C.c_int, C.c_int, vp, vp],
            "mhdp_restrict": [vp, C.c_int, vp, vp],
            "mhdp_prolong_add": [vp, C.c_int, vp, vp],
            "mhdp_coarse_solve": [vp, vp, vp],
            "mhdp_vcycle": [vp, C.c_int, vp, vp],
            "mhdp_vcycle_host": [vp, dp, dp],
            "mhdp_vcycle_host_batch": [vp, C.c_int, dp, dp],
            "mhdp_smooth_host": [vp, C.c_int, C.c_int, C.c_int, dp, dp],
            "mhdp_gmres": [vp, vp, vp, C.c_double, C.c_double, C.c_int, ip, dp, dp],
            "mhdp_coarse_solve_trace": [vp, vp, vp, C.POINTER(C.c_longlong)],
            "mhdp_setup_timings": [vp, dp, C.c_int],
            "mhdp_set_graphs": [vp, C.c_int],
            "mhdp_fgmres": [vp, vp, vp, C.c_double, C.c_double, C.c_int, ip, dp, dp],
            "mhdp_dot": [vp, vp, vp, i64, dp],
            "mhdp_set_smoother": [vp, C.c_int, C.c_int],
            "mhdp_coupled_create": [C.POINTER(vp), C.c_int, vp, C.POINTER(Mesh), C.POINTER(Params), dp, C.c_void_p],
            "mhdp_coupled_sizes": [vp, i64p],
            "mhdp_coupled_export_csr": [vp, i64p, ip, dp],
            "mhdp_coupled_apply": [vp, vp, vp],
            "mhdp_coupled_precondition": [vp, vp, vp],
            "mhdp_coupled_fgmres": [vp, vp, vp, C.c_double, C.c_double, C.c_int, ip, dp],
            "mhdp_coupled_set_smoother": [vp, C.c_int, C.c_int],
            "mhdp_coupled_last_error": [vp, C.c_char_p, C.c_int],
            "mhdp_export_csr": [vp, C.c_int, i64p, ip, dp],
            "mhdp_export_patches": [vp, C.c_int, i64p, ip],
            "mhdp_export_patch_vertices": [vp, C.c_int, ip],
            "mhdp_export_prolongation": [vp, C.c_int, i64p, ip, dp],
            "mhdp_export_patch_lu": [vp, C.c_int, i64, dp, ip],
            "mhdp_export_slots": [vp, C.c_int, dp],
            "mhdp_synchronize": [vp],
            "mhdp_last_error": [vp, C.c_char_p, C.c_int, i64p],
        }
        for name, args in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.mhdp_destroy.argtypes = [vp]
        L.mhdp_destroy.restype = None
        L.mhdp_num_levels.argtypes = [vp]
        L.mhdp_num_levels.restype = C.c_int
        L.mhdp_coupled_destroy.argtypes = [vp]
        L.mhdp_coupled_destroy.restype = None
        L.mhdp_vcycle_graphs_active.argtypes = [vp]
        L.mhdp_vcycle_graphs_active.restype = C.c_int
        L.mhdp_launch_count.argtypes = [vp]
        L.mhdp_launch_count.restype = C.c_longlong
        _lib = L
    return _lib


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _l(a):
    return a.ctypes.data_as(C.POINTER(C.c_longlong))


def _host_vec(a, shape, name):
    """Host buffer handed to C: must be a C-contiguous float64 numpy array of `shape`
    (the C side reads/writes exactly that many doubles).  Raises ValueError otherwise."""
    if not isinstance(a, np.ndarray):
        raise ValueError(f"{name}: expected a numpy array, got {type(a).__name__}")
    if a.dtype != np.float64:
        raise ValueError(f"{name}: dtype must be float64, got {a.dtype}")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name}: array must be C-contiguous")
    if a.shape != tuple(shape):
        raise ValueError(f"{name}: shape {a.shape}, expected {tuple(shape)}")
    return _d(a)


def _ptr(t):
    """Device pointer of a torch CUDA tensor (fp64, contiguous) or an int."""
    if isinstance(t, int):
        return t
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise TypeError("device vectors must be contiguous float64 CUDA tensors")
    return t.data_ptr()


def make_params(cfg, smoother: str = "richardson", smoother_its: int = 6) -> Params:
    """smoother 'richardson': nu Schwarz sweeps (north star); 'gmres': GMRES(smoother_its)
    preconditioned by the Schwarz operator, the paper's relaxation."""
    return Params(cfg.Re, cfg.Rem, cfg.S, cfg.gamma, cfg.sigma, cfg.mu, cfg.theta, cfg.nu, cfg.nu,
                  1 if smoother == "gmres" else 0, smoother_its, float(getattr(cfg, "dt", 0.0)),
                  int(getattr(cfg, "picard", 0)), int(getattr(cfg, "degree", 1)),
                  int(getattr(cfg, "weights_mode", 0)), int(getattr(cfg, "newton_reaction", 0)))


class Context:
    """One mhdp_ctx.  device=-1: host-only (assembly / export only)."""

    def __init__(self, device: int = 0, stream: int | None = None):
        self._L = lib()
        h = C.c_void_p()
        st = self._L.mhdp_create(C.byref(h), device, C.c_void_p(stream or 0))
        if st:
            raise MhdpError(st, "mhdp_create failed", -1)
        self.h = h
        self.device = device

    def close(self):
        if getattr(self, "h", None):
            self._L.mhdp_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def _chk(self, st):
        if st:
            buf = C.create_string_buffer(512)
            where = C.c_longlong(-1)
            self._L.mhdp_last_error(self.h, buf, 512, C.byref(where))
            raise MhdpError(st, buf.value.decode(), where.value)
        return st

    # ---- setup ----
    def assemble(self, cfg, w, N=None, levels=None, smoother="richardson", smoother_its=6, bn=None):
        """bn: potential of B^n for the Lorentz term of the velocity block (NEXT-4), or None."""
        mesh = Mesh(cfg.dim, N if N is not None else cfg.N, levels if levels is not None else cfg.levels)
        self._w = np.ascontiguousarray(w, np.float64)
        self._bn = None if bn is None else np.ascontiguousarray(bn, np.float64)
        p = make_params(cfg, smoother, smoother_its)
        return self._chk(self._L.mhdp_assemble_lorentz(self.h, BLOCK[cfg.block], C.byref(mesh), C.byref(p),
                                                       _d(self._w),
                                                       None if self._bn is None else self._bn.ctypes.data))

    def begin_levels(self, n_levels, cfg, smoother="richardson", smoother_its=6):
        p = make_params(cfg, smoother, smoother_its)
        return self._chk(self._L.mhdp_begin_levels(self.h, n_levels, C.byref(p)))

    def load_level(self, level, rowptr, col, val, pptr=None, pdofs=None, prow=None, pcol=None, pval=None):
        rowptr = np.ascontiguousarray(rowptr, np.int64); col = np.ascontiguousarray(col, np.int32)
        val = np.ascontiguousarray(val, np.float64)
        n = len(rowptr) - 1
        if pptr is None:
            return self._chk(self._L.mhdp_load_level(self.h, level, n, _l(rowptr), _i(col), _d(val), 0,
                                                     None, None, None, None, None))
        pptr = np.ascontiguousarray(pptr, np.int64); pdofs = np.ascontiguousarray(pdofs, np.int32)
        prow = np.ascontiguousarray(prow, np.int64); pcol = np.ascontiguousarray(pcol, np.int32)
        pval = np.ascontiguousarray(pval, np.float64)
        return self._chk(self._L.mhdp_load_level(self.h, level, n, _l(rowptr), _i(col), _d(val), len(pptr) - 1,
                                                 _l(pptr), _i(pdofs), _l(prow), _i(pcol), _d(pval)))

    def setup(self):
        return self._chk(self._L.mhdp_setup(self.h))

    def setup_timings(self):
        """{'K7_ms', 'K8_pack_ms', 'wall_s', 'K6_ms': [per level]} of the last setup"""
        L = self.num_levels()
        out = np.zeros(9 + L)
        self._chk(self._L.mhdp_setup_timings(self.h, _d(out), len(out)))
        st = out[3 + L:]
        return {"K7_ms": out[0], "K8_pack_ms": out[1], "wall_s": out[2], "K6_ms": out[3:3 + L].tolist(),
                "host_stage_s": dict(zip(["operator", "patches", "transfers", "K6", "lane_groups", "coarse"],
                                         st.tolist()))}

    def num_levels(self):
        return self._L.mhdp_num_levels(self.h)

    def info(self, level=-1):
        level = level % self.num_levels()
        out = LevelInfo()
        self._chk(self._L.mhdp_get_level_info(self.h, level, C.byref(out)))
        return {k: getattr(out, k) for k, _ in LevelInfo._fields_}

    def n(self, level=-1):
        return self.info(level)["n"]

    # ---- hot path (device) ----
    def spmv(self, x, y, level=-1):
        return self._chk(self._L.mhdp_spmv(self.h, level % self.num_levels(), _ptr(x), _ptr(y)))

    def residual(self, b, x, r, level=-1):
        return self._chk(self._L.mhdp_residual(self.h, level % self.num_levels(), _ptr(b), _ptr(x), _ptr(r)))

    def patch_apply(self, r, level=-1):
        return self._chk(self._L.mhdp_patch_apply(self.h, level % self.num_levels(), _ptr(r)))

    def patch_update(self, x, level=-1):
        return self._chk(self._L.mhdp_patch_update(self.h, level % self.num_levels(), _ptr(x)))

    def smooth(self, b, x, level=-1, nsweeps=1, x_is_zero=False):
        return self._chk(self._L.mhdp_smooth(self.h, level % self.num_levels(), nsweeps, int(x_is_zero),
                                             _ptr(b), _ptr(x)))

    def restrict(self, r, rc, level=-1):
        return self._chk(self._L.mhdp_restrict(self.h, level % self.num_levels(), _ptr(r), _ptr(rc)))

    def prolong_add(self, ec, x, level=-1):
        return self._chk(self._L.mhdp_prolong_add(self.h, level % self.num_levels(), _ptr(ec), _ptr(x)))

    def coarse_solve_trace(self, b, x):
        """one coarse solve with K8's per-block timestamps: array (2, nb, 5) of ns"""
        nb = (self.n(0) + 31) // 32
        tr = np.zeros(32 * nb, np.int64)
        self._chk(self._L.mhdp_coarse_solve_trace(self.h, _ptr(b), _ptr(x), tr.ctypes.data_as(C.POINTER(C.c_longlong))))
        return tr.reshape(2, nb, 16)

    def coarse_solve(self, b, x):
        return self._chk(self._L.mhdp_coarse_solve(self.h, _ptr(b), _ptr(x)))

    def vcycle(self, b, x, level=-1):
        return self._chk(self._L.mhdp_vcycle(self.h, level % self.num_levels(), _ptr(b), _ptr(x)))

    def vcycle_host_batch(self, b, x):
        """b, x: C-contiguous float64 host arrays of shape (nrhs, n) (pinned for overlap)"""
        if not isinstance(b, np.ndarray) or b.ndim != 2:
            raise ValueError("b: expected a 2-D numpy array (nrhs, n)")
        shape = (b.shape[0], self.n())
        return self._chk(self._L.mhdp_vcycle_host_batch(self.h, b.shape[0], _host_vec(b, shape, "b"),
                                                        _host_vec(x, shape, "x")))

    def vcycle_host(self, b, x):
        """b, x: C-contiguous float64 numpy arrays of length n (pinned or pageable)."""
        shape = (self.n(),)
        return self._chk(self._L.mhdp_vcycle_host(self.h, _host_vec(b, shape, "b"), _host_vec(x, shape, "x")))

    def smooth_host(self, b, x, level=-1, nsweeps=1, x_is_zero=False):
        level = level % self.num_levels()
        shape = (self.n(level),)
        return self._chk(self._L.mhdp_smooth_host(self.h, level, nsweeps, int(x_is_zero),
                                                  _host_vec(b, shape, "b"), _host_vec(x, shape, "x")))

    def _krylov(self, fn, b, x, rtol, atol, maxit):
        its = C.c_int(0)
        rel = C.c_double(0)
        hist = np.zeros(maxit + 1)
        st = fn(self.h, _ptr(b), _ptr(x), rtol, atol, maxit, C.byref(its), C.byref(rel),
                hist.ctypes.data_as(C.POINTER(C.c_double)))
        if st not in (0, 6):
            self._chk(st)
        self.last_history = hist[: its.value + 1].copy()   # |g_k|, k = 0..its
        return its.value, rel.value, st == 0

    def gmres(self, b, x, rtol=1e-7, atol=1e-7, maxit=200):
        """GMRES(V) (c.9); the residual history is left in self.last_history."""
        return self._krylov(self._L.mhdp_gmres, b, x, rtol, atol, maxit)

    def set_smoother(self, smoother="richardson", its=6):
        return self._chk(self._L.mhdp_set_smoother(self.h, 1 if smoother == "gmres" else 0, its))

    def fgmres(self, b, x, rtol=1e-7, atol=1e-7, maxit=100):
        return self._krylov(self._L.mhdp_fgmres, b, x, rtol, atol, maxit)

    def dot(self, a, b):
        out = C.c_double(0)
        self._chk(self._L.mhdp_dot(self.h, _ptr(a), _ptr(b), a.numel(), C.byref(out)))
        return out.value

    def synchronize(self):
        return self._chk(self._L.mhdp_synchronize(self.h))

    def set_graphs(self, enable=True):
        return self._chk(self._L.mhdp_set_graphs(self.h, int(bool(enable))))

    def graphs_active(self):
        return self._L.mhdp_vcycle_graphs_active(self.h)

    def launch_count(self):
        return self._L.mhdp_launch_count(self.h)

    # ---- export ----
    def csr(self, level=-1):
        level = level % self.num_levels()
        i = self.info(level)
        rp = np.zeros(i["n"] + 1, np.int64); ci = np.zeros(max(i["nnz"], 1), np.int32)
        v = np.zeros(max(i["nnz"], 1), np.float64)
        self._chk(self._L.mhdp_export_csr(self.h, level, _l(rp), _i(ci), _d(v)))
        return rp, ci[:i["nnz"]], v[:i["nnz"]]

    def patch_vertices(self, level=-1):
        level = level % self.num_levels()
        v = np.zeros(max(self.info(level)["npatch"], 1), np.int32)
        self._chk(self._L.mhdp_export_patch_vertices(self.h, level, _i(v)))
        return v[: self.info(level)["npatch"]]

    def patches(self, level=-1):
        level = level % self.num_levels()
        i = self.info(level)
        ptr = np.zeros(i["npatch"] + 1, np.int64); dofs = np.zeros(max(i["sum_n"], 1), np.int32)
        self._chk(self._L.mhdp_export_patches(self.h, level, _l(ptr), _i(dofs)))
        return ptr, dofs[:i["sum_n"]]

    def prolongation(self, level=-1):
        level = level % self.num_levels()
        i = self.info(level)
        rp = np.zeros(i["n"] + 1, np.int64); ci = np.zeros(max(i["p_nnz"], 1), np.int32)
        v = np.zeros(max(i["p_nnz"], 1), np.float64)
        self._chk(self._L.mhdp_export_prolongation(self.h, level, _l(rp), _i(ci), _d(v)))
        return rp, ci[:i["p_nnz"]], v[:i["p_nnz"]]

    def patch_lu(self, patch, level=-1):
        level = level % self.num_levels()
        ptr, _ = self.patches(level)
        k = int(ptr[patch + 1] - ptr[patch])
        lu = np.zeros(k * k); perm = np.zeros(k, np.int32)
        self._chk(self._L.mhdp_export_patch_lu(self.h, level, patch, _d(lu), _i(perm)))
        return lu.reshape(k, k), perm

    def slots(self, level=-1):
        level = level % self.num_levels()
        y = np.zeros(max(self.info(level)["sum_n"], 1))
        self._chk(self._L.mhdp_export_slots(self.h, level, _d(y)))
        return y


class Coupled:
    """NEXT-3: the coupled Newton system over [u | p | E | B] and the paper's outer solver
    (include/mhdp.h mhdp_coupled_*).  device=-1: host-only (assembly and export)."""

    def __init__(self, cfg, w, bn=None, device: int = 0, stream: int | None = None, smoother="richardson",
                 smoother_its=6):
        self._L = lib()
        self._w = np.ascontiguousarray(w, np.float64)
        self._bn = None if bn is None else np.ascontiguousarray(bn, np.float64)
        mesh = Mesh(cfg.dim, cfg.N, cfg.levels)
        p = make_params(cfg, smoother, smoother_its)
        h = C.c_void_p()
        st = self._L.mhdp_coupled_create(C.byref(h), device, C.c_void_p(stream or 0), C.byref(mesh), C.byref(p),
                                         _d(self._w), None if self._bn is None else self._bn.ctypes.data)
        self.h = h
        self._chk(st)
        s = np.zeros(5, np.int64)
        self._chk(self._L.mhdp_coupled_sizes(self.h, _l(s)))
        self.nu, self.np_, self.nE, self.nB, self.nnz = (int(v) for v in s)
        self.n = self.nu + self.np_ + self.nE + self.nB

    def _chk(self, st):
        if st:
            buf = C.create_string_buffer(512)
            if getattr(self, "h", None):
                self._L.mhdp_coupled_last_error(self.h, buf, 512)
            raise MhdpError(st, buf.value.decode(), -1)
        return st

    def close(self):
        if getattr(self, "h", None):
            self._L.mhdp_coupled_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def csr(self):
        rp = np.zeros(self.n + 1, np.int64); ci = np.zeros(max(self.nnz, 1), np.int32); v = np.zeros(max(self.nnz, 1))
        self._chk(self._L.mhdp_coupled_export_csr(self.h, _l(rp), _i(ci), _d(v)))
        return rp, ci[:self.nnz], v[:self.nnz]

    def apply(self, x, y):
        return self._chk(self._L.mhdp_coupled_apply(self.h, _ptr(x), _ptr(y)))

    def precondition(self, r, y):
        return self._chk(self._L.mhdp_coupled_precondition(self.h, _ptr(r), _ptr(y)))

    def fgmres(self, b, x, rtol=1e-7, atol=1e-7, maxit=50):
        its = C.c_int(0)
        rel = C.c_double(0)
        st = self._L.mhdp_coupled_fgmres(self.h, _ptr(b), _ptr(x), rtol, atol, maxit, C.byref(its), C.byref(rel))
        if st not in (0, 6):
            self._chk(st)
        return its.value, rel.value, st == 0

    def set_smoother(self, smoother="richardson", its=6):
        return self._chk(self._L.mhdp_coupled_set_smoother(self.h, 1 if smoother == "gmres" else 0, its))
