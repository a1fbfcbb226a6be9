"""ctypes wrapper of the C ORACLE (liboracle.so).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.  The product package
(paper_2104_14855_b200) never imports this module and this module never imports
the product's native library.  See orc.h for what the oracle computes and the
PAPER.md passages it follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "liboracle.so")
LIB_EXACT = os.path.join(HERE, "liboracle_exact.so")
SOURCES = ["mesh.c", "space.c", "fem.c", "solve.c", "api.c"]


def build(force: bool = False) -> str:
    """Compile the oracle (plain C, single-threaded, -ffp-contract=off: every fused
    multiply-add is an explicit fma() call of the pinned rounding order) twice:
    liboracle.so with real = double and liboracle_exact.so with real = __float128 for the
    element integrals (reading R-exact, see fem.c)."""
    srcs = [os.path.join(HERE, s) for s in SOURCES] + [os.path.join(HERE, "orc.h")]
    newest = max(os.path.getmtime(s) for s in srcs)
    for lib, extra in ((LIB, []), (LIB_EXACT, ["-DORC_EXACT"])):
        if not force and os.path.exists(lib) and os.path.getmtime(lib) >= newest:
            continue
        cmd = ["gcc", "-O2", "-std=gnu11", "-ffp-contract=off", "-mfma", "-fPIC", "-shared", *extra, "-o", lib + ".tmp"]
        cmd += [os.path.join(HERE, s) for s in SOURCES] + ["-lquadmath", "-lm"]
        subprocess.check_call(cmd)
        os.replace(lib + ".tmp", lib)
    return LIB


_libs = {}


def lib(exact: bool = False):
    if exact not in _libs:
        build()
        L = C.CDLL(LIB_EXACT if exact else LIB)
        vp, i64p, ip, dp = C.c_void_p, C.POINTER(C.c_longlong), C.POINTER(C.c_int), C.POINTER(C.c_double)
        L.orc_create.restype = vp
        L.orc_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, ip, dp]
        L.orc_create_masked.restype = vp
        L.orc_create_masked.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, dp, ip, dp, C.c_void_p, C.c_void_p]
        L.orc_destroy.argtypes = [vp]
        L.orc_level_info.argtypes = [vp, C.c_int, i64p]
        L.orc_export_csr.argtypes = [vp, C.c_int, i64p, ip, dp]
        L.orc_export_prolongation.argtypes = [vp, C.c_int, i64p, ip, dp]
        L.orc_export_patches.argtypes = [vp, C.c_int, i64p, ip, ip, ip]
        L.orc_export_mesh.argtypes = [vp, C.c_int, dp, ip, ip, ip, ip, ip, ip, ip]
        L.orc_spmv.argtypes = [vp, C.c_int, dp, dp]
        L.orc_residual.argtypes = [vp, C.c_int, dp, dp, dp]
        L.orc_patch_matrix.argtypes = [vp, C.c_int, C.c_longlong, dp]
        L.orc_patch_lu.argtypes = [vp, C.c_int, C.c_longlong, dp, ip]
        L.orc_sweep.restype = C.c_longlong
        L.orc_sweep.argtypes = [vp, C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_sweep_sample.restype = C.c_longlong
        L.orc_sweep_sample.argtypes = [vp, C.c_int, C.c_int, dp, dp, C.c_longlong, ip, dp]
        L.orc_restrict.argtypes = [vp, C.c_int, dp, dp]
        L.orc_prolong_add.argtypes = [vp, C.c_int, dp, dp]
        L.orc_coarse_solve.argtypes = [vp, dp, dp]
        L.orc_coarse_lu.argtypes = [vp, dp, ip]
        L.orc_vcycle.argtypes = [vp, dp, dp]
        L.orc_vcycle_level.argtypes = [vp, C.c_int, dp, dp]
        L.orc_gmres.argtypes = [vp, dp, dp, C.c_double, C.c_double, C.c_int, ip, dp]
        L.orc_quad_info.argtypes = [vp, C.c_int, i64p]
        L.orc_quadrature.argtypes = [vp, C.c_int, dp, dp]
        L.orc_load.argtypes = [vp, C.c_int, dp, dp]
        L.orc_eval.argtypes = [vp, C.c_int, dp, dp]
        L.orc_duality_error.restype = C.c_double
        L.orc_duality_error.argtypes = [vp, C.c_int]
        L.orc_set_patches.argtypes = [vp, C.c_int, C.c_longlong, i64p, ip]
        L.orc_dense_lu_solve.argtypes = [C.c_int, dp, dp, dp, dp, ip]
        L.orc_set_smoother.argtypes = [vp, C.c_int, C.c_int]
        L.orc_set_smoother.restype = None
        L.orc_fgmres.argtypes = [vp, dp, dp, C.c_double, C.c_double, C.c_int, ip, dp]
        L.orc_gmres_smooth.argtypes = [vp, C.c_int, C.c_int, C.c_int, dp, dp]
        L.orc_coupled_create.restype = vp
        L.orc_coupled_create.argtypes = [C.c_int, C.c_int, C.c_int, dp, ip, dp, C.c_void_p]
        L.orc_coupled_destroy.argtypes = [vp]
        L.orc_coupled_destroy.restype = None
        L.orc_coupled_sizes.argtypes = [vp, i64p]
        L.orc_coupled_sizes.restype = None
        L.orc_coupled_export.argtypes = [vp, i64p, ip, dp]
        L.orc_coupled_apply.argtypes = [vp, dp, dp]
        L.orc_coupled_precondition.argtypes = [vp, dp, dp]
        L.orc_coupled_fgmres.argtypes = [vp, dp, dp, C.c_double, C.c_double, C.c_int, ip, dp]
        L.orc_coupled_set_smoother.argtypes = [vp, C.c_int, C.c_int]
        L.orc_coupled_set_smoother.restype = None
        L.orc_dot.argtypes = [dp, dp, C.c_longlong]
        L.orc_dot.restype = C.c_double
        _libs[exact] = L
    return _libs[exact]


def _d(a):
    return a.ctypes.data_as(C.POINTER(C.c_double))


def _i(a):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _l(a):
    return a.ctypes.data_as(C.POINTER(C.c_longlong))


def dot(a, b):
    """The pinned inner product of reading R-dot."""
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    return lib().orc_dot(_d(a), _d(b), len(a))


def dense_lu_solve(a, b):
    """(x, lu, perm, status) of the oracle's dense LU (R-lu) on a row-major matrix."""
    a = np.ascontiguousarray(a, np.float64); b = np.ascontiguousarray(b, np.float64)
    n = a.shape[0]
    x = np.zeros(n); lu = np.zeros((n, n)); perm = np.zeros(n, np.int32)
    st = lib().orc_dense_lu_solve(n, _d(a), _d(b), _d(x), _d(lu), _i(perm))
    return x, lu, perm, st


class Csr:
    def __init__(self, rp, ci, v):
        self.rp, self.ci, self.v = rp, ci, v
        self.n = len(rp) - 1

    def to_scipy(self, ncols=None):
        import scipy.sparse as sp
        return sp.csr_matrix((self.v, self.ci, self.rp), shape=(self.n, ncols if ncols is not None else self.n))


class Oracle:
    """Hierarchy for one configuration (see paper_2104_14855_b200.workloads.Config)."""

    def __init__(self, cfg, w, nlev=None, N=None, cmask=None, exact=False, bn=None):
        """exact=True: element integrals in __float128 (reading R-exact): every operator
        entry is the fp64 value nearest to the exact discrete bilinear form."""
        self._L = L = lib(exact)
        self.cfg = cfg
        self.dim = cfg.dim
        self.nlev = nlev if nlev is not None else cfg.levels
        N = N if N is not None else cfg.N
        self.N = N
        dp = np.array([cfg.Re, cfg.Rem, cfg.S, cfg.gamma, cfg.sigma, cfg.mu, cfg.theta,
                       getattr(cfg, "dt", 0.0)], dtype=np.float64)
        ip = np.array([cfg.nu, cfg.nu, int(getattr(cfg, "picard", 0)), int(getattr(cfg, "degree", 1)),
                       int(getattr(cfg, "weights_mode", 0)), int(getattr(cfg, "newton_reaction", 0))],
                      dtype=np.int32)
        self._w = np.ascontiguousarray(w, dtype=np.float64)
        self._bn = None if bn is None else np.ascontiguousarray(bn, dtype=np.float64)
        self._mask = None if cmask is None else np.ascontiguousarray(cmask, dtype=np.uint8)
        self.h = L.orc_create_masked(cfg.block_id, cfg.dim, N, self.nlev, _d(dp), _i(ip), _d(self._w),
                                     None if self._mask is None else self._mask.ctypes.data,
                                     None if self._bn is None else self._bn.ctypes.data)
        if not self.h:
            raise ValueError("oracle: invalid configuration")
        self._info = {}

    def __del__(self):
        if getattr(self, "h", None):
            self._L.orc_destroy(self.h)
            self.h = None

    def info(self, level=-1):
        level = level % self.nlev
        out = np.zeros(11, dtype=np.int64)
        self._L.orc_level_info(self.h, level, _l(out))
        keys = ["n", "nnz", "npatch", "sum_n", "sum_n2", "nE", "nv", "nc", "ne", "nf", "p_nnz"]
        return dict(zip(keys, (int(v) for v in out)))

    def n(self, level=-1):
        return self.info(level)["n"]

    def csr(self, level=-1):
        level = level % self.nlev
        i = self.info(level)
        rp = np.zeros(i["n"] + 1, np.int64)
        ci = np.zeros(i["nnz"], np.int32)
        v = np.zeros(i["nnz"], np.float64)
        self._L.orc_export_csr(self.h, level, _l(rp), _i(ci), _d(v))
        return Csr(rp, ci, v)

    def prolongation(self, level=-1):
        level = level % self.nlev
        i = self.info(level)
        rp = np.zeros(i["n"] + 1, np.int64)
        ci = np.zeros(i["p_nnz"], np.int32)
        v = np.zeros(i["p_nnz"], np.float64)
        self._L.orc_export_prolongation(self.h, level, _l(rp), _i(ci), _d(v))
        return Csr(rp, ci, v)

    def patches(self, level=-1):
        level = level % self.nlev
        i = self.info(level)
        ptr = np.zeros(i["npatch"] + 1, np.int64)
        dofs = np.zeros(i["sum_n"], np.int32)
        vert = np.zeros(i["npatch"], np.int32)
        mult = np.zeros(i["n"], np.int32)
        self._L.orc_export_patches(self.h, level, _l(ptr), _i(dofs), _i(vert), _i(mult))
        return ptr, dofs, vert, mult

    def mesh(self, level=-1):
        level = level % self.nlev
        i = self.info(level)
        d = self.dim
        nfacet = i["ne"] if d == 2 else i["nf"]
        x = np.zeros(3 * i["nv"]); cv = np.zeros((d + 1) * i["nc"], np.int32)
        ev = np.zeros(2 * i["ne"], np.int32); fv = np.zeros(max(3 * i["nf"], 1), np.int32)
        fc = np.zeros(2 * nfacet, np.int32)
        dk = np.zeros(i["n"], np.int32); de = np.zeros(i["n"], np.int32); ds = np.zeros(i["n"], np.int32)
        self._L.orc_export_mesh(self.h, level, _d(x), _i(cv), _i(ev), _i(fv), _i(fc), _i(dk), _i(de), _i(ds))
        return dict(x=x.reshape(-1, 3), cv=cv.reshape(-1, d + 1), ev=ev.reshape(-1, 2),
                    fv=fv[:3 * i["nf"]].reshape(-1, 3), fcell=fc.reshape(-1, 2), dkind=dk, dent=de, dsub=ds)

    def spmv(self, x, level=-1):
        level = level % self.nlev
        x = np.ascontiguousarray(x, np.float64)
        y = np.zeros(self.n(level))
        self._L.orc_spmv(self.h, level, _d(x), _d(y))
        return y

    def residual(self, b, x, level=-1):
        level = level % self.nlev
        b = np.ascontiguousarray(b, np.float64); x = np.ascontiguousarray(x, np.float64)
        r = np.zeros(self.n(level))
        self._L.orc_residual(self.h, level, _d(b), _d(x), _d(r))
        return r

    def patch_matrix(self, patch, level=-1):
        level = level % self.nlev
        ptr = self.patches(level)[0]
        k = int(ptr[patch + 1] - ptr[patch])
        a = np.zeros(k * k)
        self._L.orc_patch_matrix(self.h, level, patch, _d(a))
        return a.reshape(k, k)

    def patch_lu(self, patch, level=-1):
        level = level % self.nlev
        ptr = self.patches(level)[0]
        k = int(ptr[patch + 1] - ptr[patch])
        a = np.zeros(k * k); perm = np.zeros(k, np.int32)
        st = self._L.orc_patch_lu(self.h, level, patch, _d(a), _i(perm))
        return a.reshape(k, k), perm, st

    def sweep(self, b, x, level=-1, nsweeps=1, x_is_zero=False):
        level = level % self.nlev
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, dtype=np.float64, copy=True) if x is not None else np.zeros(self.n(level))
        st = self._L.orc_sweep(self.h, level, nsweeps, int(x_is_zero), _d(b), _d(x))
        if st:
            raise ArithmeticError(f"oracle: singular patch {st - 1}")
        return x

    def sweep_sample(self, b, x, dofs, level=-1, x_is_zero=False):
        level = level % self.nlev
        b = np.ascontiguousarray(b, np.float64)
        x = np.ascontiguousarray(x if x is not None else np.zeros(self.n(level)), np.float64)
        dofs = np.ascontiguousarray(dofs, np.int32)
        out = np.zeros(len(dofs))
        st = self._L.orc_sweep_sample(self.h, level, int(x_is_zero), _d(b), _d(x), len(dofs), _i(dofs), _d(out))
        if st:
            raise ArithmeticError(f"oracle: singular patch {st - 1}")
        return out

    def restrict(self, r, level=-1):
        level = level % self.nlev
        r = np.ascontiguousarray(r, np.float64)
        rc = np.zeros(self.n(level - 1))
        self._L.orc_restrict(self.h, level, _d(r), _d(rc))
        return rc

    def prolong_add(self, ec, x, level=-1):
        level = level % self.nlev
        ec = np.ascontiguousarray(ec, np.float64)
        x = np.array(x, dtype=np.float64, copy=True)
        self._L.orc_prolong_add(self.h, level, _d(ec), _d(x))
        return x

    def coarse_solve(self, b):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n(0))
        if self._L.orc_coarse_solve(self.h, _d(b), _d(x)):
            raise ArithmeticError("oracle: singular coarse operator")
        return x

    def coarse_lu(self):
        n = self.n(0)
        a = np.zeros(n * n); p = np.zeros(n, np.int32)
        st = self._L.orc_coarse_lu(self.h, _d(a), _i(p))
        return a.reshape(n, n), p, st

    def vcycle(self, b, level=None):
        level = self.nlev - 1 if level is None else level % self.nlev
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n(level))
        if self._L.orc_vcycle_level(self.h, level, _d(b), _d(x)):
            raise ArithmeticError("oracle: V-cycle failed (singular patch or coarse operator)")
        return x

    def set_smoother(self, kind: str = "richardson", its: int = 6):
        """'richardson': nu sweeps (north star); 'gmres': GMRES(its) smoothing (NEXT-1)."""
        self._L.orc_set_smoother(self.h, 1 if kind == "gmres" else 0, its)

    def gmres_smooth(self, b, x, m=6, level=-1, x_is_zero=False):
        """One GMRES(m) smoothing step (R-gmres6) on a level; returns the new x."""
        level = level % self.nlev
        b = np.ascontiguousarray(b, np.float64)
        x = np.array(x, dtype=np.float64, copy=True)
        if self._L.orc_gmres_smooth(self.h, level, m, int(x_is_zero), _d(b), _d(x)):
            raise ArithmeticError("oracle: singular patch")
        return x

    def fgmres(self, b, rtol=1e-7, atol=1e-7, maxit=100):
        """Flexible GMRES with the V-cycle as variable preconditioner (R-fgmres)."""
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n())
        its = np.zeros(1, np.int32)
        hist = np.zeros(maxit + 1)
        st = self._L.orc_fgmres(self.h, _d(b), _d(x), rtol, atol, maxit, _i(its), _d(hist))
        if st == 2:
            raise ArithmeticError("oracle: FGMRES preconditioner failed")
        return x, int(its[0]), hist[: int(its[0]) + 1], st == 0

    def gmres(self, b, rtol=1e-7, atol=1e-7, maxit=200):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.n())
        its = np.zeros(1, np.int32)
        hist = np.zeros(maxit + 1)
        st = self._L.orc_gmres(self.h, _d(b), _d(x), rtol, atol, maxit, _i(its), _d(hist))
        if st == 2:
            raise ArithmeticError("oracle: GMRES preconditioner failed")
        return x, int(its[0]), hist[: int(its[0]) + 1], st == 0

    # ---- manufactured-solution helpers ----
    def quadrature(self, level=-1):
        level = level % self.nlev
        out = np.zeros(2, np.int64)
        self._L.orc_quad_info(self.h, level, _l(out))
        npts, ncomp = int(out[0]), int(out[1])
        pts = np.zeros(3 * npts); wts = np.zeros(npts)
        self._L.orc_quadrature(self.h, level, _d(pts), _d(wts))
        return pts.reshape(-1, 3), wts, ncomp

    def load(self, fvals, level=-1):
        level = level % self.nlev
        fvals = np.ascontiguousarray(fvals, np.float64)
        out = np.zeros(self.n(level))
        self._L.orc_load(self.h, level, _d(fvals), _d(out))
        return out

    def eval(self, coef, level=-1):
        level = level % self.nlev
        npts, ncomp = self.quadrature(level)[1].shape[0], self.quadrature(level)[2]
        coef = np.ascontiguousarray(coef, np.float64)
        fv = np.zeros(npts * ncomp)
        self._L.orc_eval(self.h, level, _d(coef), _d(fv))
        return fv.reshape(npts, ncomp)

    def duality_error(self, level=-1):
        return self._L.orc_duality_error(self.h, level % self.nlev)

    def set_patches(self, ptr, dofs, level=-1):
        """TEST HOOK: override the subspace decomposition of a level."""
        ptr = np.ascontiguousarray(ptr, np.int64); dofs = np.ascontiguousarray(dofs, np.int32)
        self._L.orc_set_patches(self.h, level % self.nlev, len(ptr) - 1, _l(ptr), _i(dofs))


class CoupledOracle:
    """NEXT-3: the 4x4 Newton system over [u | p | E | B] and the paper's outer
    solver: FGMRES with the block upper-triangular preconditioner.
    cfg gives dim, N, levels, Re, Rem, S, gamma, dt, picard; w: advecting potential (u^n);
    bn: B^n potential (or None: B^n = 0)."""

    def __init__(self, cfg, w, bn=None, exact=False, smoother="richardson", smoother_its=6):
        self._L = L = lib(exact)
        dp = np.array([cfg.Re, cfg.Rem, cfg.S, cfg.gamma, cfg.sigma, cfg.mu, cfg.theta,
                       getattr(cfg, "dt", 0.0)], dtype=np.float64)
        ip = np.array([cfg.nu, cfg.nu, int(getattr(cfg, "picard", 0)), int(getattr(cfg, "degree", 1)),
                       int(getattr(cfg, "weights_mode", 0)), int(getattr(cfg, "newton_reaction", 0))],
                      dtype=np.int32)
        self._w = np.ascontiguousarray(w, np.float64)
        self._bn = None if bn is None else np.ascontiguousarray(bn, np.float64)
        self.h = L.orc_coupled_create(cfg.dim, cfg.N, cfg.levels, _d(dp), _i(ip), _d(self._w),
                                      None if self._bn is None else self._bn.ctypes.data)
        if not self.h:
            raise ValueError("oracle: invalid coupled configuration")
        if smoother == "gmres":
            L.orc_coupled_set_smoother(self.h, 1, smoother_its)
        s = np.zeros(5, np.int64)
        L.orc_coupled_sizes(self.h, _l(s))
        self.nu, self.np_, self.nE, self.nB, self.nnz = (int(v) for v in s)
        self.n = self.nu + self.np_ + self.nE + self.nB

    def __del__(self):
        if getattr(self, "h", None):
            self._L.orc_coupled_destroy(self.h)
            self.h = None

    def csr(self):
        rp = np.zeros(self.n + 1, np.int64); ci = np.zeros(self.nnz, np.int32); v = np.zeros(self.nnz)
        self._L.orc_coupled_export(self.h, _l(rp), _i(ci), _d(v))
        return Csr(rp, ci, v)

    def apply(self, x):
        x = np.ascontiguousarray(x, np.float64); y = np.zeros(self.n)
        self._L.orc_coupled_apply(self.h, _d(x), _d(y))
        return y

    def precondition(self, r):
        r = np.ascontiguousarray(r, np.float64); y = np.zeros(self.n)
        if self._L.orc_coupled_precondition(self.h, _d(r), _d(y)):
            raise ArithmeticError("oracle: preconditioner failed")
        return y

    def fgmres(self, b, rtol=1e-7, atol=1e-7, maxit=50):
        b = np.ascontiguousarray(b, np.float64); x = np.zeros(self.n)
        its = np.zeros(1, np.int32); hist = np.zeros(maxit + 1)
        st = self._L.orc_coupled_fgmres(self.h, _d(b), _d(x), rtol, atol, maxit, _i(its), _d(hist))
        if st == 2:
            raise ArithmeticError("oracle: preconditioner failed")
        return x, int(its[0]), hist[: int(its[0]) + 1], st == 0
