"""Manufactured solutions for the oracle's finite-element pins (test helper).

Closed-form fields (SURVEY §8c.12 "FE correctness"), differentiated with sympy;
the discrete problems are solved with scipy's sparse direct solver on the
oracle's own CSR, and the L2 error is measured at the oracle's quadrature points.
"""
import numpy as np
import scipy.sparse.linalg as spla
import sympy as sp

X, Y, Z = sp.symbols("x y z")


def _lamb(expr, dim):
    f = sp.lambdify((X, Y, Z), expr, "numpy")
    return lambda P: np.broadcast_to(np.asarray(f(P[:, 0], P[:, 1], P[:, 2]), dtype=float), (P.shape[0],))


def eb_fields(dim, Rem, wconst, div_free_B=False, dt=0.0, picard=0):
    """dt > 0: transient B-equation source + B/dt; picard: no w x B term (NEXT-4)."""
    pi = sp.pi
    if dim == 2:
        E = sp.sin(pi * X) * sp.sin(pi * Y)
        if div_free_B:
            B = [sp.sin(pi * X) * sp.cos(pi * Y), -sp.cos(pi * X) * sp.sin(pi * Y)]
        else:
            B = [sp.sin(pi * X), sp.sin(pi * Y)]
        curlB = sp.diff(B[1], X) - sp.diff(B[0], Y)
        divB = sp.diff(B[0], X) + sp.diff(B[1], Y)
        wxB = 0 if picard else wconst[0] * B[1] - wconst[1] * B[0]
        fE = [E - curlB / Rem + wxB]
        vcurlE = [sp.diff(E, Y), -sp.diff(E, X)]
        fB = [vcurlE[k] - sp.diff(divB, v) / Rem + (B[k] / dt if dt > 0 else 0) for k, v in enumerate((X, Y))]
        exact = [E] + B
    else:
        E = [sp.sin(pi * Y) * sp.sin(pi * Z), sp.sin(pi * X) * sp.sin(pi * Z), sp.sin(pi * X) * sp.sin(pi * Y)]
        B = [sp.sin(pi * X), sp.sin(pi * Y), sp.sin(pi * Z)]

        def curl(F):
            return [sp.diff(F[2], Y) - sp.diff(F[1], Z), sp.diff(F[0], Z) - sp.diff(F[2], X),
                    sp.diff(F[1], X) - sp.diff(F[0], Y)]
        cB, cE = curl(B), curl(E)
        divB = sum(sp.diff(B[k], v) for k, v in enumerate((X, Y, Z)))
        w = wconst
        wxB = [w[1] * B[2] - w[2] * B[1], w[2] * B[0] - w[0] * B[2], w[0] * B[1] - w[1] * B[0]]
        if picard:
            wxB = [0, 0, 0]
        fE = [E[k] - cB[k] / Rem + wxB[k] for k in range(3)]
        fB = [cE[k] - sp.diff(divB, v) / Rem + (B[k] / dt if dt > 0 else 0) for k, v in enumerate((X, Y, Z))]
        exact = E + B
    return [_lamb(e, dim) for e in fE + fB], [_lamb(e, dim) for e in exact]


def vel_fields(dim, Re, wconst, dt=0.0, S=0.0, bconst=None):
    """dt > 0: transient source + u/dt; bconst: constant B^n, source + S B x (u x B) (NEXT-4)."""
    pi = sp.pi
    if dim == 2:
        psi = sp.sin(pi * X) ** 2 * sp.sin(pi * Y) ** 2
        u = [sp.diff(psi, Y), -sp.diff(psi, X)]
        vs = (X, Y)
    else:
        psi = sp.sin(pi * X) ** 2 * sp.sin(pi * Y) ** 2 * sp.sin(pi * Z) ** 2
        P = [psi, psi, psi]
        u = [sp.diff(P[2], Y) - sp.diff(P[1], Z), sp.diff(P[0], Z) - sp.diff(P[2], X),
             sp.diff(P[1], X) - sp.diff(P[0], Y)]
        vs = (X, Y, Z)
    # -(2/Re) div eps(u) = -(1/Re) Lap u for div-free u; + (w . grad) u; grad-div term vanishes
    f = []
    for k in range(dim):
        lap = sum(sp.diff(u[k], v, 2) for v in vs)
        adv = sum(wconst[j] * sp.diff(u[k], vs[j]) for j in range(dim))
        f.append(-lap / Re + adv + (u[k] / dt if dt > 0 else 0))
    if bconst is not None:
        Bc = bconst
        if dim == 2:           # u x B = u1 B2 - u2 B1 (scalar); B x s = (B2 s, -B1 s)
            s = u[0] * Bc[1] - u[1] * Bc[0]
            lor = [Bc[1] * s, -Bc[0] * s]
        else:
            uxb = [u[1] * Bc[2] - u[2] * Bc[1], u[2] * Bc[0] - u[0] * Bc[2], u[0] * Bc[1] - u[1] * Bc[0]]
            lor = [Bc[1] * uxb[2] - Bc[2] * uxb[1], Bc[2] * uxb[0] - Bc[0] * uxb[2], Bc[0] * uxb[1] - Bc[1] * uxb[0]]
        f = [f[k] + S * lor[k] for k in range(dim)]
    return [_lamb(e, dim) for e in f], [_lamb(e, dim) for e in u]


def constant_wind_potential(dim, N, wconst):
    """Potential whose discrete field (R-w) is exactly the constant wconst."""
    from paper_2104_14855_b200.workloads import vertex_coords
    P = vertex_coords(dim, N)
    if dim == 2:   # vcurl psi = (d_y psi, -d_x psi) = (w0, w1)  =>  psi = w0 y - w1 x
        return wconst[0] * P[:, 1] - wconst[1] * P[:, 0]
    c = np.asarray(wconst, float)          # A = 1/2 c x x  =>  curl A = c
    A = 0.5 * np.cross(np.broadcast_to(c, P.shape), P)
    return np.ascontiguousarray(A.ravel())


def solve_and_error(orc, fs, exact, level=-1):
    pts, wts, ncomp = orc.quadrature(level)
    fv = np.stack([f(pts) for f in fs], axis=1)
    rhs = orc.load(fv, level)
    A = orc.csr(level).to_scipy().tocsc()
    uh = spla.spsolve(A, rhs)
    vals = orc.eval(uh, level)
    ex = np.stack([e(pts) for e in exact], axis=1)
    err = (vals - ex) ** 2
    return np.sqrt(np.maximum(err.T @ wts, 0.0))   # per component
