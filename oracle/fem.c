/*
 * fem.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Finite-element bases, quadrature and assembly of the two operators whose
 * multigrid relaxation is the hot path:
 *
 *  E-B block  S~(u,p) = [[M_E, G~ - (1/Rem) A], [A^T, C]]
 *      (M_E)_ij = (phi_j, phi_i)          G~_ik = (w x psi_k, phi_i)
 *      A_ik     = (psi_k, vcurl phi_i)    (A^T)_ki = (vcurl phi_i, psi_k)
 *      C_kl     = (1/Rem)(div psi_l, div psi_k)                   Table 1
 *      2D conventions vcurl E = (d_y E, -d_x E), u x B = u1 B2 - u2 B1
 *
 *  AL velocity block (reading R-vel), trial u, test v:
 *      (2/Re)(eps u, eps v)_K  + SIPG  a_h^DG
 *      + gamma (div u, div v)
 *      - (u, div(v (x) w))_K + upwind facet terms c_h^DG (w = advecting field) P:210-216
 *
 * Bases are the dual bases of the DoF functionals of reading R-basis (SURVEY
 * §8c.2): CG1 nodal; NED1 Whitney (int_e E.t = 1); RT1 Whitney (int_f B.n = 1);
 * BDM1 flux-nodal (|f| (u.n_f)(x_a) = 1).  Each local basis function is affine and
 * stored as value at the first cell vertex plus its constant gradient.
 *
 * Integration: cell integrals with a collapsed (Duffy) 3x3(x3) Gauss-Legendre
 * rule (exact for degree <= 4 in 2D, <= 3 in 3D: the Duffy Jacobian adds one degree
 * per collapsed direction; all k = 1 cell integrands have degree <= 2; the 3D k = 2
 * assembly takes the 4-point rule).  Facet
 * integrals with a 3-point (2D) / collapsed 3x3 (3D) Gauss-Legendre rule (exact for
 * degree <= 5 / 4; facet integrands have degree <= 2 because the advecting field w_h
 * is constant per cell, reading R-w).  Nodes and weights are formed in `real` from
 * their closed forms, so in the exact build the rules are exact to ~1e-34.
 * The grad-div / div-div parts are the exact closed form of reading R-gamma:
 * div of an RT/BDM basis function on K is s/(d|K|) (RT: s/|K|), so those entries
 * equal (G * m) / d^2 with G = gamma/|K| and m an integer sum of orientation signs.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "orc.h"

/* Precision of the element integrals and of their accumulation (reading R-exact):
 * the oracle is compiled twice from this file.  liboracle.so uses real = double (fast;
 * the finite-element pins); liboracle_exact.so uses real = __float128 (113-bit), so every
 * assembled entry is the fp64 value nearest to the exact discrete bilinear form for the
 * given fp64 inputs -- the reference for the end-to-end parity tests.  The final
 * rounding of each row goes through a grid 2^-88 below the row's largest entry (see
 * finish()), so that exact ties round to even and exact cancellations give 0.         */
#ifdef ORC_EXACT
#include <quadmath.h>
typedef __float128 real;
#define RSQRT(x) sqrtq(x)
#define RFABS(x) fabsq(x)
#else
typedef double real;
#define RSQRT(x) sqrt(x)
#define RFABS(x) fabs(x)
#endif

/* ------------------------------------------------------------------------- */
/* geometry                                                                   */
/* ------------------------------------------------------------------------- */
typedef struct {
    int dim;
    real X[4][3];       /* vertices (ascending global id)   */
    real Ji[3][3];      /* inverse Jacobian                  */
    real det, vol;
    real g[4][3];       /* gradients of barycentric coords   */
} Cell;

typedef struct { real v0[3]; real G[3][3]; } Aff;  /* f(x) = v0 + G (x - X0) */

/* geometry of the simplex with vertices X (ascending global id) */
static void cell_geom_from(int d, const real X[4][3], Cell *K) {
    memset(K, 0, sizeof(*K));
    K->dim = d;
    memcpy(K->X, X, sizeof(K->X));
    real J[3][3] = {{0}};
    for (int r = 0; r < d; r++)
        for (int col = 0; col < d; col++) J[r][col] = K->X[col + 1][r] - K->X[0][r];
    if (d == 2) {
        K->det = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        K->Ji[0][0] = J[1][1] / K->det; K->Ji[0][1] = -J[0][1] / K->det;
        K->Ji[1][0] = -J[1][0] / K->det; K->Ji[1][1] = J[0][0] / K->det;
        K->vol = RFABS(K->det) / 2;
    } else {
        real co[3][3];
        co[0][0] = J[1][1] * J[2][2] - J[1][2] * J[2][1];
        co[0][1] = J[1][2] * J[2][0] - J[1][0] * J[2][2];
        co[0][2] = J[1][0] * J[2][1] - J[1][1] * J[2][0];
        co[1][0] = J[0][2] * J[2][1] - J[0][1] * J[2][2];
        co[1][1] = J[0][0] * J[2][2] - J[0][2] * J[2][0];
        co[1][2] = J[0][1] * J[2][0] - J[0][0] * J[2][1];
        co[2][0] = J[0][1] * J[1][2] - J[0][2] * J[1][1];
        co[2][1] = J[0][2] * J[1][0] - J[0][0] * J[1][2];
        co[2][2] = J[0][0] * J[1][1] - J[0][1] * J[1][0];
        K->det = J[0][0] * co[0][0] + J[0][1] * co[0][1] + J[0][2] * co[0][2];
        for (int r = 0; r < 3; r++)
            for (int col = 0; col < 3; col++) K->Ji[r][col] = co[col][r] / K->det;
        K->vol = RFABS(K->det) / 6;
    }
    for (int a = 1; a <= d; a++)
        for (int k = 0; k < d; k++) K->g[a][k] = K->Ji[a - 1][k];
    for (int k = 0; k < d; k++) {
        real s = 0;
        for (int a = 1; a <= d; a++) s += K->g[a][k];
        K->g[0][k] = -s;
    }
}

/* vertex coordinates formed in `real` from the integer lattice: x = (i,j,k)/N */
static void cell_geom(const OMesh *m, i64 c, Cell *K) {
    int d = m->dim;
    real X[4][3] = {{0}};
    for (int a = 0; a <= d; a++)
        for (int r = 0; r < d; r++) X[a][r] = (real)m->lat[3 * m->cv[c * (d + 1) + a] + r] / (real)m->N;
    cell_geom_from(d, X, K);
}

static void aff_eval(const Aff *f, const Cell *K, const real *x, real *out) {
    for (int l = 0; l < 3; l++) {
        real s = f->v0[l];
        for (int k = 0; k < K->dim; k++) s += f->G[l][k] * (x[k] - K->X[0][k]);
        out[l] = s;
    }
}

static real dot3(const real *a, const real *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
static void cross3(const real *a, const real *b, real *c) {
    c[0] = a[1] * b[2] - a[2] * b[1]; c[1] = a[2] * b[0] - a[0] * b[2]; c[2] = a[0] * b[1] - a[1] * b[0];
}

/* global facet area vector |f| n_f of the facet with ascending vertices P:
 * 2D edge (a<b): n = (t_y, -t_x) (tangent rotated clockwise);
 * 3D face (a<b<c): n ~ (x_b - x_a) x (x_c - x_a).         reading R-orient    */
static void facet_area_vector(int dim, const real P[3][3], real *A) {
    if (dim == 2) {
        A[0] = P[1][1] - P[0][1]; A[1] = -(P[1][0] - P[0][0]); A[2] = 0;
    } else {
        real u[3], v[3];
        for (int k = 0; k < 3; k++) { u[k] = P[1][k] - P[0][k]; v[k] = P[2][k] - P[0][k]; }
        cross3(u, v, A);
        for (int k = 0; k < 3; k++) A[k] /= 2;
    }
}

/* Advecting field w_h on cell K (reading R-w): exactly divergence-free, as the
 * paper requires of u^n ("we exactly enforce div u^n = 0"; BDM u^n).
 *   2D: w_h = vcurl psi_h, psi_h the CG1 interpolant of the stream function
 *       (pot = psi at the cell's vertices);
 *   3D: w_h = curl A_h, A_h the NED1 interpolant of the P1 interpolant of the
 *       vector potential (pot = A at the cell's vertices): edge circulation
 *       c_e = (A_i + A_j)/2 . (X_j - X_i), curl(lam_i grad lam_j - lam_j grad lam_i)
 *       = 2 grad lam_i x grad lam_j.
 * w_h is constant on K, normal-continuous across facets, and lies in RT_0 in BDM_1. */
static void cell_wind(const Cell *K, const double pot[4][3], real *wc) {
    wc[0] = wc[1] = wc[2] = 0;
    if (K->dim == 2) {
        real gx = 0, gy = 0;
        for (int a = 0; a < 3; a++) { gx += pot[a][0] * K->g[a][0]; gy += pot[a][0] * K->g[a][1]; }
        wc[0] = gy; wc[1] = -gx;
        return;
    }
    for (int q = 0; q < 6; q++) {
        int lv[2];
        om_edge_local_verts(3, q, lv);
        int i = lv[0], j = lv[1];
        real ce = 0;
        for (int k = 0; k < 3; k++) ce += ((real)pot[i][k] + (real)pot[j][k]) / 2 * (K->X[j][k] - K->X[i][k]);
        real cr[3];
        cross3(K->g[i], K->g[j], cr);
        for (int k = 0; k < 3; k++) wc[k] += ce * 2 * cr[k];
    }
}

static void cell_pot(const OMesh *m, i64 c, const double *pot, double out[4][3]) {
    int d = m->dim, nc = d == 2 ? 1 : 3;
    memset(out, 0, sizeof(double) * 12);
    for (int a = 0; a <= d; a++)
        for (int k = 0; k < nc; k++) out[a][k] = pot[(i64)m->cv[c * (d + 1) + a] * nc + k];
}

/* ------------------------------------------------------------------------- */
/* local bases (dual to the DoF functionals of R-basis)                        */
/* ------------------------------------------------------------------------- */
static Aff basis_cg1(const Cell *K, int a) {
    Aff f; memset(&f, 0, sizeof(f));
    f.v0[0] = a == 0 ? 1 : 0;
    for (int k = 0; k < K->dim; k++) f.G[0][k] = K->g[a][k];
    return f;
}

/* Whitney edge function lam_i grad lam_j - lam_j grad lam_i, local i < j */
static Aff basis_ned1(const Cell *K, int i, int j) {
    Aff f; memset(&f, 0, sizeof(f));
    for (int l = 0; l < 3; l++) {
        f.v0[l] = (i == 0 ? K->g[j][l] : (real)0) - (j == 0 ? K->g[i][l] : (real)0);
        for (int k = 0; k < 3; k++) f.G[l][k] = K->g[j][l] * K->g[i][k] - K->g[i][l] * K->g[j][k];
    }
    return f;
}

/* orientation sign of local facet q: +1 if the global facet normal points out of K */
static double facet_sign(const Cell *K, int q, const real A[3]) {
    int d = K->dim, opp = om_facet_opp(d, q), lv[3];
    om_facet_local_verts(d, q, lv);
    real t[3];
    for (int k = 0; k < 3; k++) t[k] = K->X[lv[0]][k] - K->X[opp][k];
    return dot3(A, t) > 0 ? 1.0 : -1.0;
}

static void facet_points(const Cell *K, int q, real P[3][3]) {
    int lv[3];
    om_facet_local_verts(K->dim, q, lv);
    memset(P, 0, sizeof(real) * 9);
    for (int a = 0; a < K->dim; a++)
        for (int k = 0; k < 3; k++) P[a][k] = K->X[lv[a]][k];
}

/* RT1: s (x - X_opp) / (d |K|)  (flux 1 through facet q along its global normal) */
static Aff basis_rt(const Cell *K, int q, double *sign) {
    Aff f; memset(&f, 0, sizeof(f));
    real P[3][3], A[3];
    facet_points(K, q, P);
    facet_area_vector(K->dim, P, A);
    double s = facet_sign(K, q, A);
    int opp = om_facet_opp(K->dim, q);
    real c = s / (K->dim * K->vol);
    for (int l = 0; l < 3; l++) {
        f.v0[l] = c * (K->X[0][l] - K->X[opp][l]);
        for (int k = 0; k < 3; k++) f.G[l][k] = (l == k && l < K->dim) ? c : (real)0;
    }
    *sign = s;
    return f;
}

/* BDM1 flux-nodal: lam_a psi, psi orthogonal to the normals of the other facets
 * through vertex a, scaled so that psi . (|f| n_f) = 1.                         */
static Aff basis_bdm(const Cell *K, int q, int ia, double *sign) {
    Aff f; memset(&f, 0, sizeof(f));
    int d = K->dim, lv[3];
    om_facet_local_verts(d, q, lv);
    real P[3][3], A[3], dir[3] = {0, 0, 0};
    facet_points(K, q, P);
    facet_area_vector(d, P, A);
    int a = lv[ia];
    if (d == 2) {
        int b = lv[1 - ia];
        dir[0] = -K->g[b][1]; dir[1] = K->g[b][0];
    } else {
        int b = lv[(ia + 1) % 3], c = lv[(ia + 2) % 3];
        cross3(K->g[b], K->g[c], dir);
    }
    real sc = dot3(dir, A);
    real psi[3] = {dir[0] / sc, dir[1] / sc, dir[2] / sc};
    for (int l = 0; l < 3; l++) {
        f.v0[l] = (a == 0 ? psi[l] : (real)0);
        for (int k = 0; k < 3; k++) f.G[l][k] = k < d ? psi[l] * K->g[a][k] : (real)0;
    }
    *sign = facet_sign(K, q, A);
    return f;
}

/* ------------------------------------------------------------------------- */
/* quadrature                                                                  */
/* ------------------------------------------------------------------------- */
static void gauss01(int q, real *x, real *w) {
    /* Gauss-Legendre nodes / weights on [0,1], formed in `real` from their closed forms */
    if (q == 3) {
        real r = RSQRT((real)3 / 5) / 2;
        x[0] = (real)1 / 2 - r; x[1] = (real)1 / 2; x[2] = (real)1 / 2 + r;
        w[0] = (real)5 / 18; w[1] = (real)8 / 18; w[2] = (real)5 / 18;
    } else { /* q == 4 */
        real s65 = RSQRT((real)6 / 5), s30 = RSQRT((real)30);
        real a = RSQRT((real)3 / 7 - (real)2 / 7 * s65);
        real b = RSQRT((real)3 / 7 + (real)2 / 7 * s65);
        real wa = (18 + s30) / 36, wb = (18 - s30) / 36;
        x[0] = (1 - b) / 2; x[1] = (1 - a) / 2; x[2] = (1 + a) / 2; x[3] = (1 + b) / 2;
        w[0] = wb / 2; w[1] = wa / 2; w[2] = wa / 2; w[3] = wb / 2;
    }
}

/* collapsed (Duffy) Gauss rule with q points per direction on the cell: physical points
 * and weights.  Gauss-Legendre in each direction is exact to degree 2q-1, and the Duffy
 * Jacobian (1-eta) / (1-eta)(1-zeta)^2 adds one degree per collapsed direction, so the
 * rule is exact to degree 2q-2 in 2D and 2q-3 in 3D: q = 3 (9 / 27 points) -> 4 / 3,
 * q = 4 -> 6 / 5.  The k = 1 assembly (cell integrands of degree <= 2) and the 2D k = 2
 * assembly (degree <= 4) use q = 3; the 3D k = 2 assembly (degree 4) uses q = 4, as do
 * the manufactured-solution helpers, whose integrands are not polynomial. */
static int cell_rule(const Cell *K, int q, real (*xq)[3], real *wq) {
    real g[4], w[4];
    gauss01(q, g, w);
    int n = 0;
    if (K->dim == 2) {
        for (int i = 0; i < q; i++)
            for (int j = 0; j < q; j++) {
                real xi1 = g[i] * (1 - g[j]), xi2 = g[j];
                real wt = w[i] * w[j] * (1 - g[j]) * RFABS(K->det);
                for (int k = 0; k < 3; k++)
                    xq[n][k] = K->X[0][k] + xi1 * (K->X[1][k] - K->X[0][k]) + xi2 * (K->X[2][k] - K->X[0][k]);
                wq[n++] = wt;
            }
    } else {
        for (int i = 0; i < q; i++)
            for (int j = 0; j < q; j++)
                for (int l = 0; l < q; l++) {
                    real xi1 = g[i] * (1 - g[j]) * (1 - g[l]), xi2 = g[j] * (1 - g[l]), xi3 = g[l];
                    real wt = w[i] * w[j] * w[l] * (1 - g[j]) * (1 - g[l]) * (1 - g[l]) * RFABS(K->det);
                    for (int k = 0; k < 3; k++)
                        xq[n][k] = K->X[0][k] + xi1 * (K->X[1][k] - K->X[0][k]) + xi2 * (K->X[2][k] - K->X[0][k]) +
                                   xi3 * (K->X[3][k] - K->X[0][k]);
                    wq[n++] = wt;
                }
    }
    return n;
}

/* facet rule (R-quad): 3-point Gauss-Legendre (2D edge) / collapsed 3x3 (3D triangle),
 * exact to degree 5 / 4; facet integrands have degree <= 2 */
static int facet_rule(int dim, const real P[3][3], real (*xq)[3], real *wq) {
    real g[3], w[3];
    gauss01(3, g, w);
    int n = 0;
    if (dim == 2) {
        real t[3] = {P[1][0] - P[0][0], P[1][1] - P[0][1], 0};
        real len = RSQRT(dot3(t, t));
        for (int i = 0; i < 3; i++) {
            for (int k = 0; k < 3; k++) xq[n][k] = P[0][k] + g[i] * t[k];
            wq[n++] = w[i] * len;
        }
    } else {
        real A[3];
        facet_area_vector(3, P, A);
        real area = RSQRT(dot3(A, A));
        for (int i = 0; i < 3; i++)
            for (int j = 0; j < 3; j++) {
                real xi1 = g[i] * (1 - g[j]), xi2 = g[j];
                for (int k = 0; k < 3; k++)
                    xq[n][k] = P[0][k] + xi1 * (P[1][k] - P[0][k]) + xi2 * (P[2][k] - P[0][k]);
                wq[n++] = w[i] * w[j] * (1 - g[j]) * 2 * area;
            }
    }
    return n;
}

/* ------------------------------------------------------------------------- */
/* CSR helpers and sparsity                                                   */
/* ------------------------------------------------------------------------- */
void oc_free(OCsr *a) { free(a->rp); free(a->ci); free(a->v); memset(a, 0, sizeof(*a)); }

i64 oc_find(const OCsr *a, i64 row, int col) {
    i64 lo = a->rp[row], hi = a->rp[row + 1] - 1;
    while (lo <= hi) {
        i64 mid = (lo + hi) / 2;
        if (a->ci[mid] == col) return mid;
        if (a->ci[mid] < col) lo = mid + 1; else hi = mid - 1;
    }
    return -1;
}

/* free DoFs (with -1 for constrained) of the local basis of cell c, in local order */
static int cell_dofs(const OMesh *m, const OSpace *s, i64 c, int *out) {
    int d = m->dim, n = 0;
    if (s->degree == 2 && d == 3 && s->block == ORC_EB) {   /* NED1_2 (edges x 2, faces x 2) then RT2 (faces x 3, cell x 3) */
        for (int q = 0; q < 6; q++) { int e0 = s->edof[m->ce[c * 6 + q]]; for (int a = 0; a < 2; a++) out[n++] = e0 < 0 ? -1 : e0 + a; }
        for (int q = 0; q < 4; q++) { int g0 = s->gdof[om_facet_of_cell(m, c, q)]; for (int a = 0; a < 2; a++) out[n++] = g0 < 0 ? -1 : g0 + a; }
        for (int q = 0; q < 4; q++) { int f0 = s->fdof[om_facet_of_cell(m, c, q)]; for (int a = 0; a < 3; a++) out[n++] = f0 < 0 ? -1 : f0 + a; }
        for (int a = 0; a < 3; a++) out[n++] = s->cdof[c] + a;
        return n;
    }
    if (s->degree == 2 && s->block == ORC_VEL) {   /* BDM2: facets x 3 (2D) / 6 (3D), then cell x 3 / 6 */
        int per = d == 2 ? 3 : 6;
        for (int q = 0; q <= d; q++) {
            int f0 = s->fdof[om_facet_of_cell(m, c, q)];
            for (int a = 0; a < per; a++) out[n++] = f0 < 0 ? -1 : f0 + a;
        }
        for (int a = 0; a < per; a++) out[n++] = s->cdof[c] + a;
        return n;
    }
    if (s->degree == 2) {             /* CG2 (vertices, edges) then RT2 (edges x 2, cell x 2) */
        for (int a = 0; a < 3; a++) out[n++] = s->vdof[m->cv[c * 3 + a]];
        for (int q = 0; q < 3; q++) out[n++] = s->edof[m->ce[c * 3 + q]];
        for (int q = 0; q < 3; q++) {
            int f0 = s->fdof[om_facet_of_cell(m, c, q)];
            out[n++] = f0 < 0 ? -1 : f0;
            out[n++] = f0 < 0 ? -1 : f0 + 1;
        }
        out[n++] = s->cdof[c]; out[n++] = s->cdof[c] + 1;
        return n;
    }
    if (s->block == ORC_EB) {
        if (d == 2) for (int a = 0; a < 3; a++) out[n++] = s->vdof[m->cv[c * 3 + a]];
        else for (int q = 0; q < 6; q++) out[n++] = s->edof[m->ce[c * 6 + q]];
        for (int q = 0; q <= d; q++) out[n++] = s->fdof[om_facet_of_cell(m, c, q)];
    } else {
        for (int q = 0; q <= d; q++) {
            int f0 = s->fdof[om_facet_of_cell(m, c, q)];
            for (int a = 0; a < d; a++) out[n++] = f0 < 0 ? -1 : f0 + a;
        }
    }
    return n;
}

static int cmp_int(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return x < y ? -1 : x > y;
}

/* Sparsity: DoFs i, j couple iff their basis functions share a cell (E-B), or
 * share a cell or the two cells of one facet (DG velocity).          */
static void build_pattern(OCsr *A, const OMesh *m, const OSpace *s) {
    i64 n = s->n;
    int ld[64];
    i64 *sp = calloc((size_t)n + 1, sizeof(i64));
    for (i64 c = 0; c < m->nc; c++) {
        int k = cell_dofs(m, s, c, ld);
        for (int t = 0; t < k; t++) if (ld[t] >= 0) sp[ld[t] + 1]++;
    }
    for (i64 d = 0; d < n; d++) sp[d + 1] += sp[d];
    int *sc = malloc(sizeof(int) * (sp[n] ? sp[n] : 1));
    i64 *fill = calloc((size_t)n, sizeof(i64));
    for (i64 c = 0; c < m->nc; c++) {
        int k = cell_dofs(m, s, c, ld);
        for (int t = 0; t < k; t++) if (ld[t] >= 0) sc[sp[ld[t]] + fill[ld[t]]++] = (int)c;
    }
    free(fill);
    A->n = n;
    A->rp = malloc(sizeof(i64) * (n + 1));
    A->rp[0] = 0;
    i64 cap = n * 16 + 16, used = 0;
    A->ci = malloc(sizeof(int) * cap);
    int *buf = malloc(sizeof(int) * 8192);
    for (i64 d = 0; d < n; d++) {
        int nb = 0;
        for (i64 t = sp[d]; t < sp[d + 1]; t++) {
            int cells[5], ncell = 0;
            i64 c = sc[t];
            cells[ncell++] = (int)c;
            if (s->block == ORC_VEL)
                for (int q = 0; q <= m->dim; q++) {
                    int f = om_facet_of_cell(m, c, q);
                    int o = m->fcell[2 * f] == c ? m->fcell[2 * f + 1] : m->fcell[2 * f];
                    if (o >= 0) cells[ncell++] = o;
                }
            for (int u = 0; u < ncell; u++) {
                int k = cell_dofs(m, s, cells[u], ld);
                for (int v = 0; v < k; v++) if (ld[v] >= 0) buf[nb++] = ld[v];
            }
        }
        qsort(buf, (size_t)nb, sizeof(int), cmp_int);
        int nu = 0;
        for (int u = 0; u < nb; u++) if (u == 0 || buf[u] != buf[u - 1]) buf[nu++] = buf[u];
        while (used + nu > cap) { cap *= 2; A->ci = realloc(A->ci, sizeof(int) * cap); }
        memcpy(A->ci + used, buf, sizeof(int) * nu);
        used += nu;
        A->rp[d + 1] = used;
    }
    A->nnz = used;
    A->ci = realloc(A->ci, sizeof(int) * (used ? used : 1));
    A->v = calloc((size_t)(used ? used : 1), sizeof(double));
    free(buf); free(sp); free(sc);
}

/* accumulator of the assembly: per nonzero, the running sum in `real` */
typedef struct {
    real *acc;
} Accum;

static void scatter(const OCsr *A, Accum *S, const int *gi, int ni, const int *gj, int nj, const real *loc, int ldl) {
    for (int i = 0; i < ni; i++) {
        if (gi[i] < 0) continue;
        for (int j = 0; j < nj; j++) {
            if (gj[j] < 0) continue;
            i64 p = oc_find(A, gi[i], gj[j]);
            S->acc[p] += loc[i * ldl + j];
        }
    }
}

/* Reading R-exact, row by row: E = exponent of the largest |entry| of the row
 * (max |x| = m 2^E, 1/2 <= m < 1, after rounding to fp64), G = 2^(E-88); every entry x
 * becomes RN53(G * nearest_integer(x / G)).  x is split as hi + lo (hi = RN53(x),
 * lo = RN53(x - hi)) and the grid rounding is done on the two doubles.               */
static double grid_round(double hi, double lo, int E) {
    double H = ldexp(hi, 88 - E), L = ldexp(lo, 88 - E);
    double N = nearbyint(H);
    double k = nearbyint((H - N) + L);
    double v = ldexp(N + k, E - 88);
    return v == 0 ? 0.0 : v;      /* exact cancellation: +0 */
}

static void finish_floor(OCsr *A, const Accum *S, const double *floor) {
    for (i64 i = 0; i < A->n; i++) {
        double mx = floor ? floor[i] : 0;
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) {
            double h = (double)S->acc[t];
            if (fabs(h) > mx) mx = fabs(h);
        }
        int E = 0;
        if (mx > 0) frexp(mx, &E);
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) {
            double h = (double)S->acc[t];
            double l = (double)(S->acc[t] - (real)h);
            A->v[t] = mx > 0 ? grid_round(h, l, E) : 0.0;
        }
    }
}

static void finish(OCsr *A, const Accum *S) { finish_floor(A, S, NULL); }

/* ------------------------------------------------------------------------- */
/* E-B block  (Table 1)                       */
/* ------------------------------------------------------------------------- */
static void assemble_eb(OCsr *A, Accum *S, signed char *cnt, const OMesh *m, const OSpace *s, const OParams *p,
                        const double *w, const unsigned char *cmask) {
    int d = m->dim, nEl = d == 2 ? 3 : 6, nBl = d + 1;
    real xq[64][3], wq[64];
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Aff E[6], B[4];
        double sB[4];
        int gE[6], gB[4];
        for (int a = 0; a < nEl; a++) {
            if (d == 2) { E[a] = basis_cg1(&K, a); gE[a] = s->vdof[m->cv[c * 3 + a]]; }
            else {
                int lv[2];
                om_edge_local_verts(3, a, lv);
                E[a] = basis_ned1(&K, lv[0], lv[1]);
                gE[a] = s->edof[m->ce[c * 6 + a]];
            }
        }
        for (int q = 0; q < nBl; q++) { B[q] = basis_rt(&K, q, &sB[q]); gB[q] = s->fdof[om_facet_of_cell(m, c, q)]; }
        /* vcurl / curl of the E basis (constant) */
        real curlE[6][3];
        for (int a = 0; a < nEl; a++) {
            if (d == 2) { curlE[a][0] = E[a].G[0][1]; curlE[a][1] = -E[a].G[0][0]; curlE[a][2] = 0; }
            else {
                curlE[a][0] = E[a].G[2][1] - E[a].G[1][2];
                curlE[a][1] = E[a].G[0][2] - E[a].G[2][0];
                curlE[a][2] = E[a].G[1][0] - E[a].G[0][1];
            }
        }
        double pot[4][3];
        real wx[3];
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        real EE[6 * 6] = {0}, EB[6 * 4] = {0}, BE[4 * 6] = {0}, BB[4 * 4] = {0};
        int nq = cell_rule(&K, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real ev[6][3], bv[4][3];
            for (int a = 0; a < nEl; a++) aff_eval(&E[a], &K, xq[t], ev[a]);
            for (int q = 0; q < nBl; q++) aff_eval(&B[q], &K, xq[t], bv[q]);
            for (int i = 0; i < nEl; i++) {
                for (int j = 0; j < nEl; j++)
                    EE[i * 6 + j] += wq[t] * (d == 2 ? ev[j][0] * ev[i][0] : dot3(ev[j], ev[i]));
                for (int k = 0; k < nBl; k++) {
                    real wxb;
                    if (d == 2) wxb = (wx[0] * bv[k][1] - wx[1] * bv[k][0]) * ev[i][0];
                    else { real cr[3]; cross3(wx, bv[k], cr); wxb = dot3(cr, ev[i]); }
                    if (p->picard) wxb = 0;                      /* delta = 0 */
                    real ab = dot3(bv[k], curlE[i]);
                    EB[i * 4 + k] += wq[t] * (wxb - ab / p->Rem);
                    BE[k * 6 + i] += wq[t] * ab;
                }
            }
            /* transient (eta = 1): (1/dt)(B, C) in the B-B block */
            if (p->dt > 0)
                for (int k = 0; k < nBl; k++)
                    for (int l = 0; l < nBl; l++) BB[k * 4 + l] += wq[t] * dot3(bv[l], bv[k]) / p->dt;
        }
        scatter(A, S, gE, nEl, gE, nEl, EE, 6);
        scatter(A, S, gE, nEl, gB, nBl, EB, 4);
        scatter(A, S, gB, nBl, gE, nEl, BE, 6);
        if (p->dt > 0) scatter(A, S, gB, nBl, gB, nBl, BB, 4);
        for (int k = 0; k < nBl; k++)
            for (int l = 0; l < nBl; l++)
                if (gB[k] >= 0 && gB[l] >= 0) cnt[oc_find(A, gB[k], gB[l])] += (signed char)(sB[k] * sB[l]);
    }
    /* C = (1/Rem)(div psi_l, div psi_k), div psi = s/|K|: exact value (Kinv*m)/Rem (R-gamma) */
    double Kinv = d == 2 ? 2.0 * m->N * m->N : 6.0 * m->N * m->N * m->N;
    for (i64 t = 0; t < A->nnz; t++)
        if (cnt[t]) S->acc[t] += (real)(Kinv * cnt[t]) / p->Rem;
}

/* ------------------------------------------------------------------------- */
/* AL velocity block (R-vel)                                                  */
/* ------------------------------------------------------------------------- */
static int vel_basis(const OMesh *m, const OSpace *s, i64 c, const Cell *K, Aff *F, double *sg, int *gi) {
    int d = m->dim, n = 0;
    for (int q = 0; q <= d; q++) {
        int f0 = s->fdof[om_facet_of_cell(m, c, q)];
        for (int a = 0; a < d; a++) {
            double sgn;
            F[n] = basis_bdm(K, q, a, &sgn);
            if (sg) sg[n] = sgn;
            gi[n] = f0 < 0 ? -1 : f0 + a;
            n++;
        }
    }
    return n;
}

static void sym_grad(const Aff *f, real e[3][3]) {
    for (int l = 0; l < 3; l++) for (int k = 0; k < 3; k++) e[l][k] = (f->G[l][k] + f->G[k][l]) / 2;
}

static void assemble_vel(OCsr *A, Accum *S, signed char *cnt, const OMesh *m, const OSpace *s, const OParams *p,
                         const double *w, const unsigned char *cmask) {
    int d = m->dim;
    real xq[64][3], wq[64];
    const real nu2 = (real)2 / p->Re;
    /* cell terms */
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Aff F[12];
        double sg[12];
        int gi[12];
        int nb = vel_basis(m, s, c, &K, F, sg, gi);
        real eps[12][3][3];
        for (int a = 0; a < nb; a++) sym_grad(&F[a], eps[a]);
        double pot[4][3];
        real wx[3], bx[3] = {0, 0, 0};
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);      /* constant on K, div w_h = 0 */
        if (p->bn) { double bp[4][3]; cell_pot(m, c, p->bn, bp); cell_wind(&K, bp, bx); }   /* B^n, NEXT-4 */
        real loc[12 * 12] = {0};
        int nq = cell_rule(&K, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[12][3];
            for (int a = 0; a < nb; a++) aff_eval(&F[a], &K, xq[t], fv[a]);
            for (int i = 0; i < nb; i++) {
                /* div(v (x) w)_l = sum_k (d_k v_l) w_k + v_l div w, div w_h = 0  (v = test fn i) */
                real dvw[3];
                for (int l = 0; l < 3; l++) {
                    real sacc = 0;
                    for (int k = 0; k < d; k++) sacc += F[i].G[l][k] * wx[k];
                    dvw[l] = sacc;
                }
                for (int j = 0; j < nb; j++) {
                    real ee = 0;
                    for (int l = 0; l < 3; l++) for (int k = 0; k < 3; k++) ee += eps[j][l][k] * eps[i][l][k];
                    real mass = p->dt > 0 ? dot3(fv[j], fv[i]) / p->dt : (real)0;   /* (eta/dt)(u, v) */
                    real lor = 0;                                 /* S (u x B^n, v x B^n), NEXT-4 */
                    if (p->bn) {
                        if (d == 2) lor = (fv[j][0] * bx[1] - fv[j][1] * bx[0]) * (fv[i][0] * bx[1] - fv[i][1] * bx[0]);
                        else { real cj[3], ci[3]; cross3(fv[j], bx, cj); cross3(fv[i], bx, ci); lor = dot3(cj, ci); }
                        lor *= p->S;
                    }
                    loc[i * 12 + j] += wq[t] * (nu2 * ee - dot3(fv[j], dvw) + mass + lor);
                }
            }
        }
        scatter(A, S, gi, nb, gi, nb, loc, 12);
        for (int i = 0; i < nb; i++)
            for (int j = 0; j < nb; j++)
                if (gi[i] >= 0 && gi[j] >= 0) cnt[oc_find(A, gi[i], gi[j])] += (signed char)(sg[i] * sg[j]);
    }
    /* facet terms: SIPG + upwind (reading R-vel) */
    static real loc[24 * 24];
    for (i64 f = 0; f < m->nfacet; f++) {
        int cp = m->fcell[2 * f], cm = m->fcell[2 * f + 1];
        if (cmask && !cmask[cp] && !(cm >= 0 && cmask[cm])) continue;
        int interior = cm >= 0;
        Cell Kp, Km;
        Aff F[24];
        double sg[24];
        int gi[24], side[24];
        cell_geom(m, cp, &Kp);
        int nb = vel_basis(m, s, cp, &Kp, F, sg, gi);
        for (int a = 0; a < nb; a++) side[a] = +1;
        if (interior) {
            cell_geom(m, cm, &Km);
            int nb2 = vel_basis(m, s, cm, &Km, F + nb, sg + nb, gi + nb);
            for (int a = nb; a < nb + nb2; a++) side[a] = -1;
            nb += nb2;
        }
        /* facet vertices (ascending global id) and K+'s outward unit normal */
        int qf = -1;
        for (int q = 0; q <= d; q++) if (om_facet_of_cell(m, cp, q) == f) qf = q;
        real P[3][3], Av[3];
        facet_points(&Kp, qf, P);
        facet_area_vector(d, P, Av);
        real an = RSQRT(dot3(Av, Av)), n[3];
        double sgn = facet_sign(&Kp, qf, Av);
        for (int k = 0; k < 3; k++) n[k] = sgn * Av[k] / an;
        real hF;
        if (d == 2) hF = an;
        else {
            hF = 0;
            for (int a = 0; a < 3; a++)
                for (int b = a + 1; b < 3; b++) {
                    real t[3] = {P[b][0] - P[a][0], P[b][1] - P[a][1], P[b][2] - P[a][2]};
                    real l = RSQRT(dot3(t, t));
                    if (l > hF) hF = l;
                }
        }
        real avg = interior ? (real)1 / 2 : (real)1;
        real pen = (real)p->sigma / ((real)p->Re * hF);
        /* Burman stabilisation: (1/2) sum_K int_{dK} mu h^2 [grad u]:[grad v] ds.
         * Reading R-mu: the jump lives on interior facets, each met from both of its cells
         * (the 1/2), so every interior facet adds mu h_F^2 int_F [grad u]:[grad v]; h_F as for
         * SIPG (edge length / longest face edge), h_F^2 taken without the square root.   */
        real hF2 = 0;
        if (d == 2) hF2 = dot3(Av, Av);
        else
            for (int a = 0; a < 3; a++)
                for (int b = a + 1; b < 3; b++) {
                    real t[3] = {P[b][0] - P[a][0], P[b][1] - P[a][1], P[b][2] - P[a][2]};
                    if (dot3(t, t) > hF2) hF2 = dot3(t, t);
                }
        real burman = interior ? (real)p->mu * hF2 : (real)0;
        double pot[4][3];
        real wx[3];
        cell_pot(m, cp, w, pot);
        cell_wind(&Kp, pot, wx);     /* w_h . n is continuous; K+'s value is used (R-w) */
        real wn = dot3(wx, n), awn = RFABS(wn);
        real epsn[24][3];
        for (int a = 0; a < nb; a++) {
            real e[3][3];
            sym_grad(&F[a], e);
            for (int l = 0; l < 3; l++) epsn[a][l] = e[l][0] * n[0] + e[l][1] * n[1] + e[l][2] * n[2];
        }
        memset(loc, 0, sizeof(loc));
        int nq = facet_rule(d, P, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[24][3];
            for (int a = 0; a < nb; a++) aff_eval(&F[a], side[a] > 0 ? &Kp : &Km, xq[t], fv[a]);
            for (int i = 0; i < nb; i++) {
                real Ji = side[i];
                for (int j = 0; j < nb; j++) {
                    real Jj = side[j];
                    real vv = dot3(fv[j], fv[i]);
                    real t1 = -nu2 * avg * dot3(epsn[j], fv[i]) * Ji;
                    real t2 = -nu2 * avg * dot3(fv[j], epsn[i]) * Jj;
                    real t3 = pen * Jj * Ji * vv;
                    real up;
                    if (interior) up = (side[j] > 0 ? (wn + awn) / 2 : -(-wn + awn) / 2) * vv * Ji;
                    else up = (wn + awn) / 2 * vv;
                    real gj = 0;                 /* [grad phi_j] : [grad phi_i] */
                    if (burman != 0)
                        for (int l = 0; l < 3; l++) for (int k = 0; k < 3; k++) gj += F[j].G[l][k] * F[i].G[l][k];
                    loc[i * 24 + j] += wq[t] * (t1 + t2 + t3 + up + burman * Jj * Ji * gj);
                }
            }
        }
        scatter(A, S, gi, nb, gi, nb, loc, 24);
    }
    /* gamma (div u, div v): div phi_{f,a} = s/(d|K|); exact value (G m)/d^2, G = gamma/|K| (R-gamma) */
    double Kinv = d == 2 ? 2.0 * m->N * m->N : 6.0 * m->N * m->N * m->N;
    double G = p->gamma * Kinv;
    for (i64 t = 0; t < A->nnz; t++)
        if (cnt[t]) S->acc[t] += (real)(G * cnt[t]) / (d * d);
}

static void assemble_eb2(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                         const unsigned char *cmask);
static void assemble_vel2(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                          const unsigned char *cmask);
static void assemble_eb2_3d(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                            const unsigned char *cmask);
static void assemble_vel2_3d(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                             const unsigned char *cmask);

int oa_assemble_masked(OCsr *A, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                       const unsigned char *cmask) {
    build_pattern(A, m, s);
    if (s->degree == 2) {
        Accum S2;
        S2.acc = calloc((size_t)(A->nnz ? A->nnz : 1), sizeof(real));
        if (s->block == ORC_VEL && m->dim == 3) assemble_vel2_3d(A, &S2, m, s, p, w, cmask);
        else if (s->block == ORC_VEL) assemble_vel2(A, &S2, m, s, p, w, cmask);
        else if (m->dim == 3) assemble_eb2_3d(A, &S2, m, s, p, w, cmask);
        else assemble_eb2(A, &S2, m, s, p, w, cmask);
        finish(A, &S2);
        free(S2.acc);
        return 0;
    }
    signed char *cnt = calloc((size_t)(A->nnz ? A->nnz : 1), 1);
    Accum S;
    S.acc = calloc((size_t)(A->nnz ? A->nnz : 1), sizeof(real));
    if (s->block == ORC_EB) assemble_eb(A, &S, cnt, m, s, p, w, cmask);
    else assemble_vel(A, &S, cnt, m, s, p, w, cmask);
    finish(A, &S);
    free(cnt); free(S.acc);
    return 0;
}

int oa_assemble(OCsr *A, const OMesh *m, const OSpace *s, const OParams *p, const double *w) {
    return oa_assemble_masked(A, m, s, p, w, NULL);
}

/* ------------------------------------------------------------------------- */
/* prolongation  ("standard prolongation operator induced by the FE     */
/* discretization"; reading R-prol: (P)_IJ = N_I^fine(phi_J^coarse))           */
/* Evaluated in integer lattice units of the fine mesh (h_fine = 1, coarse     */
/* cells have edge 2) so that every entry is an exact dyadic rational.          */
/* ------------------------------------------------------------------------- */
static int cmp_ij(const void *a, const void *b) {
    const long long *x = a, *y = b;
    if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
    if (x[1] != y[1]) return x[1] < y[1] ? -1 : 1;
    return 0;
}

/* coarse parent of fine cell cf: the coarse square/cube containing it, then the
 * coarse simplex whose coordinate ordering the fine centroid satisfies (R-mesh) */
static i64 parent_cell(const OMesh *mf, const OMesh *mc, i64 cf) {
    int d = mf->dim, nvc = d + 1;
    int csum[3] = {0, 0, 0};
    for (int a = 0; a < nvc; a++)
        for (int k = 0; k < d; k++) csum[k] += mf->lat[3 * mf->cv[cf * nvc + a] + k];
    /* containing coarse square/cube: floor(centroid / 2) */
    int cc[3] = {0, 0, 0}, rel[3];
    for (int k = 0; k < d; k++) { cc[k] = csum[k] / (2 * nvc); rel[k] = csum[k] - 2 * nvc * cc[k]; }
    int Nc = mc->N;
    if (d == 2) {
        i64 s = cc[0] + (i64)Nc * cc[1];
        return rel[0] > rel[1] ? 2 * s : 2 * s + 1;
    }
    static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    i64 cube = cc[0] + (i64)Nc * (cc[1] + (i64)Nc * cc[2]);
    for (int p = 0; p < 6; p++)
        if (rel[PERM[p][0]] > rel[PERM[p][1]] && rel[PERM[p][1]] > rel[PERM[p][2]]) return 6 * cube + p;
    return -1;
}

/* the fine DoF functional N_I (R-basis) applied to an affine field F on cell K;
 * V holds the nev vertices of the DoF's entity (same units as K) */
static double dof_functional(int block, int d, int kind, int sub, const real V[3][3], int nev, const Aff *F,
                             const Cell *K) {
    real fx[3];
    if (kind == 0) { aff_eval(F, K, V[0], fx); return fx[0]; }          /* CG1: point value       */
    if (kind == 1 && d == 3) {                                            /* NED1: int_e phi.t      */
        real mid[3] = {(V[0][0] + V[1][0]) / 2, (V[0][1] + V[1][1]) / 2, (V[0][2] + V[1][2]) / 2};
        aff_eval(F, K, mid, fx);
        real t[3] = {V[1][0] - V[0][0], V[1][1] - V[0][1], V[1][2] - V[0][2]};
        return (double)dot3(fx, t);
    }
    real A[3];
    facet_area_vector(d, V, A);
    if (block == ORC_VEL) { aff_eval(F, K, V[sub], fx); return (double)dot3(fx, A); }   /* BDM: |f|(phi.n)(x_a) */
    real sacc = 0;                                                        /* RT: flux of affine field */
    for (int a = 0; a < nev; a++) { aff_eval(F, K, V[a], fx); sacc += dot3(fx, A); }
    return (double)(sacc / nev);
}

static int op_prolongation2(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc);
static int op_prolongation3(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc);

int op_prolongation(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc) {
    if (sf->degree == 2 && mf->dim == 3) return op_prolongation3(P, mf, sf, mc, sc);
    if (sf->degree == 2) return op_prolongation2(P, mf, sf, mc, sc);
    int d = mf->dim, nvc = d + 1, nle = om_nle(d);
    memset(P, 0, sizeof(*P));
    /* lowest-index fine cell containing each entity */
    int *vfirst = malloc(sizeof(int) * mf->nv), *efirst = malloc(sizeof(int) * mf->ne),
        *ffirst = malloc(sizeof(int) * mf->nfacet);
    for (i64 t = 0; t < mf->nv; t++) vfirst[t] = -1;
    for (i64 t = 0; t < mf->ne; t++) efirst[t] = -1;
    for (i64 t = 0; t < mf->nfacet; t++) ffirst[t] = -1;
    for (i64 c = 0; c < mf->nc; c++) {
        for (int a = 0; a < nvc; a++) if (vfirst[mf->cv[c * nvc + a]] < 0) vfirst[mf->cv[c * nvc + a]] = (int)c;
        for (int q = 0; q < nle; q++) if (efirst[mf->ce[c * nle + q]] < 0) efirst[mf->ce[c * nle + q]] = (int)c;
        for (int q = 0; q < nvc; q++) { int f = om_facet_of_cell(mf, c, q); if (ffirst[f] < 0) ffirst[f] = (int)c; }
    }
    i64 cap = 1024, nt = 0;
    long long *trip = malloc(sizeof(long long) * 2 * cap);
    double *tv = malloc(sizeof(double) * cap);
    for (i64 I = 0; I < sf->n; I++) {
        int kind = sf->dkind[I], ent = sf->dent[I], sub = sf->dsub[I];
        int cf = kind == 0 ? vfirst[ent] : (kind == 1 ? efirst[ent] : ffirst[ent]);
        i64 ccell = parent_cell(mf, mc, cf);
        /* coarse cell geometry in fine lattice units */
        real X[4][3] = {{0}};
        for (int a = 0; a < nvc; a++)
            for (int k = 0; k < d; k++) X[a][k] = 2 * mc->lat[3 * mc->cv[ccell * nvc + a] + k];
        Cell K;
        cell_geom_from(d, X, &K);
        /* coarse local basis functions of the same field as DoF I */
        Aff F[12];
        int gJ[12], nb = 0;
        double sgn;
        if (sf->block == ORC_VEL) {
            for (int q = 0; q <= d; q++) {
                int f0 = sc->fdof[om_facet_of_cell(mc, ccell, q)];
                for (int a = 0; a < d; a++) { F[nb] = basis_bdm(&K, q, a, &sgn); gJ[nb++] = f0 < 0 ? -1 : f0 + a; }
            }
        } else if (kind == 2) {
            for (int q = 0; q <= d; q++) { F[nb] = basis_rt(&K, q, &sgn); gJ[nb++] = sc->fdof[om_facet_of_cell(mc, ccell, q)]; }
        } else if (d == 2) {
            for (int a = 0; a < 3; a++) { F[nb] = basis_cg1(&K, a); gJ[nb++] = sc->vdof[mc->cv[ccell * 3 + a]]; }
        } else {
            for (int q = 0; q < 6; q++) {
                int lv[2];
                om_edge_local_verts(3, q, lv);
                F[nb] = basis_ned1(&K, lv[0], lv[1]);
                gJ[nb++] = sc->edof[mc->ce[ccell * 6 + q]];
            }
        }
        /* fine entity vertices (lattice) */
        real V[3][3] = {{0}};
        int nev = 0;
        if (kind == 0) { for (int k = 0; k < d; k++) V[0][k] = mf->lat[3 * ent + k]; nev = 1; }
        else if (kind == 1 || (kind == 2 && d == 2)) {
            for (int a = 0; a < 2; a++) for (int k = 0; k < d; k++) V[a][k] = mf->lat[3 * mf->ev[2 * ent + a] + k];
            nev = 2;
        } else {
            for (int a = 0; a < 3; a++) for (int k = 0; k < 3; k++) V[a][k] = mf->lat[3 * mf->fv[3 * ent + a] + k];
            nev = 3;
        }
        for (int b = 0; b < nb; b++) {
            if (gJ[b] < 0) continue;
            double val = dof_functional(sf->block, d, kind, sub, V, nev, &F[b], &K);
            if (val == 0.0) continue;
            if (nt == cap) { cap *= 2; trip = realloc(trip, sizeof(long long) * 2 * cap); tv = realloc(tv, sizeof(double) * cap); }
            trip[2 * nt] = I; trip[2 * nt + 1] = gJ[b]; tv[nt] = val; nt++;
        }
    }
    /* sort (I,J) keeping values attached */
    long long *idx = malloc(sizeof(long long) * 3 * (nt ? nt : 1));
    for (i64 t = 0; t < nt; t++) { idx[3 * t] = trip[2 * t]; idx[3 * t + 1] = trip[2 * t + 1]; idx[3 * t + 2] = t; }
    qsort(idx, (size_t)nt, 3 * sizeof(long long), cmp_ij);
    P->n = sf->n; P->nnz = nt;
    P->rp = calloc((size_t)sf->n + 1, sizeof(i64));
    P->ci = malloc(sizeof(int) * (nt ? nt : 1));
    P->v = malloc(sizeof(double) * (nt ? nt : 1));
    for (i64 t = 0; t < nt; t++) {
        P->rp[idx[3 * t] + 1]++;
        P->ci[t] = (int)idx[3 * t + 1];
        P->v[t] = tv[idx[3 * t + 2]];
    }
    for (i64 I = 0; I < sf->n; I++) P->rp[I + 1] += P->rp[I];
    free(idx); free(trip); free(tv); free(vfirst); free(efirst); free(ffirst);
    return 0;
}

int oc_transpose(OCsr *T, const OCsr *A, i64 ncols) {
    memset(T, 0, sizeof(*T));
    T->n = ncols; T->nnz = A->nnz;
    T->rp = calloc((size_t)ncols + 1, sizeof(i64));
    T->ci = malloc(sizeof(int) * (A->nnz ? A->nnz : 1));
    T->v = malloc(sizeof(double) * (A->nnz ? A->nnz : 1));
    for (i64 t = 0; t < A->nnz; t++) T->rp[A->ci[t] + 1]++;
    for (i64 j = 0; j < ncols; j++) T->rp[j + 1] += T->rp[j];
    i64 *fill = calloc((size_t)ncols, sizeof(i64));
    for (i64 i = 0; i < A->n; i++)            /* ascending rows => each T row ascending */
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) {
            int j = A->ci[t];
            i64 p = T->rp[j] + fill[j]++;
            T->ci[p] = (int)i; T->v[p] = A->v[t];
        }
    free(fill);
    return 0;
}

/* ------------------------------------------------------------------------- */
/* load vectors and field evaluation at the cell quadrature points (used only   */
/* by the manufactured-solution pins of tests/test_oracle_mms.py)               */
/* layout per point: E-B 2D [E, B1, B2]; E-B 3D [E1,E2,E3, B1,B2,B3];           */
/* velocity [u1, .., u_dim]                                                     */
/* ------------------------------------------------------------------------- */
static int local_basis(const OMesh *m, const OSpace *s, i64 c, const Cell *K, Aff *F, int *gi, int *off,
                       int *ncomp) {
    int d = m->dim, n = 0;
    double sg;
    if (s->block == ORC_VEL) {
        n = vel_basis(m, s, c, K, F, NULL, gi);
        for (int a = 0; a < n; a++) { off[a] = 0; ncomp[a] = d; }
        return n;
    }
    int nE = d == 2 ? 1 : 3;
    if (d == 2)
        for (int a = 0; a < 3; a++) { F[n] = basis_cg1(K, a); gi[n] = s->vdof[m->cv[c * 3 + a]]; off[n] = 0; ncomp[n++] = 1; }
    else
        for (int q = 0; q < 6; q++) {
            int lv[2];
            om_edge_local_verts(3, q, lv);
            F[n] = basis_ned1(K, lv[0], lv[1]); gi[n] = s->edof[m->ce[c * 6 + q]]; off[n] = 0; ncomp[n++] = 3;
        }
    for (int q = 0; q <= d; q++) {
        F[n] = basis_rt(K, q, &sg); gi[n] = s->fdof[om_facet_of_cell(m, c, q)]; off[n] = nE; ncomp[n++] = d;
    }
    return n;
}

int oa_ncomp(const OSpace *s) { return s->block == ORC_VEL ? s->dim : (s->dim == 2 ? 3 : 6); }
int oa_nq(int dim) { return dim == 2 ? 16 : 64; }

void oa_quadrature(const OMesh *m, double *pts, double *wts) {
    int nq = oa_nq(m->dim);
    real xq[64][3], wq[64];
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        cell_rule(&K, 4, xq, wq);
        for (int t = 0; t < nq; t++) {
            for (int k = 0; k < 3; k++) pts[3 * (nq * c + t) + k] = (double)xq[t][k];
            wts[nq * c + t] = (double)wq[t];
        }
    }
}

static void oa_load2(const OMesh *m, const OSpace *s, const double *fv, double *out);
static void oa_eval2(const OMesh *m, const OSpace *s, const double *coef, double *fv);
static double oa_duality_error2(const OMesh *m, const OSpace *s);
static void oa_load3(const OMesh *m, const OSpace *s, const double *fv, double *out);
static void oa_eval3(const OMesh *m, const OSpace *s, const double *coef, double *fv);
static double oa_duality_error3(const OMesh *m, const OSpace *s);

void oa_load(const OMesh *m, const OSpace *s, const double *fv, double *out) {
    if (s->degree == 2 && m->dim == 3) { oa_load3(m, s, fv, out); return; }
    if (s->degree == 2) { oa_load2(m, s, fv, out); return; }
    int nq = oa_nq(m->dim), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(out, 0, sizeof(double) * s->n);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Aff F[16];
        int gi[16], off[16], ncp[16];
        int nb = local_basis(m, s, c, &K, F, gi, off, ncp);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < nb; a++) {
            if (gi[a] < 0) continue;
            real acc = 0;
            for (int t = 0; t < nq; t++) {
                real v[3];
                aff_eval(&F[a], &K, xq[t], v);
                const double *f = fv + ((i64)c * nq + t) * nc + off[a];
                real dd = 0;
                for (int k = 0; k < ncp[a]; k++) dd += f[k] * v[k];
                acc += wq[t] * dd;
            }
            out[gi[a]] += (double)acc;
        }
    }
}

void oa_eval(const OMesh *m, const OSpace *s, const double *coef, double *fv) {
    if (s->degree == 2 && m->dim == 3) { oa_eval3(m, s, coef, fv); return; }
    if (s->degree == 2) { oa_eval2(m, s, coef, fv); return; }
    int nq = oa_nq(m->dim), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(fv, 0, sizeof(double) * m->nc * nq * nc);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Aff F[16];
        int gi[16], off[16], ncp[16];
        int nb = local_basis(m, s, c, &K, F, gi, off, ncp);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < nb; a++) {
            if (gi[a] < 0) continue;
            for (int t = 0; t < nq; t++) {
                real v[3];
                aff_eval(&F[a], &K, xq[t], v);
                double *f = fv + ((i64)c * nq + t) * nc + off[a];
                for (int k = 0; k < ncp[a]; k++) f[k] += coef[gi[a]] * (double)v[k];
            }
        }
    }
}

/* max |N_i(phi_j) - delta_ij| over the local bases of every cell of the mesh
 * (DoF duality of R-basis).  Each cell's functionals are applied to
 * that cell's own basis functions, matched through the global DoF numbering.   */
double oa_duality_error(const OMesh *m, const OSpace *s) {
    if (s->degree == 2 && m->dim == 3) return oa_duality_error3(m, s);
    if (s->degree == 2) return oa_duality_error2(m, s);
    int d = m->dim;
    double worst = 0;
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Aff F[16];
        int gi[16], off[16], ncp[16];
        int nb = local_basis(m, s, c, &K, F, gi, off, ncp);
        for (int i = 0; i < nb; i++) {
            if (gi[i] < 0) continue;
            int kind = s->dkind[gi[i]], ent = s->dent[gi[i]], sub = s->dsub[gi[i]], nev;
            real V[3][3] = {{0}};
            if (kind == 0) { for (int k = 0; k < d; k++) V[0][k] = (real)m->lat[3 * ent + k] / m->N; nev = 1; }
            else if (kind == 1 || d == 2) {
                for (int a = 0; a < 2; a++) for (int k = 0; k < d; k++) V[a][k] = (real)m->lat[3 * m->ev[2 * ent + a] + k] / m->N;
                nev = 2;
            } else {
                for (int a = 0; a < 3; a++) for (int k = 0; k < 3; k++) V[a][k] = (real)m->lat[3 * m->fv[3 * ent + a] + k] / m->N;
                nev = 3;
            }
            for (int j = 0; j < nb; j++) {
                if (gi[j] < 0 || off[j] != off[i]) continue;
                double v = dof_functional(s->block, d, kind, sub, V, nev, &F[j], &K);
                double e = fabs(v - (gi[i] == gi[j] ? 1.0 : 0.0));
                if (e > worst) worst = e;
            }
        }
    }
    return worst;
}

/* ------------------------------------------------------------------------- */
/* NEXT-3: coupling blocks of the linearised 4x4 system (Table 1   */
/* P:253-280) between the velocity space (BDM1, u), the pressure (DG0, one    */
/* indicator per cell, cell order) and the E-B spaces, on one mesh.           */
/*   Bt_{i,q} = -(q, div v_i)                    (u rows, p columns)          */
/*   J_{i,e}  = S (B^n x E_e, v_i)               (u rows, E columns)          */
/*   Dt_{i,k} = S (B_k x (u^n x B^n), v_i) + S (B^n x (u^n x B_k), v_i)       */
/*              (D~1 + D~2; J~ = S (B x E^n, v) vanishes: E^n = 0, R-coupled) */
/*   G_{e,i}  = (v_i x B^n, F_e)                 (E rows, u columns)          */
/* with u^n = w_h and B^n = curl of the B^n potential (both constant per cell,*/
/* R-w); picard (delta = 0) drops the tilde terms.  2D conventions P:38-53:   */
/* u x B = u1 B2 - u2 B1 (scalar), B x E = (B2 E, -B1 E).                     */
/* Cross-space patterns: row and column DoFs couple iff they share a cell.    */
/* ------------------------------------------------------------------------- */
static void cross_pattern(OCsr *A, i64 nrows, const OMesh *m, int (*rows_of)(const OMesh *, const void *, i64, int *),
                          const void *sx, int (*cols_of)(const OMesh *, const void *, i64, int *), const void *sy) {
    i64 *cnt = calloc((size_t)nrows + 1, sizeof(i64));
    int rl[32], cl[32];
    for (i64 c = 0; c < m->nc; c++) {
        int nr = rows_of(m, sx, c, rl), ncl = cols_of(m, sy, c, cl), k = 0;
        for (int t = 0; t < ncl; t++) k += cl[t] >= 0;
        for (int t = 0; t < nr; t++) if (rl[t] >= 0) cnt[rl[t] + 1] += k;
    }
    for (i64 r = 0; r < nrows; r++) cnt[r + 1] += cnt[r];
    int *tmp = malloc(sizeof(int) * (cnt[nrows] ? cnt[nrows] : 1));
    i64 *fill = calloc((size_t)nrows, sizeof(i64));
    for (i64 c = 0; c < m->nc; c++) {
        int nr = rows_of(m, sx, c, rl), ncl = cols_of(m, sy, c, cl);
        for (int t = 0; t < nr; t++) {
            if (rl[t] < 0) continue;
            for (int u = 0; u < ncl; u++) if (cl[u] >= 0) tmp[cnt[rl[t]] + fill[rl[t]]++] = cl[u];
        }
    }
    A->n = nrows;
    A->rp = malloc(sizeof(i64) * (nrows + 1));
    A->rp[0] = 0;
    A->ci = malloc(sizeof(int) * (cnt[nrows] ? cnt[nrows] : 1));
    i64 used = 0;
    for (i64 r = 0; r < nrows; r++) {
        int *b = tmp + cnt[r];
        i64 k = cnt[r + 1] - cnt[r];
        qsort(b, (size_t)k, sizeof(int), cmp_int);
        for (i64 t = 0; t < k; t++) if (t == 0 || b[t] != b[t - 1]) A->ci[used++] = b[t];
        A->rp[r + 1] = used;
    }
    A->nnz = used;
    A->v = calloc((size_t)(used ? used : 1), sizeof(double));
    free(tmp); free(cnt); free(fill);
}

static int vel_dofs_cb(const OMesh *m, const void *s, i64 c, int *out) { return cell_dofs(m, (const OSpace *)s, c, out); }
static int eb_E_dofs_cb(const OMesh *m, const void *s, i64 c, int *out) {
    const OSpace *sp = s;
    int tmp[16], k = cell_dofs(m, sp, c, tmp), nE = m->dim == 2 ? 3 : 6;
    for (int t = 0; t < nE; t++) out[t] = tmp[t];
    (void)k;
    return nE;
}
static int eb_B_dofs_cb(const OMesh *m, const void *s, i64 c, int *out) {
    const OSpace *sp = s;
    int tmp[16], nE = m->dim == 2 ? 3 : 6;
    cell_dofs(m, sp, c, tmp);
    for (int t = 0; t <= m->dim; t++) out[t] = tmp[nE + t] < 0 ? -1 : tmp[nE + t] - (int)sp->nE;   /* B index from 0 */
    return m->dim + 1;
}
static int cell_id_cb(const OMesh *m, const void *s, i64 c, int *out) { (void)m; (void)s; out[0] = (int)c; return 1; }

/* 2D/3D "x" conventions */
static void xcross(int d, const real *a, const real *b, real *c) {   /* vector x vector */
    if (d == 2) { c[0] = a[0] * b[1] - a[1] * b[0]; c[1] = c[2] = 0; }   /* scalar in c[0] */
    else cross3(a, b, c);
}
static void xscale(int d, const real *B, const real *s, real *c) {    /* B x (scalar or vector) */
    if (d == 2) { c[0] = B[1] * s[0]; c[1] = -B[0] * s[0]; c[2] = 0; }
    else cross3(B, s, c);
}

int oa_assemble_coupling(OCsr *Bt, OCsr *J, OCsr *Dt, OCsr *G, const OMesh *m, const OSpace *sv, const OSpace *se,
                         const OParams *p, const double *w, const double *bn, const double *floor_u,
                         const double *floor_E) {
    int d = m->dim, nE = d == 2 ? 3 : 6;
    i64 nB = se->n - se->nE;
    cross_pattern(Bt, sv->n, m, vel_dofs_cb, sv, cell_id_cb, NULL);
    cross_pattern(J, sv->n, m, vel_dofs_cb, sv, eb_E_dofs_cb, se);
    cross_pattern(Dt, sv->n, m, vel_dofs_cb, sv, eb_B_dofs_cb, se);
    cross_pattern(G, se->nE, m, eb_E_dofs_cb, se, vel_dofs_cb, sv);
    (void)nB;
    Accum SB, SJ, SD, SG;
    SB.acc = calloc((size_t)(Bt->nnz ? Bt->nnz : 1), sizeof(real));
    SJ.acc = calloc((size_t)(J->nnz ? J->nnz : 1), sizeof(real));
    SD.acc = calloc((size_t)(Dt->nnz ? Dt->nnz : 1), sizeof(real));
    SG.acc = calloc((size_t)(G->nnz ? G->nnz : 1), sizeof(real));
    real xq[64][3], wq[64];
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Aff F[12], E[6], B[4];
        double sg[12], sB;
        int gv[12], gE[6], gB[4], gc = (int)c;
        int nv = vel_basis(m, sv, c, &K, F, sg, gv);
        for (int a = 0; a < nE; a++) {
            if (d == 2) { E[a] = basis_cg1(&K, a); gE[a] = se->vdof[m->cv[c * 3 + a]]; }
            else {
                int lv[2];
                om_edge_local_verts(3, a, lv);
                E[a] = basis_ned1(&K, lv[0], lv[1]);
                gE[a] = se->edof[m->ce[c * 6 + a]];
            }
        }
        for (int q = 0; q <= d; q++) {
            B[q] = basis_rt(&K, q, &sB);
            int f = se->fdof[om_facet_of_cell(m, c, q)];
            gB[q] = f < 0 ? -1 : f - (int)se->nE;
        }
        double pot[4][3], bp[4][3];
        real wx[3], bx[3] = {0, 0, 0}, wxb[3];
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        if (bn) { cell_pot(m, c, bn, bp); cell_wind(&K, bp, bx); }
        xcross(d, wx, bx, wxb);                        /* u^n x B^n (scalar in 2D) */
        real lB[12] = {0}, lJ[12 * 6] = {0}, lD[12 * 4] = {0}, lG[6 * 12] = {0};
        int nq = cell_rule(&K, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[12][3], ev[6][3], bv[4][3];
            for (int a = 0; a < nv; a++) aff_eval(&F[a], &K, xq[t], fv[a]);
            for (int a = 0; a < nE; a++) aff_eval(&E[a], &K, xq[t], ev[a]);
            for (int q = 0; q <= d; q++) aff_eval(&B[q], &K, xq[t], bv[q]);
            for (int i = 0; i < nv; i++) {
                real dv = 0;
                for (int k = 0; k < d; k++) dv += F[i].G[k][k];
                lB[i] += wq[t] * (-dv);                                   /* -(q, div v) */
                for (int e = 0; e < nE; e++) {                            /* S (B^n x E, v) */
                    real c3[3];
                    xscale(d, bx, ev[e], c3);
                    lJ[i * 6 + e] += wq[t] * p->S * dot3(c3, fv[i]);
                    real g3[3];                                          /* (v x B^n, F) */
                    xcross(d, fv[i], bx, g3);
                    lG[e * 12 + i] += wq[t] * (d == 2 ? g3[0] * ev[e][0] : dot3(g3, ev[e]));
                }
                if (!p->picard)
                    for (int k = 0; k <= d; k++) {                        /* D~1 + D~2 */
                        real t1[3], t2[3], ub[3];
                        xscale(d, bv[k], wxb, t1);                        /* B x (u^n x B^n) */
                        xcross(d, wx, bv[k], ub);                         /* u^n x B        */
                        xscale(d, bx, ub, t2);                            /* B^n x (u^n x B) */
                        lD[i * 4 + k] += wq[t] * p->S * (dot3(t1, fv[i]) + dot3(t2, fv[i]));
                    }
            }
        }
        scatter(Bt, &SB, gv, nv, &gc, 1, lB, 1);
        scatter(J, &SJ, gv, nv, gE, nE, lJ, 6);
        scatter(Dt, &SD, gv, nv, gB, d + 1, lD, 4);
        scatter(G, &SG, gE, nE, gv, nv, lG, 12);
    }
    /* reading R-cgrid: each coupling row is rounded on the grid of the whole Newton row,
     * i.e. the grid exponent is floored by the max |entry| of the diagonal block's row */
    finish_floor(Bt, &SB, floor_u); finish_floor(J, &SJ, floor_u); finish_floor(Dt, &SD, floor_u);
    finish_floor(G, &SG, floor_E);
    free(SB.acc); free(SJ.acc); free(SD.acc); free(SG.acc);
    return 0;
}

/* ========================================================================= */
/* NEXT-2: degree k = 2 for the 2D E-B block, E in CG2, B in RT2      */
/* (the 2D complex CG2 -> RT2 -> DG1 of P:188).  Reading R-basis2:      */
/*   CG2: point values at the vertices and at the edge midpoints;              */
/*   RT2 (dim 8 = P1^2 + x P1~): per edge e = (a < b) with the global normal   */
/*     n_e of R-orient, N_{e,s}(B) = int_e (B.n_e) lambda_s ds with lambda_0 = */
/*     lambda_a, lambda_1 = lambda_b (N_{e,0} + N_{e,1} = the k = 1 flux); per */
/*     cell N_{K,r}(B) = N int_K B_r dx, r = x, y (N cells per side).          */
/* Local bases are dual to these functionals: the functionals applied to a    */
/* primal basis of the local space give a matrix that is inverted in `real`.  */
/* Every integrand is a polynomial of degree <= 4: the q = 3 cell rule and the */
/* 3-point edge rule are exact (R-quad).                                       */
/* ========================================================================= */
typedef struct { real c[2][6]; } Q2;   /* 2 components in xi = x - X0: 1, xi, eta, xi^2, xi eta, eta^2 */

static void q2_eval(const Q2 *f, const Cell *K, const real *x, real *out) {
    real a = x[0] - K->X[0][0], b = x[1] - K->X[0][1];
    real mo[6] = {1, a, b, a * a, a * b, b * b};
    for (int l = 0; l < 2; l++) {
        real s = 0;
        for (int k = 0; k < 6; k++) s += f->c[l][k] * mo[k];
        out[l] = s;
    }
    out[2] = 0;
}

static void q2_grad(const Q2 *f, const Cell *K, const real *x, real g[2][2]) {
    real a = x[0] - K->X[0][0], b = x[1] - K->X[0][1];
    for (int l = 0; l < 2; l++) {
        g[l][0] = f->c[l][1] + 2 * f->c[l][3] * a + f->c[l][4] * b;
        g[l][1] = f->c[l][2] + f->c[l][4] * a + 2 * f->c[l][5] * b;
    }
}

/* lambda_a = L[0] + L[1] xi + L[2] eta */
static void bary_lin(const Cell *K, int a, real *L) { L[0] = a == 0 ? 1 : 0; L[1] = K->g[a][0]; L[2] = K->g[a][1]; }
static real bary_at(const Cell *K, int a, const real *x) {
    real L[3];
    bary_lin(K, a, L);
    return L[0] + L[1] * (x[0] - K->X[0][0]) + L[2] * (x[1] - K->X[0][1]);
}

/* coefficients of s * A * B for linears A, B */
static void lin_mul(const real *A, const real *B, real s, real *c) {
    c[0] = s * A[0] * B[0];
    c[1] = s * (A[0] * B[1] + A[1] * B[0]);
    c[2] = s * (A[0] * B[2] + A[2] * B[0]);
    c[3] = s * A[1] * B[1];
    c[4] = s * (A[1] * B[2] + A[2] * B[1]);
    c[5] = s * A[2] * B[2];
}

/* CG2, local DoF a: a < 3 vertex a, lambda_a (2 lambda_a - 1); a = 3 + q local edge q
 * (vertices i < j), 4 lambda_i lambda_j.  Scalar in component 0. */
static Q2 basis_cg2(const Cell *K, int a) {
    Q2 f;
    memset(&f, 0, sizeof f);
    if (a < 3) {
        real L[3], L2[3];
        bary_lin(K, a, L);
        L2[0] = 2 * L[0] - 1; L2[1] = 2 * L[1]; L2[2] = 2 * L[2];
        lin_mul(L, L2, 1, f.c[0]);
    } else {
        int lv[2];
        om_edge_local_verts(2, a - 3, lv);
        real Li[3], Lj[3];
        bary_lin(K, lv[0], Li);
        bary_lin(K, lv[1], Lj);
        lin_mul(Li, Lj, 4, f.c[0]);
    }
    return f;
}

/* the 8 RT2 functionals of cell K (local order: edge q = 0..2, s = 0, 1; then r = 0, 1)
 * applied to the vector field f; Ncells = cells per side of K's mesh */
static void rt2_functionals(const Cell *K, int Ncells, const Q2 *f, real *out) {
    real xq[64][3], wq[64];
    for (int q = 0; q < 3; q++) {
        int lv[2];
        om_facet_local_verts(2, q, lv);
        real P[3][3], A[3];
        facet_points(K, q, P);
        facet_area_vector(2, P, A);
        real len = RSQRT(dot3(A, A));
        int nq = facet_rule(2, P, xq, wq);
        for (int s = 0; s < 2; s++) {
            real acc = 0;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q2_eval(f, K, xq[t], v);
                acc += wq[t] * (dot3(v, A) / len) * bary_at(K, lv[s], xq[t]);
            }
            out[2 * q + s] = acc;
        }
    }
    int nq = cell_rule(K, 3, xq, wq);
    for (int r = 0; r < 2; r++) {
        real acc = 0;
        for (int t = 0; t < nq; t++) {
            real v[3];
            q2_eval(f, K, xq[t], v);
            acc += wq[t] * v[r];
        }
        out[6 + r] = (real)Ncells * acc;
    }
}

/* Gauss-Jordan inverse with partial pivoting (n <= 20), row-major */
static int mat_inv(int n, const real *a, real *inv) {
    real w[30][60];
    for (int i = 0; i < n; i++)
        for (int j = 0; j < 2 * n; j++) w[i][j] = j < n ? a[i * n + j] : (real)(j - n == i);
    for (int k = 0; k < n; k++) {
        int p = k;
        for (int i = k + 1; i < n; i++) if (RFABS(w[i][k]) > RFABS(w[p][k])) p = i;
        if (w[p][k] == 0) return 1;
        if (p != k) for (int j = 0; j < 2 * n; j++) { real t = w[k][j]; w[k][j] = w[p][j]; w[p][j] = t; }
        real piv = w[k][k];
        for (int j = 0; j < 2 * n; j++) w[k][j] /= piv;
        for (int i = 0; i < n; i++)
            if (i != k && w[i][k] != 0) {
                real l = w[i][k];
                for (int j = 0; j < 2 * n; j++) w[i][j] -= l * w[k][j];
            }
    }
    for (int i = 0; i < n; i++) for (int j = 0; j < n; j++) inv[i * n + j] = w[i][n + j];
    return 0;
}

/* RT2 local basis dual to rt2_functionals: primal basis e_x, xi e_x, eta e_x, e_y,
 * xi e_y, eta e_y, xi (xi, eta), eta (xi, eta) */
static void basis_rt2(const Cell *K, int Ncells, Q2 *B) {
    Q2 p[8];
    memset(p, 0, sizeof p);
    p[0].c[0][0] = 1; p[1].c[0][1] = 1; p[2].c[0][2] = 1;
    p[3].c[1][0] = 1; p[4].c[1][1] = 1; p[5].c[1][2] = 1;
    p[6].c[0][3] = 1; p[6].c[1][4] = 1;
    p[7].c[0][4] = 1; p[7].c[1][5] = 1;
    real M[64], C[64], col[8];
    for (int j = 0; j < 8; j++) {
        rt2_functionals(K, Ncells, &p[j], col);
        for (int i = 0; i < 8; i++) M[i * 8 + j] = col[i];
    }
    mat_inv(8, M, C);
    for (int j = 0; j < 8; j++) {
        memset(&B[j], 0, sizeof(Q2));
        for (int k = 0; k < 8; k++)
            for (int l = 0; l < 2; l++)
                for (int t = 0; t < 6; t++) B[j].c[l][t] += C[k * 8 + j] * p[k].c[l][t];
    }
}

/* BDM2 (velocity, k = 2; reading R-basis2): per local facet q (vertices lv0 < lv1, area
 * vector A = |f| n_f of the global orientation) N_{q,s}(u) = u(x_s) . A at x_0 = X_lv0,
 * x_1 = X_lv1, x_2 = the midpoint; per cell N_{K,e}(u) = int_K u . omega_e for the Whitney
 * functions omega_e = lam_i grad lam_j - lam_j grad lam_i of the local edges e = (i < j)
 * in the order (0,1), (0,2), (1,2).  Local order: q = 0..2 x s = 0..2, then e = 0..2. */
static void whitney_at(const Cell *K, int e, const real *x, real *out) {
    int lv[2];
    om_edge_local_verts(2, e, lv);
    real li = bary_at(K, lv[0], x), lj = bary_at(K, lv[1], x);
    for (int r = 0; r < 2; r++) out[r] = li * K->g[lv[1]][r] - lj * K->g[lv[0]][r];
    out[2] = 0;
}

static void bdm2_functionals(const Cell *K, const Q2 *f, real *out) {
    for (int q = 0; q < 3; q++) {
        real P[3][3], A[3], v[3];
        facet_points(K, q, P);
        facet_area_vector(2, P, A);
        real X[3][3] = {{P[0][0], P[0][1], 0}, {P[1][0], P[1][1], 0},
                        {(P[0][0] + P[1][0]) / 2, (P[0][1] + P[1][1]) / 2, 0}};
        for (int s = 0; s < 3; s++) { q2_eval(f, K, X[s], v); out[3 * q + s] = v[0] * A[0] + v[1] * A[1]; }
    }
    real xq[64][3], wq[64];
    int nq = cell_rule(K, 3, xq, wq);
    for (int e = 0; e < 3; e++) {
        real acc = 0;
        for (int t = 0; t < nq; t++) {
            real v[3], om[3];
            q2_eval(f, K, xq[t], v);
            whitney_at(K, e, xq[t], om);
            acc += wq[t] * (v[0] * om[0] + v[1] * om[1]);
        }
        out[9 + e] = acc;
    }
}

/* BDM2 local basis dual to bdm2_functionals, from the monomial basis of P2^2 */
static void basis_bdm2(const Cell *K, Q2 *B) {
    Q2 p[12];
    memset(p, 0, sizeof p);
    for (int l = 0; l < 2; l++) for (int k = 0; k < 6; k++) p[6 * l + k].c[l][k] = 1;
    real M[144], C[144], col[12];
    for (int j = 0; j < 12; j++) {
        bdm2_functionals(K, &p[j], col);
        for (int i = 0; i < 12; i++) M[i * 12 + j] = col[i];
    }
    mat_inv(12, M, C);
    for (int j = 0; j < 12; j++) {
        memset(&B[j], 0, sizeof(Q2));
        for (int k = 0; k < 12; k++)
            for (int l = 0; l < 2; l++)
                for (int t = 0; t < 6; t++) B[j].c[l][t] += C[k * 12 + j] * p[k].c[l][t];
    }
}

static void cell_dofs_vel2(const OMesh *m, const OSpace *s, i64 c, int *g) {
    for (int q = 0; q < 3; q++) {
        int f0 = s->fdof[om_facet_of_cell(m, c, q)];
        for (int a = 0; a < 3; a++) g[3 * q + a] = f0 < 0 ? -1 : f0 + a;
    }
    for (int a = 0; a < 3; a++) g[9 + a] = s->cdof[c] + a;
}

/* AL velocity block at k = 2 (same forms as assemble_vel, R-vel):
 * cell terms (2/Re)(eps u, eps v) - (u, div(v (x) w)) + gamma (div u, div v)
 * [+ (1/dt)(u, v) + S (u x B^n, v x B^n)], facet terms SIPG (sigma from the parameters,
 * 10 k^2 = 40 at k = 2) + upwind; every integrand by quadrature (degree <= 4). */
static void assemble_vel2(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                          const unsigned char *cmask) {
    real xq[64][3], wq[64];
    const real nu2 = (real)2 / p->Re;
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Q2 F[12];
        int gi[12];
        basis_bdm2(&K, F);
        cell_dofs_vel2(m, s, c, gi);
        double pot[4][3];
        real wx[3], bx[3] = {0, 0, 0};
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        if (p->bn) { double bp[4][3]; cell_pot(m, c, p->bn, bp); cell_wind(&K, bp, bx); }
        real loc[144] = {0};
        int nq = cell_rule(&K, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[12][3], G[12][2][2], ep[12][2][2], dv[12], gw[12][2];
            for (int a = 0; a < 12; a++) {
                q2_eval(&F[a], &K, xq[t], fv[a]);
                q2_grad(&F[a], &K, xq[t], G[a]);
                for (int l = 0; l < 2; l++) for (int k = 0; k < 2; k++) ep[a][l][k] = (G[a][l][k] + G[a][k][l]) / 2;
                dv[a] = G[a][0][0] + G[a][1][1];
                for (int l = 0; l < 2; l++) gw[a][l] = G[a][l][0] * wx[0] + G[a][l][1] * wx[1];
            }
            for (int i = 0; i < 12; i++)
                for (int j = 0; j < 12; j++) {
                    real ee = 0;
                    for (int l = 0; l < 2; l++) for (int k = 0; k < 2; k++) ee += ep[j][l][k] * ep[i][l][k];
                    real v = nu2 * ee - (fv[j][0] * gw[i][0] + fv[j][1] * gw[i][1]) + (real)p->gamma * dv[j] * dv[i];
                    if (p->dt > 0) v += (fv[j][0] * fv[i][0] + fv[j][1] * fv[i][1]) / p->dt;
                    if (p->bn)
                        v += p->S * (fv[j][0] * bx[1] - fv[j][1] * bx[0]) * (fv[i][0] * bx[1] - fv[i][1] * bx[0]);
                    loc[i * 12 + j] += wq[t] * v;
                }
        }
        scatter(A, S, gi, 12, gi, 12, loc, 12);
    }
    static real floc[24 * 24];
    for (i64 f = 0; f < m->nfacet; f++) {
        int cp = m->fcell[2 * f], cm = m->fcell[2 * f + 1];
        if (cmask && !cmask[cp] && !(cm >= 0 && cmask[cm])) continue;
        int interior = cm >= 0, nb = 12;
        Cell Kp, Km;
        Q2 F[24];
        int gi[24], side[24];
        cell_geom(m, cp, &Kp);
        basis_bdm2(&Kp, F);
        cell_dofs_vel2(m, s, cp, gi);
        for (int a = 0; a < 12; a++) side[a] = +1;
        if (interior) {
            cell_geom(m, cm, &Km);
            basis_bdm2(&Km, F + 12);
            cell_dofs_vel2(m, s, cm, gi + 12);
            for (int a = 12; a < 24; a++) side[a] = -1;
            nb = 24;
        }
        int qf = -1;
        for (int q = 0; q < 3; q++) if (om_facet_of_cell(m, cp, q) == f) qf = q;
        real P[3][3], Av[3];
        facet_points(&Kp, qf, P);
        facet_area_vector(2, P, Av);
        real an = RSQRT(dot3(Av, Av)), n[3];
        double sgn = facet_sign(&Kp, qf, Av);
        for (int k = 0; k < 3; k++) n[k] = sgn * Av[k] / an;
        real avg = interior ? (real)1 / 2 : (real)1;
        real pen = (real)p->sigma / ((real)p->Re * an);
        double pot[4][3];
        real wx[3];
        cell_pot(m, cp, w, pot);
        cell_wind(&Kp, pot, wx);
        real wn = dot3(wx, n), awn = RFABS(wn);
        memset(floc, 0, sizeof(floc));
        int nq = facet_rule(2, P, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[24][3], en[24][2];
            for (int a = 0; a < nb; a++) {
                const Cell *Ka = side[a] > 0 ? &Kp : &Km;
                real G[2][2];
                q2_eval(&F[a], Ka, xq[t], fv[a]);
                q2_grad(&F[a], Ka, xq[t], G);
                for (int l = 0; l < 2; l++)
                    en[a][l] = (G[l][0] + G[0][l]) / 2 * n[0] + (G[l][1] + G[1][l]) / 2 * n[1];
            }
            for (int i = 0; i < nb; i++) {
                real Ji = side[i];
                for (int j = 0; j < nb; j++) {
                    real Jj = side[j];
                    real vv = fv[j][0] * fv[i][0] + fv[j][1] * fv[i][1];
                    real t1 = -nu2 * avg * (en[j][0] * fv[i][0] + en[j][1] * fv[i][1]) * Ji;
                    real t2 = -nu2 * avg * (fv[j][0] * en[i][0] + fv[j][1] * en[i][1]) * Jj;
                    real t3 = pen * Jj * Ji * vv;
                    real up;
                    if (interior) up = (side[j] > 0 ? (wn + awn) / 2 : -(-wn + awn) / 2) * vv * Ji;
                    else up = (wn + awn) / 2 * vv;
                    floc[i * 24 + j] += wq[t] * (t1 + t2 + t3 + up);
                }
            }
        }
        scatter(A, S, gi, nb, gi, nb, floc, 24);
    }
}

/* global free DoFs of the CG2 and RT2 local bases of cell c */
static void cell_dofs2(const OMesh *m, const OSpace *s, i64 c, int *gE, int *gB) {
    for (int a = 0; a < 3; a++) gE[a] = s->vdof[m->cv[c * 3 + a]];
    for (int q = 0; q < 3; q++) gE[3 + q] = s->edof[m->ce[c * 3 + q]];
    for (int q = 0; q < 3; q++) {
        int f0 = s->fdof[om_facet_of_cell(m, c, q)];
        gB[2 * q] = f0 < 0 ? -1 : f0;
        gB[2 * q + 1] = f0 < 0 ? -1 : f0 + 1;
    }
    gB[6] = s->cdof[c]; gB[7] = s->cdof[c] + 1;
}

/* E-B block at k = 2 (same forms as assemble_eb):
 *   E rows: (E, F) - (1/Rem)(B, vcurl F) + delta (u^n x B, F)
 *   B rows: (eta/dt)(B, C) + (vcurl E, C) + (1/Rem)(div B, div C)                 */
static void assemble_eb2(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                         const unsigned char *cmask) {
    real xq[64][3], wq[64];
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Q2 E[6], B[8];
        int gE[6], gB[8];
        for (int a = 0; a < 6; a++) E[a] = basis_cg2(&K, a);
        basis_rt2(&K, m->N, B);
        cell_dofs2(m, s, c, gE, gB);
        double pot[4][3];
        real wx[3];
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        real EE[36] = {0}, EB[48] = {0}, BE[48] = {0}, BB[64] = {0};
        int nq = cell_rule(&K, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real ev[6][3], curlE[6][2], bv[8][3], divB[8];
            for (int a = 0; a < 6; a++) {
                real g[2][2];
                q2_eval(&E[a], &K, xq[t], ev[a]);
                q2_grad(&E[a], &K, xq[t], g);
                curlE[a][0] = g[0][1]; curlE[a][1] = -g[0][0];
            }
            for (int k = 0; k < 8; k++) {
                real g[2][2];
                q2_eval(&B[k], &K, xq[t], bv[k]);
                q2_grad(&B[k], &K, xq[t], g);
                divB[k] = g[0][0] + g[1][1];
            }
            for (int i = 0; i < 6; i++) {
                for (int j = 0; j < 6; j++) EE[i * 6 + j] += wq[t] * ev[j][0] * ev[i][0];
                for (int k = 0; k < 8; k++) {
                    real wxb = p->picard ? 0 : (wx[0] * bv[k][1] - wx[1] * bv[k][0]) * ev[i][0];
                    real ab = bv[k][0] * curlE[i][0] + bv[k][1] * curlE[i][1];
                    EB[i * 8 + k] += wq[t] * (wxb - ab / p->Rem);
                    BE[k * 6 + i] += wq[t] * ab;
                }
            }
            for (int k = 0; k < 8; k++)
                for (int l = 0; l < 8; l++) {
                    real v = divB[l] * divB[k] / p->Rem;
                    if (p->dt > 0) v += (bv[l][0] * bv[k][0] + bv[l][1] * bv[k][1]) / p->dt;
                    BB[k * 8 + l] += wq[t] * v;
                }
        }
        scatter(A, S, gE, 6, gE, 6, EE, 6);
        scatter(A, S, gE, 6, gB, 8, EB, 8);
        scatter(A, S, gB, 8, gE, 6, BE, 6);
        scatter(A, S, gB, 8, gB, 8, BB, 8);
    }
}

/* the fine functional of free DoF I (k = 2) applied to the coarse local basis function F
 * living on coarse cell Kc; physical coordinates */
static real dof_functional2(const OMesh *mf, const OSpace *sf, i64 I, const Q2 *F, const Cell *Kc) {
    int kind = sf->dkind[I], ent = sf->dent[I], sub = sf->dsub[I];
    real v[3];
    if (sf->block == ORC_VEL) {                 /* BDM2 functionals of the fine mesh */
        if (kind == 2) {
            real P[3][3] = {{0}}, A[3];
            for (int a = 0; a < 2; a++)
                for (int k = 0; k < 2; k++) P[a][k] = (real)mf->lat[3 * mf->ev[2 * ent + a] + k] / mf->N;
            facet_area_vector(2, P, A);
            real x[3] = {sub == 2 ? (P[0][0] + P[1][0]) / 2 : P[sub][0], sub == 2 ? (P[0][1] + P[1][1]) / 2 : P[sub][1], 0};
            q2_eval(F, Kc, x, v);
            return v[0] * A[0] + v[1] * A[1];
        }
        Cell Kf;
        cell_geom(mf, ent, &Kf);
        real xq[64][3], wq[64], acc = 0;
        int nq = cell_rule(&Kf, 3, xq, wq);
        for (int t = 0; t < nq; t++) {
            real om[3];
            q2_eval(F, Kc, xq[t], v);
            whitney_at(&Kf, sub, xq[t], om);
            acc += wq[t] * (v[0] * om[0] + v[1] * om[1]);
        }
        return acc;
    }
    if (kind == 0) {
        real x[3] = {(real)mf->lat[3 * ent] / mf->N, (real)mf->lat[3 * ent + 1] / mf->N, 0};
        q2_eval(F, Kc, x, v);
        return v[0];
    }
    real P[3][3] = {{0}};
    if (kind <= 2)
        for (int a = 0; a < 2; a++)
            for (int k = 0; k < 2; k++) P[a][k] = (real)mf->lat[3 * mf->ev[2 * ent + a] + k] / mf->N;
    if (kind == 1) {
        real x[3] = {(P[0][0] + P[1][0]) / 2, (P[0][1] + P[1][1]) / 2, 0};
        q2_eval(F, Kc, x, v);
        return v[0];
    }
    real xq[64][3], wq[64];
    if (kind == 2) {
        real A[3];
        facet_area_vector(2, P, A);
        real len = RSQRT(dot3(A, A));
        real t[3] = {P[1][0] - P[0][0], P[1][1] - P[0][1], 0};
        int nq = facet_rule(2, P, xq, wq);
        real acc = 0;
        for (int q = 0; q < nq; q++) {
            q2_eval(F, Kc, xq[q], v);
            real d[3] = {xq[q][0] - P[0][0], xq[q][1] - P[0][1], 0};
            real lam1 = dot3(d, t) / dot3(t, t);
            acc += wq[q] * (dot3(v, A) / len) * (sub == 0 ? 1 - lam1 : lam1);
        }
        return acc;
    }
    Cell Kf;
    cell_geom(mf, ent, &Kf);
    int nq = cell_rule(&Kf, 3, xq, wq);
    real acc = 0;
    for (int q = 0; q < nq; q++) {
        q2_eval(F, Kc, xq[q], v);
        acc += wq[q] * v[sub];
    }
    return (real)mf->N * acc;
}

/* R-prol at k = 2: P_IJ = N_I^fine(phi_J^coarse), evaluated on the parent coarse cell of
 * a fine cell containing DoF I's entity, in `real`; each row rounded as in R-exact. */
static int op_prolongation2(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc) {
    memset(P, 0, sizeof(*P));
    int *vfirst = malloc(sizeof(int) * mf->nv), *efirst = malloc(sizeof(int) * mf->ne);
    for (i64 t = 0; t < mf->nv; t++) vfirst[t] = -1;
    for (i64 t = 0; t < mf->ne; t++) efirst[t] = -1;
    for (i64 c = 0; c < mf->nc; c++) {
        for (int a = 0; a < 3; a++) if (vfirst[mf->cv[c * 3 + a]] < 0) vfirst[mf->cv[c * 3 + a]] = (int)c;
        for (int q = 0; q < 3; q++) if (efirst[mf->ce[c * 3 + q]] < 0) efirst[mf->ce[c * 3 + q]] = (int)c;
    }
    i64 cap = 1024, nt = 0;
    long long *idx = malloc(sizeof(long long) * 3 * cap);
    real *tv = malloc(sizeof(real) * cap);
    for (i64 I = 0; I < sf->n; I++) {
        int kind = sf->dkind[I], ent = sf->dent[I];
        int cf = kind == 0 ? vfirst[ent] : (kind == 3 ? ent : efirst[ent]);
        i64 ccell = parent_cell(mf, mc, cf);
        Cell Kc;
        cell_geom(mc, ccell, &Kc);
        Q2 F[12];
        int gE[6], gB[8], gV[12], nb;
        const int *gJ;
        if (sf->block == ORC_VEL) { basis_bdm2(&Kc, F); cell_dofs_vel2(mc, sc, ccell, gV); nb = 12; gJ = gV; }
        else {
            cell_dofs2(mc, sc, ccell, gE, gB);
            if (kind <= 1) { for (int a = 0; a < 6; a++) F[a] = basis_cg2(&Kc, a); nb = 6; gJ = gE; }
            else { basis_rt2(&Kc, mc->N, F); nb = 8; gJ = gB; }
        }
        for (int b = 0; b < nb; b++) {
            if (gJ[b] < 0) continue;
            real val = dof_functional2(mf, sf, I, &F[b], &Kc);
            if (nt == cap) { cap *= 2; idx = realloc(idx, sizeof(long long) * 3 * cap); tv = realloc(tv, sizeof(real) * cap); }
            idx[3 * nt] = I; idx[3 * nt + 1] = gJ[b]; idx[3 * nt + 2] = nt; tv[nt] = val; nt++;
        }
    }
    qsort(idx, (size_t)nt, 3 * sizeof(long long), cmp_ij);
    /* row rounding (R-exact grid); zeros dropped.  Reading R-prol2: the exact entries are
     * rationals with small denominators, so |x| < 2^-30 max|row| can only be the residue
     * of an exact cancellation (it is 0 exactly; the fp64 build cannot reach the grid). */
    P->n = sf->n;
    P->rp = calloc((size_t)sf->n + 1, sizeof(i64));
    P->ci = malloc(sizeof(int) * (nt ? nt : 1));
    P->v = malloc(sizeof(double) * (nt ? nt : 1));
    i64 used = 0;
    for (i64 t0 = 0; t0 < nt;) {
        i64 t1 = t0;
        while (t1 < nt && idx[3 * t1] == idx[3 * t0]) t1++;
        double mx = 0;
        for (i64 t = t0; t < t1; t++) { double h = (double)tv[idx[3 * t + 2]]; if (fabs(h) > mx) mx = fabs(h); }
        int E = 0;
        if (mx > 0) frexp(mx, &E);
        for (i64 t = t0; t < t1; t++) {
            real x = tv[idx[3 * t + 2]];
            double h = (double)x, l = (double)(x - (real)h);
            double v = (mx > 0 && fabs(h) >= ldexp(mx, -30)) ? grid_round(h, l, E) : 0.0;
            if (v == 0.0) continue;
            P->ci[used] = (int)idx[3 * t + 1];
            P->v[used] = v;
            used++;
            P->rp[idx[3 * t] + 1]++;
        }
        t0 = t1;
    }
    for (i64 i = 0; i < sf->n; i++) P->rp[i + 1] += P->rp[i];
    P->nnz = used;
    free(idx); free(tv); free(vfirst); free(efirst);
    return 0;
}

/* k = 2 local basis for the MMS helpers: E (component 0 of the E-B field triple) then B */
static int local_basis2(const OMesh *m, const OSpace *s, i64 c, const Cell *K, Q2 *F, int *gi, int *off, int *ncp) {
    if (s->block == ORC_VEL) {
        basis_bdm2(K, F);
        cell_dofs_vel2(m, s, c, gi);
        for (int a = 0; a < 12; a++) { off[a] = 0; ncp[a] = 2; }
        return 12;
    }
    int gE[6], gB[8];
    cell_dofs2(m, s, c, gE, gB);
    for (int a = 0; a < 6; a++) { F[a] = basis_cg2(K, a); gi[a] = gE[a]; off[a] = 0; ncp[a] = 1; }
    basis_rt2(K, m->N, F + 6);
    for (int k = 0; k < 8; k++) { gi[6 + k] = gB[k]; off[6 + k] = 1; ncp[6 + k] = 2; }
    return 14;
}

static void oa_load2(const OMesh *m, const OSpace *s, const double *fv, double *out) {
    int nq = oa_nq(2), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(out, 0, sizeof(double) * s->n);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q2 F[14];
        int gi[14], off[14], ncp[14];
        int nb = local_basis2(m, s, c, &K, F, gi, off, ncp);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < nb; a++) {
            if (gi[a] < 0) continue;
            real acc = 0;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q2_eval(&F[a], &K, xq[t], v);
                const double *f = fv + ((i64)c * nq + t) * nc + off[a];
                real d = 0;
                for (int k = 0; k < ncp[a]; k++) d += f[k] * v[k];
                acc += wq[t] * d;
            }
            out[gi[a]] += (double)acc;
        }
    }
}

static void oa_eval2(const OMesh *m, const OSpace *s, const double *coef, double *fv) {
    int nq = oa_nq(2), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(fv, 0, sizeof(double) * m->nc * nq * nc);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q2 F[14];
        int gi[14], off[14], ncp[14];
        int nb = local_basis2(m, s, c, &K, F, gi, off, ncp);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < nb; a++) {
            if (gi[a] < 0) continue;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q2_eval(&F[a], &K, xq[t], v);
                double *f = fv + ((i64)c * nq + t) * nc + off[a];
                for (int k = 0; k < ncp[a]; k++) f[k] += coef[gi[a]] * (double)v[k];
            }
        }
    }
}

/* duality N_i(phi_j) = delta_ij at k = 2: the global fine functionals (dof_functional2,
 * written independently of rt2_functionals) applied to each cell's local basis */
static double oa_duality_error2(const OMesh *m, const OSpace *s) {
    double worst = 0;
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q2 F[14];
        int gi[14], off[14], ncp[14];
        int nb = local_basis2(m, s, c, &K, F, gi, off, ncp);
        for (int i = 0; i < nb; i++) {
            if (gi[i] < 0) continue;
            for (int j = 0; j < nb; j++) {
                if (gi[j] < 0 || off[j] != off[i]) continue;
                double v = (double)dof_functional2(m, s, gi[i], &F[j], &K);
                double e = fabs(v - (gi[i] == gi[j] ? 1.0 : 0.0));
                if (e > worst) worst = e;
            }
        }
    }
    return worst;
}

/* ========================================================================= */
/* NEXT-2 in 3D: degree k = 2 for the E-B block, E in NED1_2, B in RT2 (*/
/* P:654; complex CG2 -> NED1_2 -> RT2 -> DG1).  Reading R-basis2-3D:   */
/*   NED1_2 (dim 20): per edge e = (a < b), t_e = x_b - x_a,                  */
/*     N_{e,s}(E) = int_e (E . t_e / |e|) lambda_s ds (lambda_0 = lambda_a,    */
/*     lambda_1 = lambda_b); per face f = (a < b < c), t_0 = x_b - x_a,        */
/*     t_1 = x_c - x_a, N_{f,s}(E) = N int_f E . t_s dA;                       */
/*   RT2 (dim 15): per face f, unit normal n_f of R-orient,                   */
/*     N_{f,s}(B) = int_f (B . n_f) lambda_{v_s} dA; per cell N int_K B_r dx.  */
/* Local bases dual to these functionals (primal bases inverted in `real`).    */
/* ========================================================================= */
typedef struct { real c[3][10]; } Q3;   /* 3 components in xi - X0: 1,x,y,z,xx,xy,xz,yy,yz,zz */

static void q3_mono(const Cell *K, const real *x, real *mo) {
    real a = x[0] - K->X[0][0], b = x[1] - K->X[0][1], c = x[2] - K->X[0][2];
    mo[0] = 1; mo[1] = a; mo[2] = b; mo[3] = c; mo[4] = a * a; mo[5] = a * b; mo[6] = a * c;
    mo[7] = b * b; mo[8] = b * c; mo[9] = c * c;
}
static void q3_eval(const Q3 *f, const Cell *K, const real *x, real *out) {
    real mo[10];
    q3_mono(K, x, mo);
    for (int l = 0; l < 3; l++) { real s = 0; for (int k = 0; k < 10; k++) s += f->c[l][k] * mo[k]; out[l] = s; }
}
/* g[l][k] = d_k f_l */
static void q3_grad(const Q3 *f, const Cell *K, const real *x, real g[3][3]) {
    real a = x[0] - K->X[0][0], b = x[1] - K->X[0][1], c = x[2] - K->X[0][2];
    for (int l = 0; l < 3; l++) {
        const real *q = f->c[l];
        g[l][0] = q[1] + 2 * q[4] * a + q[5] * b + q[6] * c;
        g[l][1] = q[2] + q[5] * a + 2 * q[7] * b + q[8] * c;
        g[l][2] = q[3] + q[6] * a + q[8] * b + 2 * q[9] * c;
    }
}
static real bary3_at(const Cell *K, int a, const real *x) {
    real s = a == 0 ? 1 : 0;
    for (int k = 0; k < 3; k++) s += K->g[a][k] * (x[k] - K->X[0][k]);
    return s;
}

/* the 20 NED1_2 functionals of cell K (local order: edge q = 0..5 x s = 0,1; face q = 0..3 x s) */
static void ned2_functionals(const Cell *K, int Ncells, const Q3 *f, real *out) {
    real g[3], w[3];
    gauss01(3, g, w);
    for (int q = 0; q < 6; q++) {
        int lv[2];
        om_edge_local_verts(3, q, lv);
        real t[3], len2 = 0;
        for (int k = 0; k < 3; k++) { t[k] = K->X[lv[1]][k] - K->X[lv[0]][k]; len2 += t[k] * t[k]; }
        real len = RSQRT(len2);
        for (int s = 0; s < 2; s++) {
            real acc = 0;
            for (int i = 0; i < 3; i++) {
                real x[3], v[3];
                for (int k = 0; k < 3; k++) x[k] = K->X[lv[0]][k] + g[i] * t[k];
                q3_eval(f, K, x, v);
                real lam = s == 0 ? 1 - g[i] : g[i];
                acc += w[i] * len * (dot3(v, t) / len) * lam;
            }
            out[2 * q + s] = acc;
        }
    }
    real xq[64][3], wq[64];
    for (int q = 0; q < 4; q++) {
        int lv[3];
        om_facet_local_verts(3, q, lv);
        real P[3][3];
        facet_points(K, q, P);
        int nq = facet_rule(3, P, xq, wq);
        for (int s = 0; s < 2; s++) {
            real t[3];
            for (int k = 0; k < 3; k++) t[k] = P[s + 1][k] - P[0][k];
            real acc = 0;
            for (int i = 0; i < nq; i++) { real v[3]; q3_eval(f, K, xq[i], v); acc += wq[i] * dot3(v, t); }
            out[12 + 2 * q + s] = (real)Ncells * acc;
        }
    }
}

/* the 15 RT2 functionals of cell K in 3D (local order: face q = 0..3 x s = 0..2, then r) */
static void rt2_3d_functionals(const Cell *K, int Ncells, const Q3 *f, real *out) {
    real xq[64][3], wq[64];
    for (int q = 0; q < 4; q++) {
        int lv[3];
        om_facet_local_verts(3, q, lv);
        real P[3][3], A[3];
        facet_points(K, q, P);
        facet_area_vector(3, P, A);
        real area = RSQRT(dot3(A, A));
        int nq = facet_rule(3, P, xq, wq);
        for (int s = 0; s < 3; s++) {
            real acc = 0;
            for (int i = 0; i < nq; i++) {
                real v[3];
                q3_eval(f, K, xq[i], v);
                acc += wq[i] * (dot3(v, A) / area) * bary3_at(K, lv[s], xq[i]);
            }
            out[3 * q + s] = acc;
        }
    }
    int nq = cell_rule(K, 3, xq, wq);
    for (int r = 0; r < 3; r++) {
        real acc = 0;
        for (int i = 0; i < nq; i++) { real v[3]; q3_eval(f, K, xq[i], v); acc += wq[i] * v[r]; }
        out[12 + r] = (real)Ncells * acc;
    }
}

static int q3_pair(int i, int j) {            /* monomial index of xi_i xi_j */
    static const int M[3][3] = {{4, 5, 6}, {5, 7, 8}, {6, 8, 9}};
    return M[i][j];
}

/* primal bases: P1^3 (12), then RT2: xi_s x (3); NED1_2: xi_s (x cross e_r), s != r (6),
 * and the diagonal combinations xi_0 (x x e_0) - xi_1 (x x e_1), xi_1 (x x e_1) - xi_2 (x x e_2) */
static int primal3(int ned, Q3 *p) {
    int n = 0;
    memset(p, 0, sizeof(Q3) * 20);
    for (int r = 0; r < 3; r++)
        for (int k = 0; k < 4; k++) p[n++].c[r][k] = 1;
    if (!ned) {
        for (int s = 0; s < 3; s++) { for (int l = 0; l < 3; l++) p[n].c[l][q3_pair(s, l)] = 1; n++; }
        return n;
    }
    /* x cross e_r: r = 0: (0, z, -y); r = 1: (-z, 0, x); r = 2: (y, -x, 0) */
    static const int XC[3][3][2] = {{{-1, 0}, {2, 1}, {1, -1}}, {{2, -1}, {-1, 0}, {0, 1}}, {{1, 1}, {0, -1}, {-1, 0}}};
    Q3 F[3][3];
    memset(F, 0, sizeof F);
    for (int s = 0; s < 3; s++)
        for (int r = 0; r < 3; r++)
            for (int l = 0; l < 3; l++)
                if (XC[r][l][0] >= 0) F[s][r].c[l][q3_pair(s, XC[r][l][0])] = XC[r][l][1];
    for (int s = 0; s < 3; s++)
        for (int r = 0; r < 3; r++)
            if (s != r) p[n++] = F[s][r];
    for (int l = 0; l < 3; l++)
        for (int k = 0; k < 10; k++) {
            p[n].c[l][k] = F[0][0].c[l][k] - F[1][1].c[l][k];
            p[n + 1].c[l][k] = F[1][1].c[l][k] - F[2][2].c[l][k];
        }
    n += 2;
    return n;
}

static void basis3(const Cell *K, int Ncells, int ned, Q3 *B) {
    Q3 p[20];
    int n = primal3(ned, p);
    real M[400], C[400], col[20];
    for (int j = 0; j < n; j++) {
        if (ned) ned2_functionals(K, Ncells, &p[j], col); else rt2_3d_functionals(K, Ncells, &p[j], col);
        for (int i = 0; i < n; i++) M[i * n + j] = col[i];
    }
    mat_inv(n, M, C);
    for (int j = 0; j < n; j++) {
        memset(&B[j], 0, sizeof(Q3));
        for (int k = 0; k < n; k++)
            for (int l = 0; l < 3; l++)
                for (int t = 0; t < 10; t++) B[j].c[l][t] += C[k * n + j] * p[k].c[l][t];
    }
}

static void cell_dofs3(const OMesh *m, const OSpace *s, i64 c, int *gE, int *gB) {
    int all[35];
    cell_dofs(m, s, c, all);
    for (int a = 0; a < 20; a++) gE[a] = all[a];
    for (int a = 0; a < 15; a++) gB[a] = all[20 + a];
}

static void assemble_eb2_3d(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                            const unsigned char *cmask) {
    real xq[64][3], wq[64];
    static real EE[400], EB[300], BE[300], BB[225];
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Q3 E[20], B[15];
        int gE[20], gB[15];
        basis3(&K, m->N, 1, E);
        basis3(&K, m->N, 0, B);
        cell_dofs3(m, s, c, gE, gB);
        double pot[4][3];
        real wx[3];
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        memset(EE, 0, sizeof EE); memset(EB, 0, sizeof EB); memset(BE, 0, sizeof BE); memset(BB, 0, sizeof BB);
        /* q = 4: the collapsed Gauss rule gains degree from its Jacobian ((1-eta)(1-zeta)^2 in
         * 3D), so 3 points are exact only to degree 3 there; the k = 2 mass and u^n x B
         * integrands have degree 4 (q = 4: exact to degree 5) */
        int nq = cell_rule(&K, 4, xq, wq);
        for (int t = 0; t < nq; t++) {
            real ev[20][3], ce[20][3], bv[15][3], db[15];
            for (int a = 0; a < 20; a++) {
                real g[3][3];
                q3_eval(&E[a], &K, xq[t], ev[a]);
                q3_grad(&E[a], &K, xq[t], g);
                ce[a][0] = g[2][1] - g[1][2]; ce[a][1] = g[0][2] - g[2][0]; ce[a][2] = g[1][0] - g[0][1];
            }
            for (int k = 0; k < 15; k++) {
                real g[3][3];
                q3_eval(&B[k], &K, xq[t], bv[k]);
                q3_grad(&B[k], &K, xq[t], g);
                db[k] = g[0][0] + g[1][1] + g[2][2];
            }
            for (int i = 0; i < 20; i++) {
                for (int j = 0; j < 20; j++) EE[i * 20 + j] += wq[t] * dot3(ev[j], ev[i]);
                for (int k = 0; k < 15; k++) {
                    real wxb = 0;
                    if (!p->picard) { real cr[3]; cross3(wx, bv[k], cr); wxb = dot3(cr, ev[i]); }
                    real ab = dot3(bv[k], ce[i]);
                    EB[i * 15 + k] += wq[t] * (wxb - ab / p->Rem);
                    BE[k * 20 + i] += wq[t] * ab;
                }
            }
            for (int k = 0; k < 15; k++)
                for (int l = 0; l < 15; l++) {
                    real v = db[l] * db[k] / p->Rem;
                    if (p->dt > 0) v += dot3(bv[l], bv[k]) / p->dt;
                    BB[k * 15 + l] += wq[t] * v;
                }
        }
        scatter(A, S, gE, 20, gE, 20, EE, 20);
        scatter(A, S, gE, 20, gB, 15, EB, 15);
        scatter(A, S, gB, 15, gE, 20, BE, 20);
        scatter(A, S, gB, 15, gB, 15, BB, 15);
    }
}

/* local index in cell K (of mesh m, cell c) of global vertex v */
static int local_vertex(const OMesh *m, i64 c, int v) {
    for (int a = 0; a < 4; a++) if (m->cv[c * 4 + a] == v) return a;
    return -1;
}

/* the fine functional of free DoF I (3D k = 2) applied to F living on coarse cell Kc;
 * owner = a fine cell containing the DoF's entity */
static real dof_functional3(const OMesh *mf, const OSpace *sf, i64 I, const Q3 *F, const Cell *Kc, i64 owner) {
    int kind = sf->dkind[I], ent = sf->dent[I], sub = sf->dsub[I];
    real v[3], xq[64][3], wq[64];
    if (kind == 1) {
        real P0[3], t[3], len2 = 0, g[3], w[3];
        for (int k = 0; k < 3; k++) {
            P0[k] = (real)mf->lat[3 * mf->ev[2 * ent] + k] / mf->N;
            t[k] = (real)mf->lat[3 * mf->ev[2 * ent + 1] + k] / mf->N - P0[k];
            len2 += t[k] * t[k];
        }
        real len = RSQRT(len2), acc = 0;
        gauss01(3, g, w);
        for (int i = 0; i < 3; i++) {
            real x[3];
            for (int k = 0; k < 3; k++) x[k] = P0[k] + g[i] * t[k];
            q3_eval(F, Kc, x, v);
            acc += w[i] * len * (dot3(v, t) / len) * (sub == 0 ? 1 - g[i] : g[i]);
        }
        return acc;
    }
    if (kind == 3) {
        Cell Kf;
        cell_geom(mf, ent, &Kf);
        int nq = cell_rule(&Kf, 3, xq, wq);
        real acc = 0;
        for (int i = 0; i < nq; i++) { q3_eval(F, Kc, xq[i], v); acc += wq[i] * v[sub]; }
        return (real)mf->N * acc;
    }
    real P[3][3];
    for (int a = 0; a < 3; a++)
        for (int k = 0; k < 3; k++) P[a][k] = (real)mf->lat[3 * mf->fv[3 * ent + a] + k] / mf->N;
    int nq = facet_rule(3, P, xq, wq);
    real acc = 0;
    if (kind == 4) {
        real t[3];
        for (int k = 0; k < 3; k++) t[k] = P[sub + 1][k] - P[0][k];
        for (int i = 0; i < nq; i++) { q3_eval(F, Kc, xq[i], v); acc += wq[i] * dot3(v, t); }
        return (real)mf->N * acc;
    }
    real A[3];
    facet_area_vector(3, P, A);
    real area = RSQRT(dot3(A, A));
    Cell Kf;
    cell_geom(mf, owner, &Kf);
    int la = local_vertex(mf, owner, mf->fv[3 * ent + sub]);
    for (int i = 0; i < nq; i++) {
        q3_eval(F, Kc, xq[i], v);
        acc += wq[i] * (dot3(v, A) / area) * bary3_at(&Kf, la, xq[i]);
    }
    return acc;
}

/* ========================================================================= */
/* NEXT-2 in 3D, AL velocity block: BDM2.  Reading            */
/* R-basis2-vel in 3D: per face f (vertices a < b < c, area vector A = |f| n_f */
/* of R-orient) N_{f,s}(u) = u(x_s) . A at x_0..2 = x_a, x_b, x_c, x_3 = mid(a,b),*/
/* x_4 = mid(a,c), x_5 = mid(b,c) (the P2 nodes of the face); per cell         */
/* N_{K,e}(u) = int_K u . (lam_i grad lam_j - lam_j grad lam_i) for the 6 edges */
/* e = (i < j) in the local order (0,1) (0,2) (0,3) (1,2) (1,3) (2,3).  Local  */
/* basis dual to these, from the monomial basis of P2^3 (inverted in `real`).  */
/* ========================================================================= */
static void face_nodes(const real P[3][3], real X[6][3]) {
    for (int k = 0; k < 3; k++) {
        X[0][k] = P[0][k]; X[1][k] = P[1][k]; X[2][k] = P[2][k];
        X[3][k] = (P[0][k] + P[1][k]) / 2; X[4][k] = (P[0][k] + P[2][k]) / 2; X[5][k] = (P[1][k] + P[2][k]) / 2;
    }
}

static void whitney3_at(const Cell *K, int e, const real *x, real *out) {
    int lv[2];
    om_edge_local_verts(3, e, lv);
    real li = bary3_at(K, lv[0], x), lj = bary3_at(K, lv[1], x);
    for (int r = 0; r < 3; r++) out[r] = li * K->g[lv[1]][r] - lj * K->g[lv[0]][r];
}

/* the 30 BDM2 functionals of cell K (local order: face q = 0..3 x s = 0..5, then e) */
static void bdm2_3d_functionals(const Cell *K, const Q3 *f, real *out) {
    for (int q = 0; q < 4; q++) {
        real P[3][3], A[3], X[6][3], v[3];
        facet_points(K, q, P);
        facet_area_vector(3, P, A);
        face_nodes(P, X);
        for (int s = 0; s < 6; s++) { q3_eval(f, K, X[s], v); out[6 * q + s] = dot3(v, A); }
    }
    real xq[64][3], wq[64];
    int nq = cell_rule(K, 3, xq, wq);      /* degree 3: exact in 3D (R-quad) */
    for (int e = 0; e < 6; e++) {
        real acc = 0;
        for (int t = 0; t < nq; t++) {
            real v[3], om[3];
            q3_eval(f, K, xq[t], v);
            whitney3_at(K, e, xq[t], om);
            acc += wq[t] * dot3(v, om);
        }
        out[24 + e] = acc;
    }
}

static void basis_bdm2_3d(const Cell *K, Q3 *B) {
    Q3 p[30];
    memset(p, 0, sizeof p);
    for (int l = 0; l < 3; l++) for (int k = 0; k < 10; k++) p[10 * l + k].c[l][k] = 1;
    real M[900], C[900], col[30];
    for (int j = 0; j < 30; j++) {
        bdm2_3d_functionals(K, &p[j], col);
        for (int i = 0; i < 30; i++) M[i * 30 + j] = col[i];
    }
    mat_inv(30, M, C);
    for (int j = 0; j < 30; j++) {
        memset(&B[j], 0, sizeof(Q3));
        for (int k = 0; k < 30; k++)
            for (int l = 0; l < 3; l++)
                for (int t = 0; t < 10; t++) B[j].c[l][t] += C[k * 30 + j] * p[k].c[l][t];
    }
}

/* AL velocity block at k = 2 in 3D: the forms of assemble_vel2 (R-vel) with
 * 3-vectors; cell integrals by the 4-point collapsed rule (degree 4, R-quad), facet
 * integrals by the collapsed 3x3 triangle rule (degree 4); h_F = longest face edge, as
 * the k = 1 3D assembly. */
static void assemble_vel2_3d(OCsr *A, Accum *S, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                             const unsigned char *cmask) {
    real xq[64][3], wq[64];
    const real nu2 = (real)2 / p->Re;
    static real loc[900], floc[3600];
    for (i64 c = 0; c < m->nc; c++) {
        if (cmask && !cmask[c]) continue;
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[30];
        int gi[30];
        basis_bdm2_3d(&K, F);
        cell_dofs(m, s, c, gi);
        double pot[4][3];
        real wx[3], bx[3] = {0, 0, 0};
        cell_pot(m, c, w, pot);
        cell_wind(&K, pot, wx);
        if (p->bn) { double bp[4][3]; cell_pot(m, c, p->bn, bp); cell_wind(&K, bp, bx); }
        memset(loc, 0, sizeof(loc));
        int nq = cell_rule(&K, 4, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[30][3], ep[30][3][3], dv[30], gw[30][3];
            for (int a = 0; a < 30; a++) {
                real G[3][3];
                q3_eval(&F[a], &K, xq[t], fv[a]);
                q3_grad(&F[a], &K, xq[t], G);
                for (int l = 0; l < 3; l++) for (int k = 0; k < 3; k++) ep[a][l][k] = (G[l][k] + G[k][l]) / 2;
                dv[a] = G[0][0] + G[1][1] + G[2][2];
                for (int l = 0; l < 3; l++) gw[a][l] = G[l][0] * wx[0] + G[l][1] * wx[1] + G[l][2] * wx[2];
            }
            for (int i = 0; i < 30; i++)
                for (int j = 0; j < 30; j++) {
                    real ee = 0;
                    for (int l = 0; l < 3; l++) for (int k = 0; k < 3; k++) ee += ep[j][l][k] * ep[i][l][k];
                    real v = nu2 * ee - dot3(fv[j], gw[i]) + (real)p->gamma * dv[j] * dv[i];
                    if (p->dt > 0) v += dot3(fv[j], fv[i]) / p->dt;
                    if (p->bn) { real cj[3], ci[3]; cross3(fv[j], bx, cj); cross3(fv[i], bx, ci); v += p->S * dot3(cj, ci); }
                    loc[i * 30 + j] += wq[t] * v;
                }
        }
        scatter(A, S, gi, 30, gi, 30, loc, 30);
    }
    for (i64 f = 0; f < m->nfacet; f++) {
        int cp = m->fcell[2 * f], cm = m->fcell[2 * f + 1];
        if (cmask && !cmask[cp] && !(cm >= 0 && cmask[cm])) continue;
        int interior = cm >= 0, nb = 30;
        Cell Kp, Km;
        Q3 F[60];
        int gi[60], side[60];
        cell_geom(m, cp, &Kp);
        basis_bdm2_3d(&Kp, F);
        cell_dofs(m, s, cp, gi);
        for (int a = 0; a < 30; a++) side[a] = +1;
        if (interior) {
            cell_geom(m, cm, &Km);
            basis_bdm2_3d(&Km, F + 30);
            cell_dofs(m, s, cm, gi + 30);
            for (int a = 30; a < 60; a++) side[a] = -1;
            nb = 60;
        }
        int qf = -1;
        for (int q = 0; q < 4; q++) if (om_facet_of_cell(m, cp, q) == f) qf = q;
        real P[3][3], Av[3];
        facet_points(&Kp, qf, P);
        facet_area_vector(3, P, Av);
        real an = RSQRT(dot3(Av, Av)), n[3];
        double sgn = facet_sign(&Kp, qf, Av);
        for (int k = 0; k < 3; k++) n[k] = sgn * Av[k] / an;
        real hF = 0;
        for (int a = 0; a < 3; a++)
            for (int b = a + 1; b < 3; b++) {
                real t[3] = {P[b][0] - P[a][0], P[b][1] - P[a][1], P[b][2] - P[a][2]};
                real l = RSQRT(dot3(t, t));
                if (l > hF) hF = l;
            }
        real avg = interior ? (real)1 / 2 : (real)1;
        real pen = (real)p->sigma / ((real)p->Re * hF);
        double pot[4][3];
        real wx[3];
        cell_pot(m, cp, w, pot);
        cell_wind(&Kp, pot, wx);
        real wn = dot3(wx, n), awn = RFABS(wn);
        memset(floc, 0, sizeof(floc));
        int nq = facet_rule(3, P, xq, wq);
        for (int t = 0; t < nq; t++) {
            real fv[60][3], en[60][3];
            for (int a = 0; a < nb; a++) {
                const Cell *Ka = side[a] > 0 ? &Kp : &Km;
                real G[3][3];
                q3_eval(&F[a], Ka, xq[t], fv[a]);
                q3_grad(&F[a], Ka, xq[t], G);
                for (int l = 0; l < 3; l++) {
                    real acc = 0;
                    for (int k = 0; k < 3; k++) acc += (G[l][k] + G[k][l]) / 2 * n[k];
                    en[a][l] = acc;
                }
            }
            for (int i = 0; i < nb; i++) {
                real Ji = side[i];
                for (int j = 0; j < nb; j++) {
                    real Jj = side[j];
                    real vv = dot3(fv[j], fv[i]);
                    real t1 = -nu2 * avg * dot3(en[j], fv[i]) * Ji;
                    real t2 = -nu2 * avg * dot3(fv[j], en[i]) * Jj;
                    real t3 = pen * Jj * Ji * vv;
                    real up;
                    if (interior) up = (side[j] > 0 ? (wn + awn) / 2 : -(-wn + awn) / 2) * vv * Ji;
                    else up = (wn + awn) / 2 * vv;
                    floc[i * 60 + j] += wq[t] * (t1 + t2 + t3 + up);
                }
            }
        }
        scatter(A, S, gi, nb, gi, nb, floc, 60);
    }
}

/* the fine BDM2 functional of free DoF I (3D) applied to F living on coarse cell Kc */
static real dof_functional_v3(const OMesh *mf, const OSpace *sf, i64 I, const Q3 *F, const Cell *Kc) {
    int kind = sf->dkind[I], ent = sf->dent[I], sub = sf->dsub[I];
    real v[3];
    if (kind == 2) {
        real P[3][3], A[3], X[6][3];
        for (int a = 0; a < 3; a++)
            for (int k = 0; k < 3; k++) P[a][k] = (real)mf->lat[3 * mf->fv[3 * ent + a] + k] / mf->N;
        facet_area_vector(3, P, A);
        face_nodes(P, X);
        q3_eval(F, Kc, X[sub], v);
        return dot3(v, A);
    }
    Cell Kf;
    cell_geom(mf, ent, &Kf);
    real xq[64][3], wq[64], om[3], acc = 0;
    int nq = cell_rule(&Kf, 3, xq, wq);
    for (int t = 0; t < nq; t++) {
        q3_eval(F, Kc, xq[t], v);
        whitney3_at(&Kf, sub, xq[t], om);
        acc += wq[t] * dot3(v, om);
    }
    return acc;
}

static int op_prolongation3(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc) {
    memset(P, 0, sizeof(*P));
    int *efirst = malloc(sizeof(int) * mf->ne), *ffirst = malloc(sizeof(int) * mf->nfacet);
    for (i64 t = 0; t < mf->ne; t++) efirst[t] = -1;
    for (i64 t = 0; t < mf->nfacet; t++) ffirst[t] = -1;
    for (i64 c = 0; c < mf->nc; c++) {
        for (int q = 0; q < 6; q++) if (efirst[mf->ce[c * 6 + q]] < 0) efirst[mf->ce[c * 6 + q]] = (int)c;
        for (int q = 0; q < 4; q++) { int f = om_facet_of_cell(mf, c, q); if (ffirst[f] < 0) ffirst[f] = (int)c; }
    }
    i64 cap = 1024, nt = 0;
    long long *idx = malloc(sizeof(long long) * 3 * cap);
    real *tv = malloc(sizeof(real) * cap);
    for (i64 I = 0; I < sf->n; I++) {
        int kind = sf->dkind[I], ent = sf->dent[I];
        int cf = kind == 1 ? efirst[ent] : (kind == 3 ? ent : ffirst[ent]);
        i64 ccell = parent_cell(mf, mc, cf);
        Cell Kc;
        cell_geom(mc, ccell, &Kc);
        if (sf->block == ORC_VEL) {                      /* BDM2: all 30 coarse functions */
            Q3 Fv[30];
            int gv[30];
            basis_bdm2_3d(&Kc, Fv);
            cell_dofs(mc, sc, ccell, gv);
            for (int b = 0; b < 30; b++) {
                if (gv[b] < 0) continue;
                real val = dof_functional_v3(mf, sf, I, &Fv[b], &Kc);
                if (nt == cap) { cap *= 2; idx = realloc(idx, sizeof(long long) * 3 * cap); tv = realloc(tv, sizeof(real) * cap); }
                idx[3 * nt] = I; idx[3 * nt + 1] = gv[b]; idx[3 * nt + 2] = nt; tv[nt] = val; nt++;
            }
            continue;
        }
        Q3 F[20];
        int gE[20], gB[15], nb;
        const int *gJ;
        cell_dofs3(mc, sc, ccell, gE, gB);
        if (kind == 1 || kind == 4) { basis3(&Kc, mc->N, 1, F); nb = 20; gJ = gE; }
        else { basis3(&Kc, mc->N, 0, F); nb = 15; gJ = gB; }
        for (int b = 0; b < nb; b++) {
            if (gJ[b] < 0) continue;
            real val = dof_functional3(mf, sf, I, &F[b], &Kc, cf);
            if (nt == cap) { cap *= 2; idx = realloc(idx, sizeof(long long) * 3 * cap); tv = realloc(tv, sizeof(real) * cap); }
            idx[3 * nt] = I; idx[3 * nt + 1] = gJ[b]; idx[3 * nt + 2] = nt; tv[nt] = val; nt++;
        }
    }
    qsort(idx, (size_t)nt, 3 * sizeof(long long), cmp_ij);
    P->n = sf->n;
    P->rp = calloc((size_t)sf->n + 1, sizeof(i64));
    P->ci = malloc(sizeof(int) * (nt ? nt : 1));
    P->v = malloc(sizeof(double) * (nt ? nt : 1));
    i64 used = 0;
    for (i64 t0 = 0; t0 < nt;) {            /* row rounding as R-prol2 */
        i64 t1 = t0;
        while (t1 < nt && idx[3 * t1] == idx[3 * t0]) t1++;
        double mx = 0;
        for (i64 t = t0; t < t1; t++) { double h = (double)tv[idx[3 * t + 2]]; if (fabs(h) > mx) mx = fabs(h); }
        int E = 0;
        if (mx > 0) frexp(mx, &E);
        for (i64 t = t0; t < t1; t++) {
            real x = tv[idx[3 * t + 2]];
            double h = (double)x, l = (double)(x - (real)h);
            double v = (mx > 0 && fabs(h) >= ldexp(mx, -30)) ? grid_round(h, l, E) : 0.0;
            if (v == 0.0) continue;
            P->ci[used] = (int)idx[3 * t + 1];
            P->v[used] = v;
            used++;
            P->rp[idx[3 * t] + 1]++;
        }
        t0 = t1;
    }
    for (i64 i = 0; i < sf->n; i++) P->rp[i + 1] += P->rp[i];
    P->nnz = used;
    free(idx); free(tv); free(efirst); free(ffirst);
    return 0;
}

static void oa_load3v(const OMesh *m, const OSpace *s, const double *fv, double *out) {
    int nq = oa_nq(3), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(out, 0, sizeof(double) * s->n);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[30];
        int g[30];
        basis_bdm2_3d(&K, F);
        cell_dofs(m, s, c, g);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < 30; a++) {
            if (g[a] < 0) continue;
            real acc = 0;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q3_eval(&F[a], &K, xq[t], v);
                const double *f = fv + ((i64)c * nq + t) * nc;
                acc += wq[t] * (f[0] * v[0] + f[1] * v[1] + f[2] * v[2]);
            }
            out[g[a]] += (double)acc;
        }
    }
}

static void oa_eval3v(const OMesh *m, const OSpace *s, const double *coef, double *fv) {
    int nq = oa_nq(3), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(fv, 0, sizeof(double) * m->nc * nq * nc);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[30];
        int g[30];
        basis_bdm2_3d(&K, F);
        cell_dofs(m, s, c, g);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < 30; a++) {
            if (g[a] < 0) continue;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q3_eval(&F[a], &K, xq[t], v);
                double *f = fv + ((i64)c * nq + t) * nc;
                for (int k = 0; k < 3; k++) f[k] += coef[g[a]] * (double)v[k];
            }
        }
    }
}

static double oa_duality_error3v(const OMesh *m, const OSpace *s) {
    double worst = 0;
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[30];
        int g[30];
        basis_bdm2_3d(&K, F);
        cell_dofs(m, s, c, g);
        for (int i = 0; i < 30; i++) {
            if (g[i] < 0) continue;
            for (int j = 0; j < 30; j++) {
                if (g[j] < 0) continue;
                double v = (double)dof_functional_v3(m, s, g[i], &F[j], &K);
                double e = fabs(v - (g[i] == g[j] ? 1.0 : 0.0));
                if (e > worst) worst = e;
            }
        }
    }
    return worst;
}

static void oa_load3(const OMesh *m, const OSpace *s, const double *fv, double *out) {
    if (s->block == ORC_VEL) { oa_load3v(m, s, fv, out); return; }
    int nq = oa_nq(3), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(out, 0, sizeof(double) * s->n);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[35];
        int g[35];
        basis3(&K, m->N, 1, F);
        basis3(&K, m->N, 0, F + 20);
        cell_dofs3(m, s, c, g, g + 20);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < 35; a++) {
            if (g[a] < 0) continue;
            int off = a < 20 ? 0 : 3;
            real acc = 0;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q3_eval(&F[a], &K, xq[t], v);
                const double *f = fv + ((i64)c * nq + t) * nc + off;
                acc += wq[t] * (f[0] * v[0] + f[1] * v[1] + f[2] * v[2]);
            }
            out[g[a]] += (double)acc;
        }
    }
}

static void oa_eval3(const OMesh *m, const OSpace *s, const double *coef, double *fv) {
    if (s->block == ORC_VEL) { oa_eval3v(m, s, coef, fv); return; }
    int nq = oa_nq(3), nc = oa_ncomp(s);
    real xq[64][3], wq[64];
    memset(fv, 0, sizeof(double) * m->nc * nq * nc);
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[35];
        int g[35];
        basis3(&K, m->N, 1, F);
        basis3(&K, m->N, 0, F + 20);
        cell_dofs3(m, s, c, g, g + 20);
        cell_rule(&K, 4, xq, wq);
        for (int a = 0; a < 35; a++) {
            if (g[a] < 0) continue;
            int off = a < 20 ? 0 : 3;
            for (int t = 0; t < nq; t++) {
                real v[3];
                q3_eval(&F[a], &K, xq[t], v);
                double *f = fv + ((i64)c * nq + t) * nc + off;
                for (int k = 0; k < 3; k++) f[k] += coef[g[a]] * (double)v[k];
            }
        }
    }
}

static double oa_duality_error3(const OMesh *m, const OSpace *s) {
    if (s->block == ORC_VEL) return oa_duality_error3v(m, s);
    double worst = 0;
    for (i64 c = 0; c < m->nc; c++) {
        Cell K;
        cell_geom(m, c, &K);
        Q3 F[35];
        int g[35];
        basis3(&K, m->N, 1, F);
        basis3(&K, m->N, 0, F + 20);
        cell_dofs3(m, s, c, g, g + 20);
        for (int i = 0; i < 35; i++) {
            if (g[i] < 0) continue;
            for (int j = 0; j < 35; j++) {
                if (g[j] < 0 || (i < 20) != (j < 20)) continue;
                double v = (double)dof_functional3(m, s, g[i], &F[j], &K, c);
                double e = fabs(v - (g[i] == g[j] ? 1.0 : 0.0));
                if (e > worst) worst = e;
            }
        }
    }
    return worst;
}
