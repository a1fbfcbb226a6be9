/*
 * api.c -- ORACLE public entry points (TEST INFRASTRUCTURE ONLY; see orc.h).
 *
 * A context holds the nested hierarchy, each level's operator assembled
 * by rediscretisation (reading R-coarse / SURVEY A5), its vertex-star patches
 * (P:567-571), the prolongations and the coarse dense LU (stand-in for
 * MUMPS; reading R-coarse).  Levels are numbered 0 = coarsest.
 *
 *   sweep   : one parallel subspace-correction step
 *             r = b - A x;  y_i = A_i^-1 R_i r;  x_d <- fma(theta w_d, c_d, x_d)
 *             with c_d = sum_{i ∋ d} y_i[k_i(d)] (ascending i), w_d = 1/m_d (R-weights)
 *   vcycle  : V_l(b): l=0 coarse LU solve; else nu_pre sweeps from x = 0, restrict
 *             r with P^T, recurse, prolong-add, nu_post sweeps (R-vcycle)
 *   gmres   : right-preconditioned by the V-cycle, x0 = 0, modified Gram-Schmidt,
 *             Givens, no restart; stop when |g_{k+1}| <= max(rtol |b|, atol)
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "orc.h"

typedef struct {
    OMesh m;
    OSpace s;
    OCsr A;
    OPatches pt;
    double **lu;      /* per patch n_i*n_i row-major factor (lazy) */
    int **perm;
    OCsr P, PT;       /* to the next coarser level (l >= 1) */
    double *w;        /* potential of the advecting field on this level's vertices (R-w) */
    double *bn;       /* potential of B^n on this level's vertices (NEXT-4), or NULL */
} OLevel;

typedef struct {
    int block, dim, nlev;
    int degree;       /* element degree k (NEXT-2) */
    int weights_mode; /* 0 by degree, 1 per-DoF 1/m_d, 2 uniform 1/max m_d */
    OParams p;
    double theta;
    int smoother, smoother_its;   /* 0: nu_pre / nu_post Richardson sweeps; 1: GMRES(m) (NEXT-1) */
    OLevel *lv;
    double *clu;      /* coarse LU (row-major n0*n0) */
    int *cperm;
    int cstat;        /* status of the coarse factorisation */
    int status;
} OCtx;

static void level_free(OLevel *L) {
    if (L->lu) {
        for (i64 i = 0; i < L->pt.np; i++) { free(L->lu[i]); free(L->perm[i]); }
        free(L->lu); free(L->perm);
    }
    oc_free(&L->A); oc_free(&L->P); oc_free(&L->PT);
    opt_free(&L->pt); os_free(&L->s); om_free(&L->m); free(L->w); free(L->bn);
}

void orc_destroy(OCtx *c) {
    if (!c) return;
    for (int l = 0; l < c->nlev; l++) level_free(&c->lv[l]);
    free(c->lv); free(c->clu); free(c->cperm); free(c);
}

/* dparams: Re, Rem, S, gamma, sigma, mu, theta, dt ; iparams: nu_pre, nu_post, picard, degree
 * w_fine: potential of the advecting field at the finest vertices (vertex order of
 *         R-mesh): 2D stream function psi (1 per vertex), 3D vector potential A (3 per vertex).
 * cmask_fine: NULL, or a finest-level cell mask (only then: assemble the finest
 * level restricted to it and build no coarser level; used for bounded samples). */
OCtx *orc_create_masked(int block, int dim, int N, int nlev, const double *dparams, const int *iparams,
                        const double *w_fine, const unsigned char *cmask_fine, const double *bn_fine) {
    if ((block != ORC_EB && block != ORC_VEL) || (dim != 2 && dim != 3) || nlev < 1 || N < 1) return NULL;
    if (N % (1 << (nlev - 1))) return NULL;
    OCtx *c = calloc(1, sizeof(OCtx));
    c->block = block; c->dim = dim; c->nlev = nlev;
    c->p.Re = dparams[0]; c->p.Rem = dparams[1]; c->p.S = dparams[2]; c->p.gamma = dparams[3];
    c->p.sigma = dparams[4]; c->p.mu = dparams[5]; c->theta = dparams[6];
    c->p.nu_pre = iparams[0]; c->p.nu_post = iparams[1];
    c->p.dt = dparams[7]; c->p.picard = iparams[2];
    int degree = iparams[3];
    if (!(degree == 1 || degree == 2)) { free(c); return NULL; }
    c->degree = degree;
    /* iparams[4] weights_mode (0 by degree, 1 per-DoF 1/m_d, 2 uniform 1/max m_d);
     * iparams[5] newton_reaction: (u . grad u^n, v) of Table 1 row F -- R-w makes
     * u^n constant on every cell, so the cellwise term is identically zero (reading
     * R-newton): the flag is accepted and the operator is unchanged                      */
    c->weights_mode = iparams[4];
    if (c->weights_mode < 0 || c->weights_mode > 2 || iparams[5] < 0 || iparams[5] > 1) { free(c); return NULL; }
    c->lv = calloc((size_t)nlev, sizeof(OLevel));
    int lo = cmask_fine ? nlev - 1 : 0;
    for (int l = nlev - 1; l >= lo; l--) {
        OLevel *L = &c->lv[l];
        int Nl = N >> (nlev - 1 - l), step = 1 << (nlev - 1 - l);
        om_build(&L->m, dim, Nl);
        os_build(&L->s, &L->m, block, degree);
        /* w on this level: injection of the finest vertex values (R-w) */
        int nc = dim == 2 ? 1 : 3;
        L->w = malloc(sizeof(double) * nc * L->m.nv);
        for (i64 v = 0; v < L->m.nv; v++) {
            int i = L->m.lat[3 * v] * step, j = L->m.lat[3 * v + 1] * step, k = L->m.lat[3 * v + 2] * step;
            i64 fv = dim == 2 ? i + (i64)(N + 1) * j : i + (i64)(N + 1) * (j + (i64)(N + 1) * k);
            for (int t = 0; t < nc; t++) L->w[v * nc + t] = w_fine[fv * nc + t];
        }
        if (bn_fine) {      /* B^n potential, injected like w (NEXT-4) */
            L->bn = malloc(sizeof(double) * nc * L->m.nv);
            for (i64 v = 0; v < L->m.nv; v++) {
                int i = L->m.lat[3 * v] * step, j = L->m.lat[3 * v + 1] * step, k = L->m.lat[3 * v + 2] * step;
                i64 fv = dim == 2 ? i + (i64)(N + 1) * j : i + (i64)(N + 1) * (j + (i64)(N + 1) * k);
                for (int t = 0; t < nc; t++) L->bn[v * nc + t] = bn_fine[fv * nc + t];
            }
        }
        c->p.bn = L->bn;
        oa_assemble_masked(&L->A, &L->m, &L->s, &c->p, L->w, l == nlev - 1 ? cmask_fine : NULL);
        opt_build(&L->pt, &L->m, &L->s);
    }
    if (!cmask_fine)
        for (int l = 1; l < nlev; l++) {
            op_prolongation(&c->lv[l].P, &c->lv[l].m, &c->lv[l].s, &c->lv[l - 1].m, &c->lv[l - 1].s);
            oc_transpose(&c->lv[l].PT, &c->lv[l].P, c->lv[l - 1].s.n);
        }
    return c;
}

OCtx *orc_create(int block, int dim, int N, int nlev, const double *dparams, const int *iparams,
                 const double *w_fine) {
    return orc_create_masked(block, dim, N, nlev, dparams, iparams, w_fine, NULL, NULL);
}

/* out: n, nnz, npatch, sum_n, sum_n2, nE, nv, nc, ne, nf, P nnz */
int orc_level_info(const OCtx *c, int l, i64 *out) {
    if (!c || l < 0 || l >= c->nlev) return 1;
    const OLevel *L = &c->lv[l];
    i64 s2 = 0;
    for (i64 i = 0; i < L->pt.np; i++) { i64 k = L->pt.ptr[i + 1] - L->pt.ptr[i]; s2 += k * k; }
    out[0] = L->s.n; out[1] = L->A.nnz; out[2] = L->pt.np; out[3] = L->pt.np ? L->pt.ptr[L->pt.np] : 0;
    out[4] = s2; out[5] = L->s.nE; out[6] = L->m.nv; out[7] = L->m.nc; out[8] = L->m.ne; out[9] = L->m.nf;
    out[10] = L->P.nnz;
    return 0;
}

int orc_export_csr(const OCtx *c, int l, i64 *rp, int *ci, double *v) {
    const OCsr *A = &c->lv[l].A;
    memcpy(rp, A->rp, sizeof(i64) * (A->n + 1));
    memcpy(ci, A->ci, sizeof(int) * A->nnz);
    memcpy(v, A->v, sizeof(double) * A->nnz);
    return 0;
}

int orc_export_prolongation(const OCtx *c, int l, i64 *rp, int *ci, double *v) {
    if (l < 1) return 1;
    const OCsr *A = &c->lv[l].P;
    memcpy(rp, A->rp, sizeof(i64) * (A->n + 1));
    memcpy(ci, A->ci, sizeof(int) * A->nnz);
    memcpy(v, A->v, sizeof(double) * A->nnz);
    return 0;
}

int orc_export_patches(const OCtx *c, int l, i64 *ptr, int *dofs, int *vert, int *mult) {
    const OPatches *pt = &c->lv[l].pt;
    memcpy(ptr, pt->ptr, sizeof(i64) * (pt->np + 1));
    memcpy(dofs, pt->dofs, sizeof(int) * pt->ptr[pt->np]);
    memcpy(vert, pt->vert, sizeof(int) * pt->np);
    memcpy(mult, pt->mult, sizeof(int) * c->lv[l].s.n);
    return 0;
}

/* mesh export for tests: x (nv*3), cv (nc*(d+1)), ev (ne*2), fv (nf*3), fcell (nfacet*2),
 * dof entity maps (n each) */
int orc_export_mesh(const OCtx *c, int l, double *x, int *cv, int *ev, int *fv, int *fcell, int *dkind,
                    int *dent, int *dsub) {
    const OLevel *L = &c->lv[l];
    const OMesh *m = &L->m;
    if (x) memcpy(x, m->x, sizeof(double) * 3 * m->nv);
    if (cv) memcpy(cv, m->cv, sizeof(int) * (m->dim + 1) * m->nc);
    if (ev) memcpy(ev, m->ev, sizeof(int) * 2 * m->ne);
    if (fv && m->nf) memcpy(fv, m->fv, sizeof(int) * 3 * m->nf);
    if (fcell) memcpy(fcell, m->fcell, sizeof(int) * 2 * m->nfacet);
    if (dkind) memcpy(dkind, L->s.dkind, sizeof(int) * L->s.n);
    if (dent) memcpy(dent, L->s.dent, sizeof(int) * L->s.n);
    if (dsub) memcpy(dsub, L->s.dsub, sizeof(int) * L->s.n);
    return 0;
}

/* ---------------- order-defined kernels (R-order) ---------------- */

/* r = b - A x: row sums as an fma chain from +0.0 in ascending column order */
static void residual(const OCsr *A, const double *b, const double *x, double *r) {
    for (i64 i = 0; i < A->n; i++) {
        double s = 0.0;
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) s = fma(A->v[t], x[A->ci[t]], s);
        r[i] = b[i] - s;
    }
}

int orc_spmv(const OCtx *c, int l, const double *x, double *y) {
    const OCsr *A = &c->lv[l].A;
    for (i64 i = 0; i < A->n; i++) {
        double s = 0.0;
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) s = fma(A->v[t], x[A->ci[t]], s);
        y[i] = s;
    }
    return 0;
}

int orc_residual(const OCtx *c, int l, const double *b, const double *x, double *r) {
    residual(&c->lv[l].A, b, x, r);
    return 0;
}

/* dense principal submatrix A_i = R_i A R_i^T */
static void patch_matrix(const OLevel *L, i64 i, double *a, double *amax) {
    const OPatches *pt = &L->pt;
    int n = (int)(pt->ptr[i + 1] - pt->ptr[i]);
    const int *dofs = pt->dofs + pt->ptr[i];
    double mx = 0;
    for (int r = 0; r < n; r++)
        for (int q = 0; q < n; q++) {
            i64 p = oc_find(&L->A, dofs[r], dofs[q]);
            a[(i64)r * n + q] = p >= 0 ? L->A.v[p] : 0.0;
            if (fabs(a[(i64)r * n + q]) > mx) mx = fabs(a[(i64)r * n + q]);
        }
    *amax = mx;
}

int orc_patch_matrix(const OCtx *c, int l, i64 i, double *a) {
    double amax;
    patch_matrix(&c->lv[l], i, a, &amax);
    return 0;
}

/* returns 0 or 1 + (patch index) of the first singular patch */
static i64 factor_level(OCtx *c, int l) {
    OLevel *L = &c->lv[l];
    if (L->lu) return 0;
    L->lu = calloc((size_t)L->pt.np, sizeof(double *));
    L->perm = calloc((size_t)L->pt.np, sizeof(int *));
    for (i64 i = 0; i < L->pt.np; i++) {
        int n = (int)(L->pt.ptr[i + 1] - L->pt.ptr[i]);
        double amax;
        L->lu[i] = malloc(sizeof(double) * n * n);
        L->perm[i] = malloc(sizeof(int) * n);
        patch_matrix(L, i, L->lu[i], &amax);
        if (od_lu(L->lu[i], n, L->perm[i], amax)) return i + 1;
    }
    return 0;
}

int orc_patch_lu(OCtx *c, int l, i64 i, double *lu, int *perm) {
    OLevel *L = &c->lv[l];
    int n = (int)(L->pt.ptr[i + 1] - L->pt.ptr[i]);
    double amax;
    patch_matrix(L, i, lu, &amax);
    return od_lu(lu, n, perm, amax);
}

/* one sweep S(x; b) on level l (R-sweep). returns 0 / 1+patch if singular */
/* update weight of DoF d ("u^{k+1} = u^k + sum_i w_i du_i"):
 * R-weights (k = 1): the partition of unity theta / m_d;
 * R-weights2 (k = 2): the uniform theta / max_d m_d -- a per-subspace damping parameter,
 * which keeps every local kernel correction in the kernel (at k = 2 the multiplicities
 * differ inside a patch: facet DoFs 2, cell DoFs 3, so 1/m_d would not).            */
static double dof_weight(const OCtx *c, const OPatches *pt, i64 d) {
    /* weights_mode: 1 = per-DoF 1/m_d, 2 = uniform 1/max m_d, 0 = by degree */
    const int uniform = c->weights_mode == 2 || (c->weights_mode == 0 && c->degree == 2);
    if (uniform) return c->theta * (1.0 / (pt->mmax > 0 ? pt->mmax : 1));
    return c->theta * (1.0 / pt->mult[d]);
}

static i64 sweep(OCtx *c, int l, int x_is_zero, const double *b, double *x) {
    OLevel *L = &c->lv[l];
    i64 bad = factor_level(c, l);
    if (bad) return bad;
    i64 n = L->s.n;
    const OPatches *pt = &L->pt;
    double *r = malloc(sizeof(double) * n);
    double *y = malloc(sizeof(double) * (pt->ptr[pt->np] ? pt->ptr[pt->np] : 1));
    double *rl = malloc(sizeof(double) * 512);
    if (x_is_zero) { for (i64 d = 0; d < n; d++) { r[d] = b[d]; x[d] = 0.0; } }
    else residual(&L->A, b, x, r);
    for (i64 i = 0; i < pt->np; i++) {
        int ni = (int)(pt->ptr[i + 1] - pt->ptr[i]);
        for (int k = 0; k < ni; k++) rl[k] = r[pt->dofs[pt->ptr[i] + k]];
        od_lu_solve(L->lu[i], ni, L->perm[i], rl, y + pt->ptr[i]);
    }
    for (i64 d = 0; d < n; d++) {
        double cd = 0.0;
        for (i64 t = pt->dptr[d]; t < pt->dptr[d + 1]; t++) cd += y[pt->dslot[t]];
        double wd = dof_weight(c, pt, d);
        x[d] = fma(wd, cd, x[d]);
    }
    free(r); free(y); free(rl);
    return 0;
}

i64 orc_sweep(OCtx *c, int l, int nsweeps, int x_is_zero, const double *b, double *x) {
    for (int s = 0; s < nsweeps; s++) {
        i64 st = sweep(c, l, x_is_zero && s == 0, b, x);
        if (st) return st;
    }
    return 0;
}

/* x_new[d] for the sampled DoFs after ONE sweep, computing only the patches that
 * contain them (same arithmetic as sweep(); used at full sizes). */
i64 orc_sweep_sample(OCtx *c, int l, int x_is_zero, const double *b, const double *x, i64 ns, const int *dofs,
                     double *out) {
    OLevel *L = &c->lv[l];
    const OPatches *pt = &L->pt;
    double *a = malloc(sizeof(double) * 512 * 512);
    int *perm = malloc(sizeof(int) * 512);
    double *rl = malloc(sizeof(double) * 512), *yl = malloc(sizeof(double) * 512);
    /* slot -> patch via binary search on ptr */
    for (i64 s = 0; s < ns; s++) {
        int d = dofs[s];
        double cd = 0.0;
        for (i64 t = pt->dptr[d]; t < pt->dptr[d + 1]; t++) {
            i64 slot = pt->dslot[t], lo = 0, hi = pt->np - 1;
            while (lo < hi) { i64 mid = (lo + hi + 1) / 2; if (pt->ptr[mid] <= slot) lo = mid; else hi = mid - 1; }
            i64 i = lo;
            int ni = (int)(pt->ptr[i + 1] - pt->ptr[i]);
            double amax;
            patch_matrix(L, i, a, &amax);
            if (od_lu(a, ni, perm, amax)) { free(a); free(perm); free(rl); free(yl); return i + 1; }
            for (int k = 0; k < ni; k++) {
                int e = pt->dofs[pt->ptr[i] + k];
                if (x_is_zero) rl[k] = b[e];
                else {
                    double sacc = 0.0;
                    for (i64 q = L->A.rp[e]; q < L->A.rp[e + 1]; q++) sacc = fma(L->A.v[q], x[L->A.ci[q]], sacc);
                    rl[k] = b[e] - sacc;
                }
            }
            od_lu_solve(a, ni, perm, rl, yl);
            cd += yl[slot - pt->ptr[i]];
        }
        double wd = dof_weight(c, pt, d);
        out[s] = fma(wd, cd, x_is_zero ? 0.0 : x[d]);
    }
    free(a); free(perm); free(rl); free(yl);
    return 0;
}

/* ---------------- transfer (R-vcycle: ascending fma chains from +0.0) ---------------- */
int orc_restrict(const OCtx *c, int l, const double *r, double *rc) {
    const OCsr *T = &c->lv[l].PT;
    for (i64 J = 0; J < T->n; J++) {
        double s = 0.0;
        for (i64 t = T->rp[J]; t < T->rp[J + 1]; t++) s = fma(T->v[t], r[T->ci[t]], s);
        rc[J] = s;
    }
    return 0;
}

int orc_prolong_add(const OCtx *c, int l, const double *ec, double *x) {
    const OCsr *P = &c->lv[l].P;
    for (i64 I = 0; I < P->n; I++) {
        double s = 0.0;
        for (i64 t = P->rp[I]; t < P->rp[I + 1]; t++) s = fma(P->v[t], ec[P->ci[t]], s);
        x[I] = x[I] + s;
    }
    return 0;
}

/* ---------------- coarse solve (dense LU, R-coarse) ----------------
 * SURVEY 8(c.8) "l = 0: return the coarse LU solve": the coarse operator is factored
 * by R-lu (od_lu, the stand-in for MUMPS) and every coarse solve is the R-lu
 * forward/back substitution of c.6 (od_lu_solve) -- no other arithmetic.          */
static int coarse_factor(OCtx *c) {
    if (c->clu) return c->cstat;
    OLevel *L = &c->lv[0];
    i64 n = L->s.n;
    c->clu = calloc((size_t)((n * n) > 0 ? n * n : 1), sizeof(double));
    c->cperm = malloc(sizeof(int) * (n ? n : 1));
    double amax = 0;
    for (i64 i = 0; i < n; i++)
        for (i64 t = L->A.rp[i]; t < L->A.rp[i + 1]; t++) {
            c->clu[i * n + L->A.ci[t]] = L->A.v[t];
            if (fabs(L->A.v[t]) > amax) amax = fabs(L->A.v[t]);
        }
    c->cstat = od_lu(c->clu, (int)n, c->cperm, amax);
    return c->cstat;
}

int orc_coarse_solve(OCtx *c, const double *b, double *x) {
    if (coarse_factor(c)) return 1;
    od_lu_solve(c->clu, (int)c->lv[0].s.n, c->cperm, b, x);
    return 0;
}

int orc_coarse_lu(OCtx *c, double *lu, int *perm) {
    int st = coarse_factor(c);
    i64 n = c->lv[0].s.n;
    memcpy(lu, c->clu, sizeof(double) * n * n);
    memcpy(perm, c->cperm, sizeof(int) * n);
    return st;
}

static int gmres_smooth(OCtx *c, int l, int m, int x_is_zero, const double *b, double *x);

static int vcycle(OCtx *c, int l, const double *b, double *x) {
    if (l == 0) return orc_coarse_solve(c, b, x);
    OLevel *L = &c->lv[l];
    i64 n = L->s.n, nc = c->lv[l - 1].s.n;
    for (i64 d = 0; d < n; d++) x[d] = 0.0;
    if (c->smoother == 1) {
        if (gmres_smooth(c, l, c->smoother_its, 1, b, x)) return 1;
    } else {
        int zero = 1;
        for (int s = 0; s < c->p.nu_pre; s++) { if (sweep(c, l, zero, b, x)) return 1; zero = 0; }
    }
    double *r = malloc(sizeof(double) * n), *rc = malloc(sizeof(double) * nc), *ec = malloc(sizeof(double) * nc);
    residual(&L->A, b, x, r);
    orc_restrict(c, l, r, rc);
    int st = vcycle(c, l - 1, rc, ec);
    if (!st) {
        orc_prolong_add(c, l, ec, x);
        if (c->smoother == 1) st = gmres_smooth(c, l, c->smoother_its, 0, b, x) ? 1 : 0;
        else
            for (int s = 0; s < c->p.nu_post; s++) if (sweep(c, l, 0, b, x)) { st = 1; break; }
    }
    free(r); free(rc); free(ec);
    return st;
}

int orc_vcycle(OCtx *c, const double *b, double *x) { return vcycle(c, c->nlev - 1, b, x); }
int orc_vcycle_level(OCtx *c, int l, const double *b, double *x) { return vcycle(c, l, b, x); }

/* GMRES(V) (c.9): right-preconditioned by the V-cycle, x0 = 0, modified
 * Gram-Schmidt, Givens rotations, no restart; stop when |g_{k+1}| <= max(rtol |b|, atol).
 * The V-cycle is linear (fixed sweep counts), so GMRES that stores Z_k = V v_k is the
 * same iteration as FGMRES: both run orc_fgmres.  c.9 fixes no reduction order for the
 * inner products; they follow reading R-dot, so that the residual history
 * is order-defined and can be compared bit for bit.  hist[k] = |g_k|.   */
int orc_fgmres(OCtx *c, const double *b, double *x, double rtol, double atol, int maxit, int *its_out,
               double *hist);
int orc_gmres(OCtx *c, const double *b, double *x, double rtol, double atol, int maxit, int *its_out,
              double *hist) {
    return orc_fgmres(c, b, x, rtol, atol, maxit, its_out, hist);
}

/* manufactured-solution helpers: quadrature points/weights of every cell, load
 * vector (f, phi_i) and evaluation of a discrete field at those points */
int orc_quad_info(const OCtx *c, int l, i64 *out) {
    const OLevel *L = &c->lv[l];
    out[0] = L->m.nc * oa_nq(L->m.dim); out[1] = oa_ncomp(&L->s);
    return 0;
}
int orc_quadrature(const OCtx *c, int l, double *pts, double *wts) {
    oa_quadrature(&c->lv[l].m, pts, wts);
    return 0;
}
int orc_load(const OCtx *c, int l, const double *fv, double *out) {
    oa_load(&c->lv[l].m, &c->lv[l].s, fv, out);
    return 0;
}
int orc_eval(const OCtx *c, int l, const double *coef, double *fv) {
    oa_eval(&c->lv[l].m, &c->lv[l].s, coef, fv);
    return 0;
}

double orc_duality_error(const OCtx *c, int l) { return oa_duality_error(&c->lv[l].m, &c->lv[l].s); }

/* TEST HOOK: replace level l's subspace decomposition by the given one (ascending
 * DoF lists); used to pin the sweep machinery against special decompositions
 * (e.g. one patch covering every DoF => one sweep from zero is the direct solve). */
int orc_set_patches(OCtx *c, int l, i64 np, const i64 *ptr, const int *dofs) {
    OLevel *L = &c->lv[l];
    if (L->lu) {
        for (i64 i = 0; i < L->pt.np; i++) { free(L->lu[i]); free(L->perm[i]); }
        free(L->lu); free(L->perm); L->lu = NULL; L->perm = NULL;
    }
    i64 n = L->s.n, used = ptr[np];
    OPatches *pt = &L->pt;
    opt_free(pt);
    pt->np = np;
    pt->vert = calloc((size_t)np + 1, sizeof(int));
    pt->ptr = malloc(sizeof(i64) * (np + 1));
    memcpy(pt->ptr, ptr, sizeof(i64) * (np + 1));
    pt->dofs = malloc(sizeof(int) * (used ? used : 1));
    memcpy(pt->dofs, dofs, sizeof(int) * used);
    pt->mult = calloc((size_t)n, sizeof(int));
    for (i64 t = 0; t < used; t++) pt->mult[dofs[t]]++;
    pt->mmax = 0;
    for (i64 d = 0; d < n; d++) if (pt->mult[d] > pt->mmax) pt->mmax = pt->mult[d];
    pt->dptr = calloc((size_t)n + 1, sizeof(i64));
    for (i64 d = 0; d < n; d++) pt->dptr[d + 1] = pt->dptr[d] + pt->mult[d];
    pt->dslot = malloc(sizeof(i64) * (used ? used : 1));
    i64 *f2 = calloc((size_t)n, sizeof(i64));
    for (i64 t = 0; t < used; t++) { int d = dofs[t]; pt->dslot[pt->dptr[d] + f2[d]++] = t; }
    free(f2);
    return 0;
}

/* dense LU (R-lu) of a row-major n x n matrix and one solve; returns od_lu's status */
int orc_dense_lu_solve(int n, const double *a, const double *b, double *x, double *lu_out, int *perm_out) {
    double amax = 0;
    for (i64 t = 0; t < (i64)n * n; t++) { lu_out[t] = a[t]; if (fabs(a[t]) > amax) amax = fabs(a[t]); }
    int st = od_lu(lu_out, n, perm_out, amax);
    if (!st) od_lu_solve(lu_out, n, perm_out, b, x);
    return st;
}

/* ===================================================================================
 * NEXT-1: the paper's relaxation -- "six preconditioned GMRES iterations
 * as the smoother on each level" -- and flexible GMRES as the outermost Krylov
 * solver, with the paper's 1e-7 / 1e-7 Euclidean tolerances.
 * Readings: R-dot (pinned reduction order of inner products), R-gmres6
 * (left preconditioning by the Schwarz operator B r = S(0; r), modified Gram-Schmidt,
 * Givens rotations, x0 = current iterate, exactly m iterations unless breakdown),
 * R-fgmres (right flexible preconditioning by the GMRES-smoothed V-cycle, x0 = 0).
 * =================================================================================== */

/* R-dot: blocks of 256 consecutive entries, each an fma chain from +0.0 in ascending
 * order; block sums combined by a pairwise tree (level by level, s_k = s_2k + s_2k+1,
 * an odd last entry carried up).                                                    */
double od_dot(const double *a, const double *b, i64 n) {
    if (n <= 0) return 0.0;
    i64 m = (n + 255) / 256;
    double *s = malloc(sizeof(double) * m);
    for (i64 B = 0; B < m; B++) {
        double acc = 0.0;
        for (i64 i = 256 * B; i < n && i < 256 * (B + 1); i++) acc = fma(a[i], b[i], acc);
        s[B] = acc;
    }
    while (m > 1) {
        i64 h = m / 2;
        for (i64 k = 0; k < h; k++) s[k] = s[2 * k] + s[2 * k + 1];
        if (m & 1) s[h] = s[m - 1];
        m = h + (m & 1);
    }
    double r = s[0];
    free(s);
    return r;
}

/* the Schwarz operator as a preconditioner: z = B r = one sweep from zero with rhs r */
static int apply_B(OCtx *c, int l, const double *r, double *z) {
    return sweep(c, l, 1, r, z) ? 1 : 0;
}

/* Givens / least-squares state shared by GMRES(m) and FGMRES; H is (m+1) x m row-major.
 * Every product and sum is rounded separately (no fma): the GPU mirrors these steps. */
static void givens_column(double *H, int m, double *cs, double *sn, double *g, int k) {
    for (int i = 0; i < k; i++) {
        double a = H[i * m + k], bb = H[(i + 1) * m + k];
        H[i * m + k] = cs[i] * a + sn[i] * bb;
        H[(i + 1) * m + k] = -sn[i] * a + cs[i] * bb;
    }
    double a = H[k * m + k], bb = H[(k + 1) * m + k];
    double rr = sqrt(a * a + bb * bb);
    cs[k] = a / rr;
    sn[k] = bb / rr;
    H[k * m + k] = rr;
    H[(k + 1) * m + k] = 0.0;
    g[k + 1] = -sn[k] * g[k];
    g[k] = cs[k] * g[k];
}

static void back_substitute(const double *H, int m, const double *g, int kk, double *y) {
    for (int i = kk - 1; i >= 0; i--) {
        double s = g[i];
        for (int j = i + 1; j < kk; j++) s = s - H[i * m + j] * y[j];
        y[i] = s / H[i * m + i];
    }
}

/* GMRES(m) smoothing step (R-gmres6): x <- x + V y minimising ||B(b - A x)|| over the
 * Krylov space of B A; x_is_zero: x = 0 on entry (the residual is b).               */
static int gmres_smooth(OCtx *c, int l, int m, int x_is_zero, const double *b, double *x) {
    OLevel *L = &c->lv[l];
    i64 n = L->s.n;
    double *r = malloc(sizeof(double) * n), *t = malloc(sizeof(double) * n), *w = malloc(sizeof(double) * n);
    double *V = malloc(sizeof(double) * n * (m + 1));
    double *H = calloc((size_t)(m + 1) * m, sizeof(double)), *cs = calloc(m, sizeof(double)),
           *sn = calloc(m, sizeof(double)), *g = calloc(m + 1, sizeof(double)), *y = calloc(m, sizeof(double));
    int st = 0, kk = 0;
    if (x_is_zero) { for (i64 i = 0; i < n; i++) { r[i] = b[i]; x[i] = 0.0; } }
    else residual(&L->A, b, x, r);
    if (apply_B(c, l, r, w)) { st = 1; goto done; }
    double beta = sqrt(od_dot(w, w, n));
    if (beta == 0.0) goto done;
    for (i64 i = 0; i < n; i++) V[i] = w[i] / beta;
    g[0] = beta;
    for (int k = 0; k < m; k++) {
        orc_spmv(c, l, V + k * n, t);
        if (apply_B(c, l, t, w)) { st = 1; goto done; }
        for (int i = 0; i <= k; i++) {
            double h = od_dot(w, V + i * n, n);
            H[i * m + k] = h;
            for (i64 j = 0; j < n; j++) w[j] = fma(-h, V[i * n + j], w[j]);
        }
        double hn = sqrt(od_dot(w, w, n));
        H[(k + 1) * m + k] = hn;
        givens_column(H, m, cs, sn, g, k);
        kk = k + 1;
        if (hn == 0.0) break;
        if (k + 1 < m) for (i64 j = 0; j < n; j++) V[(k + 1) * n + j] = w[j] / hn;
    }
    back_substitute(H, m, g, kk, y);
    for (int i = 0; i < kk; i++)
        for (i64 j = 0; j < n; j++) x[j] = fma(y[i], V[i * n + j], x[j]);
done:
    free(r); free(t); free(w); free(V); free(H); free(cs); free(sn); free(g); free(y);
    return st;
}

void orc_set_smoother(OCtx *c, int kind, int its) {
    c->smoother = kind;
    c->smoother_its = its;
}

/* flexible GMRES (R-fgmres) with the current V-cycle as a variable right preconditioner;
 * hist[k] = |g_k|, k = 0..its.  Returns 0 converged, 1 maxit, 2 preconditioner failure. */
int orc_fgmres(OCtx *c, const double *b, double *x, double rtol, double atol, int maxit, int *its_out,
               double *hist) {
    int l = c->nlev - 1;
    i64 n = c->lv[l].s.n;
    double beta = sqrt(od_dot(b, b, n));
    double tol = rtol * beta > atol ? rtol * beta : atol;
    for (i64 i = 0; i < n; i++) x[i] = 0.0;
    hist[0] = beta;
    *its_out = 0;
    if (beta <= tol) return 0;
    int m = maxit;
    double *V = malloc(sizeof(double) * n * (m + 1)), *Z = malloc(sizeof(double) * n * m);
    double *H = calloc((size_t)(m + 1) * m, sizeof(double)), *cs = calloc(m, sizeof(double)),
           *sn = calloc(m, sizeof(double)), *g = calloc(m + 1, sizeof(double)), *y = calloc(m, sizeof(double));
    double *w = malloc(sizeof(double) * n);
    for (i64 i = 0; i < n; i++) V[i] = b[i] / beta;
    g[0] = beta;
    int k, conv = 0, fail = 0;
    for (k = 0; k < m; k++) {
        if (vcycle(c, l, V + k * n, Z + k * n)) { fail = 1; break; }
        orc_spmv(c, l, Z + k * n, w);
        for (int i = 0; i <= k; i++) {
            double h = od_dot(w, V + i * n, n);
            H[i * m + k] = h;
            for (i64 j = 0; j < n; j++) w[j] = fma(-h, V[i * n + j], w[j]);
        }
        double hn = sqrt(od_dot(w, w, n));
        H[(k + 1) * m + k] = hn;
        givens_column(H, m, cs, sn, g, k);
        hist[k + 1] = fabs(g[k + 1]);
        if (fabs(g[k + 1]) <= tol) { k++; conv = 1; break; }
        if (hn == 0.0) { k++; break; }
        for (i64 j = 0; j < n; j++) V[(k + 1) * n + j] = w[j] / hn;
    }
    if (!fail) {
        back_substitute(H, m, g, k, y);
        for (int i = 0; i < k; i++)
            for (i64 j = 0; j < n; j++) x[j] = fma(y[i], Z[i * n + j], x[j]);
        *its_out = k;
    }
    free(V); free(Z); free(H); free(cs); free(sn); free(g); free(y); free(w);
    return fail ? 2 : (conv ? 0 : 1);
}

/* test access to the pinned inner product */
double orc_dot(const double *a, const double *b, i64 n) { return od_dot(a, b, n); }

/* one GMRES(m) smoothing step on level l (test access; x in/out) */
int orc_gmres_smooth(OCtx *c, int l, int m, int x_is_zero, const double *b, double *x) {
    return gmres_smooth(c, l, m, x_is_zero, b, x);
}

/* ===================================================================================
 * NEXT-3: the paper's outer solver.  FGMRES on the Newton
 * system [[F+D, B^T, J, J~+D~1+D~2], [B, 0, 0, 0], [G, 0, M_E, G~-A/Rem],
 * [0, 0, A^T, C]] with the block upper-triangular preconditioner
 *   P = [[I, -M~^-1 K], [0, I]] diag(M~^-1, S~^-1),   S~ = the E-B block,
 * M~^-1 = two iterations of FGMRES on the (u,p) block preconditioned by the
 * hydrodynamic block preconditioner: y_p = -(1/Re + gamma) M_p^-1 s_p,
 * y_u = V_u(s_u - B^T y_p);  S~^-1 = two iterations of FGMRES on the E-B block with the
 * E-B V-cycle.  Readings: R-coupled (E^n = 0, so J~ = 0; u^n = w_h, B^n from its
 * potential), R-outer (orders of the sums, inner FGMRES(2) exactly 2 iterations).
 * =================================================================================== */
typedef struct {
    OCtx *vel, *eb;
    OCsr A;          /* coupled operator over [u | p | E | B]                     */
    OCsr Mup;        /* rows/cols (u, p)                                          */
    OCsr K;          /* u rows x [E | B] columns: [J | J~ + D~1 + D~2]            */
    OCsr Bt;         /* u rows x p columns                                        */
    i64 nu, np, nE, nB, n;
    double cS, Kinv; /* -(1/Re + gamma), 1/|K|                                    */
} OCoupled;

static void csr_chain(const OCsr *A, const double *x, double *y) {
    for (i64 i = 0; i < A->n; i++) {
        double s = 0.0;
        for (i64 t = A->rp[i]; t < A->rp[i + 1]; t++) s = fma(A->v[t], x[A->ci[t]], s);
        y[i] = s;
    }
}

/* append row r of B (columns shifted by `shift`) to the CSR under construction */
typedef struct { i64 *rp; int *ci; double *v; i64 used, cap, rows; } Builder;
static void b_push(Builder *b, const OCsr *B, i64 r, i64 shift) {
    for (i64 t = B->rp[r]; t < B->rp[r + 1]; t++) {
        if (b->used == b->cap) { b->cap *= 2; b->ci = realloc(b->ci, sizeof(int) * b->cap); b->v = realloc(b->v, sizeof(double) * b->cap); }
        b->ci[b->used] = (int)(B->ci[t] + shift); b->v[b->used] = B->v[t]; b->used++;
    }
}
static void b_endrow(Builder *b) { b->rp[++b->rows] = b->used; }
static void b_init(Builder *b, i64 nrows) {
    b->rp = malloc(sizeof(i64) * (nrows + 1)); b->rp[0] = 0; b->rows = 0;
    b->cap = 1024; b->used = 0; b->ci = malloc(sizeof(int) * b->cap); b->v = malloc(sizeof(double) * b->cap);
}
static void b_done(Builder *b, OCsr *A) { A->n = b->rows; A->nnz = b->used; A->rp = b->rp; A->ci = b->ci; A->v = b->v; }

void orc_coupled_destroy(OCoupled *c) {
    if (!c) return;
    orc_destroy(c->vel); orc_destroy(c->eb);
    oc_free(&c->A); oc_free(&c->Mup); oc_free(&c->K); oc_free(&c->Bt);
    free(c);
}

OCoupled *orc_coupled_create(int dim, int N, int nlev, const double *dparams, const int *iparams, const double *w,
                             const double *bn) {
    OCoupled *c = calloc(1, sizeof(OCoupled));
    c->vel = orc_create_masked(ORC_VEL, dim, N, nlev, dparams, iparams, w, NULL, bn);
    c->eb = orc_create_masked(ORC_EB, dim, N, nlev, dparams, iparams, w, NULL, bn);
    if (!c->vel || !c->eb) { orc_coupled_destroy(c); return NULL; }
    int top = nlev - 1;
    OLevel *Lv = &c->vel->lv[top], *Le = &c->eb->lv[top];
    OParams p = c->vel->p;
    p.bn = Lv->bn;
    OCsr J, Dt, G, B;
    double *fu = calloc((size_t)Lv->A.n, sizeof(double)), *fE = calloc((size_t)Le->A.n, sizeof(double));
    for (i64 i = 0; i < Lv->A.n; i++)
        for (i64 t = Lv->A.rp[i]; t < Lv->A.rp[i + 1]; t++) if (fabs(Lv->A.v[t]) > fu[i]) fu[i] = fabs(Lv->A.v[t]);
    for (i64 i = 0; i < Le->A.n; i++)
        for (i64 t = Le->A.rp[i]; t < Le->A.rp[i + 1]; t++) if (fabs(Le->A.v[t]) > fE[i]) fE[i] = fabs(Le->A.v[t]);
    oa_assemble_coupling(&c->Bt, &J, &Dt, &G, &Lv->m, &Lv->s, &Le->s, &p, Lv->w, Lv->bn, fu, fE);
    free(fu); free(fE);
    oc_transpose(&B, &c->Bt, Lv->m.nc);
    c->nu = Lv->s.n; c->np = Lv->m.nc; c->nE = Le->s.nE; c->nB = Le->s.n - Le->s.nE;
    c->n = c->nu + c->np + c->nE + c->nB;
    c->cS = -(1.0 / p.Re + p.gamma);
    c->Kinv = dim == 2 ? 2.0 * N * N : 6.0 * (double)N * N * N;
    i64 su = 0, sp = c->nu, sE = c->nu + c->np, sB = sE + c->nE;
    Builder bA, bM, bK;
    b_init(&bA, c->n); b_init(&bM, c->nu + c->np); b_init(&bK, c->nu);
    for (i64 i = 0; i < c->nu; i++) {
        b_push(&bA, &Lv->A, i, su); b_push(&bA, &c->Bt, i, sp); b_push(&bA, &J, i, sE); b_push(&bA, &Dt, i, sB);
        b_endrow(&bA);
        b_push(&bM, &Lv->A, i, 0); b_push(&bM, &c->Bt, i, c->nu); b_endrow(&bM);
        b_push(&bK, &J, i, 0); b_push(&bK, &Dt, i, c->nE); b_endrow(&bK);
    }
    for (i64 q = 0; q < c->np; q++) {
        b_push(&bA, &B, q, su); b_endrow(&bA);
        b_push(&bM, &B, q, 0); b_endrow(&bM);
    }
    for (i64 e = 0; e < c->nE; e++) { b_push(&bA, &G, e, su); b_push(&bA, &Le->A, e, sE); b_endrow(&bA); }
    for (i64 k = 0; k < c->nB; k++) { b_push(&bA, &Le->A, c->nE + k, sE); b_endrow(&bA); }
    b_done(&bA, &c->A); b_done(&bM, &c->Mup); b_done(&bK, &c->K);
    oc_free(&J); oc_free(&Dt); oc_free(&G); oc_free(&B);
    return c;
}

/* generic right-preconditioned flexible GMRES; fixed != 0: exactly m iterations (stop
 * only at breakdown), else stop when |g_k+1| <= max(rtol |b|, atol).  Returns 0/1/2 as
 * orc_fgmres; hist may be NULL.                                                      */
typedef int (*opfn)(void *, const double *, double *);
static int fgmres_gen(i64 n, opfn A, void *ac, opfn P, void *pc, const double *b, double *x, int m, int fixed,
                      double rtol, double atol, int *its_out, double *hist) {
    double beta = sqrt(od_dot(b, b, n));
    double tol = rtol * beta > atol ? rtol * beta : atol;
    for (i64 i = 0; i < n; i++) x[i] = 0.0;
    if (hist) hist[0] = beta;
    if (its_out) *its_out = 0;
    if (beta == 0.0 || (!fixed && beta <= tol)) return 0;
    double *V = malloc(sizeof(double) * n * (m + 1)), *Z = malloc(sizeof(double) * n * m), *w = malloc(sizeof(double) * n);
    double *H = calloc((size_t)(m + 1) * m, sizeof(double)), *cs = calloc(m, sizeof(double)),
           *sn = calloc(m, sizeof(double)), *g = calloc(m + 1, sizeof(double)), *y = calloc(m, sizeof(double));
    for (i64 i = 0; i < n; i++) V[i] = b[i] / beta;
    g[0] = beta;
    int k, conv = 0, fail = 0;
    for (k = 0; k < m; k++) {
        if (P(pc, V + k * n, Z + k * n)) { fail = 1; break; }
        A(ac, Z + k * n, w);
        for (int i = 0; i <= k; i++) {
            double h = od_dot(w, V + i * n, n);
            H[i * m + k] = h;
            for (i64 j = 0; j < n; j++) w[j] = fma(-h, V[i * n + j], w[j]);
        }
        double hn = sqrt(od_dot(w, w, n));
        H[(k + 1) * m + k] = hn;
        givens_column(H, m, cs, sn, g, k);
        if (hist) hist[k + 1] = fabs(g[k + 1]);
        if (!fixed && fabs(g[k + 1]) <= tol) { k++; conv = 1; break; }
        if (hn == 0.0) { k++; break; }
        if (k + 1 < m) for (i64 j = 0; j < n; j++) V[(k + 1) * n + j] = w[j] / hn;
    }
    if (!fail) {
        back_substitute(H, m, g, k, y);
        for (int i = 0; i < k; i++)
            for (i64 j = 0; j < n; j++) x[j] = fma(y[i], Z[i * n + j], x[j]);
        if (its_out) *its_out = k;
    }
    free(V); free(Z); free(w); free(H); free(cs); free(sn); free(g); free(y);
    return fail ? 2 : (conv || fixed ? 0 : 1);
}

static int op_csr(void *a, const double *x, double *y) { csr_chain((const OCsr *)a, x, y); return 0; }
static int op_eb_vcycle(void *cc, const double *r, double *z) {
    OCoupled *c = cc;
    return vcycle(c->eb, c->eb->nlev - 1, r, z);
}
static int op_eb_A(void *cc, const double *x, double *y) {
    OCoupled *c = cc;
    csr_chain(&c->eb->lv[c->eb->nlev - 1].A, x, y);
    return 0;
}
/* hydrodynamic block preconditioner Q: y_p = (cS s_p) Kinv;  y_u = V_u(s_u - B^T y_p) */
static int op_hydro(void *cc, const double *s, double *y) {
    OCoupled *c = cc;
    double *yp = y + c->nu, *t = malloc(sizeof(double) * c->nu);
    for (i64 q = 0; q < c->np; q++) yp[q] = (c->cS * s[c->nu + q]) * c->Kinv;
    for (i64 i = 0; i < c->nu; i++) {
        double acc = 0.0;
        for (i64 k = c->Bt.rp[i]; k < c->Bt.rp[i + 1]; k++) acc = fma(c->Bt.v[k], yp[c->Bt.ci[k]], acc);
        t[i] = s[i] - acc;
    }
    int st = vcycle(c->vel, c->vel->nlev - 1, t, y);
    free(t);
    return st;
}
static int op_Mup(void *cc, const double *x, double *y) { csr_chain(&((OCoupled *)cc)->Mup, x, y); return 0; }

/* the block upper-triangular preconditioner (R-outer) */
int orc_coupled_precondition(OCoupled *c, const double *r, double *y) {
    i64 nup = c->nu + c->np, neb = c->nE + c->nB;
    const double *rEB = r + nup;
    double *yEB = y + nup;
    if (fgmres_gen(neb, op_eb_A, c, op_eb_vcycle, c, rEB, yEB, 2, 1, 0, 0, NULL, NULL)) return 1;
    double *z = malloc(sizeof(double) * nup);
    for (i64 i = 0; i < c->nu; i++) {
        double acc = 0.0;
        for (i64 k = c->K.rp[i]; k < c->K.rp[i + 1]; k++) acc = fma(c->K.v[k], yEB[c->K.ci[k]], acc);
        z[i] = r[i] - acc;
    }
    for (i64 q = 0; q < c->np; q++) z[c->nu + q] = r[c->nu + q];
    int st = fgmres_gen(nup, op_Mup, c, op_hydro, c, z, y, 2, 1, 0, 0, NULL, NULL) ? 1 : 0;
    free(z);
    return st;
}
static int op_prec(void *cc, const double *r, double *y) { return orc_coupled_precondition((OCoupled *)cc, r, y); }

int orc_coupled_apply(OCoupled *c, const double *x, double *y) { csr_chain(&c->A, x, y); return 0; }

int orc_coupled_fgmres(OCoupled *c, const double *b, double *x, double rtol, double atol, int maxit, int *its,
                       double *hist) {
    return fgmres_gen(c->n, op_csr, &c->A, op_prec, c, b, x, maxit, 0, rtol, atol, its, hist);
}

void orc_coupled_sizes(const OCoupled *c, i64 *out) {
    out[0] = c->nu; out[1] = c->np; out[2] = c->nE; out[3] = c->nB; out[4] = c->A.nnz;
}
int orc_coupled_export(const OCoupled *c, i64 *rp, int *ci, double *v) {
    memcpy(rp, c->A.rp, sizeof(i64) * (c->n + 1));
    memcpy(ci, c->A.ci, sizeof(int) * c->A.nnz);
    memcpy(v, c->A.v, sizeof(double) * c->A.nnz);
    return 0;
}
void orc_coupled_set_smoother(OCoupled *c, int kind, int its) {
    orc_set_smoother(c->vel, kind, its);
    orc_set_smoother(c->eb, kind, its);
}
