/*
 * space.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Free DoFs and vertex-star patches.
 *   - Spaces: E in CG1 (2D) / NED1_1 (3D), B in RT_1, velocity in
 *     BDM_1.  Boundary conditions E=0 / E x n = 0, B.n = 0, u.n = 0 imposed
 *     strongly by removing the constrained DoFs (reading R-bc).
 *   - Free-DoF order (reading R-num): E-B: free E DoFs in entity order, then free
 *     B DoFs in facet order.  Velocity: free facets in order, the `dim` DoFs of one
 *     facet contiguous, ordered by the facet's ascending vertices.
 *   - Patches (P:567-571 eq. stardecomp): V_i = { v in V_h : supp v subset K_i },
 *     K_i = the cells sharing vertex i.  One patch per vertex in ascending order,
 *     empty patches dropped (reading R-patch / SURVEY A1).  A free DoF lies in
 *     V_i iff its entity contains vertex i.
 */
#include <stdlib.h>
#include <string.h>
#include "orc.h"

/* k = 2 velocity (BDM2, 2D; reading R-num2): 3 DoFs per interior facet (facet order; sub
 * 0/1 = |f| u.n at the lower/higher vertex, 2 = at the midpoint), then 3 per cell (cell
 * order; sub e = moment against the Whitney function of local edge e).                  */
static int os_build2_vel(OSpace *s, const OMesh *m) {
    s->vdof = malloc(sizeof(int) * m->nv);
    s->edof = malloc(sizeof(int) * m->ne);
    s->fdof = malloc(sizeof(int) * m->nfacet);
    s->cdof = malloc(sizeof(int) * m->nc);
    for (i64 v = 0; v < m->nv; v++) s->vdof[v] = -1;
    for (i64 e = 0; e < m->ne; e++) s->edof[e] = -1;
    i64 n = 0;
    const int per = m->dim == 2 ? 3 : 6;      /* P2 on a facet: 3 (edge) / 6 (triangle); cell: 3 / 6 */
    for (i64 f = 0; f < m->nfacet; f++) { s->fdof[f] = m->fcell[2 * f + 1] >= 0 ? (int)n : -1; if (s->fdof[f] >= 0) n += per; }
    for (i64 c = 0; c < m->nc; c++) { s->cdof[c] = (int)n; n += per; }
    s->n = n;
    s->dkind = malloc(sizeof(int) * (n ? n : 1));
    s->dent = malloc(sizeof(int) * (n ? n : 1));
    s->dsub = malloc(sizeof(int) * (n ? n : 1));
    for (i64 f = 0; f < m->nfacet; f++)
        if (s->fdof[f] >= 0)
            for (int a = 0; a < per; a++) { s->dkind[s->fdof[f] + a] = 2; s->dent[s->fdof[f] + a] = (int)f; s->dsub[s->fdof[f] + a] = a; }
    for (i64 c = 0; c < m->nc; c++)
        for (int a = 0; a < per; a++) { s->dkind[s->cdof[c] + a] = 3; s->dent[s->cdof[c] + a] = (int)c; s->dsub[s->cdof[c] + a] = a; }
    return 0;
}

/* k = 2 in 3D, E-B block (NED1_2 x RT2; reading R-num2): E: 2 DoFs per free edge (edge
 * order; sub 0/1 = moment against lambda of the lower/higher vertex), then 2 per interior
 * face (face order; sub s = moment against the tangent x_{v_{s+1}} - x_{v_0}); B: 3 per
 * interior face (face order; sub s = moment against lambda of the s-th face vertex), then
 * 3 per cell (cell order; sub r = component).  Boundary DoFs removed (R-bc).           */
static int os_build2_eb3(OSpace *s, const OMesh *m) {
    s->vdof = malloc(sizeof(int) * m->nv);
    s->edof = malloc(sizeof(int) * m->ne);
    s->fdof = malloc(sizeof(int) * m->nfacet);
    s->gdof = malloc(sizeof(int) * m->nfacet);
    s->cdof = malloc(sizeof(int) * m->nc);
    for (i64 v = 0; v < m->nv; v++) s->vdof[v] = -1;
    i64 n = 0;
    for (i64 e = 0; e < m->ne; e++) { s->edof[e] = m->ebnd[e] ? -1 : (int)n; if (s->edof[e] >= 0) n += 2; }
    for (i64 f = 0; f < m->nfacet; f++) { s->gdof[f] = m->fcell[2 * f + 1] >= 0 ? (int)n : -1; if (s->gdof[f] >= 0) n += 2; }
    s->nE = n;
    for (i64 f = 0; f < m->nfacet; f++) { s->fdof[f] = m->fcell[2 * f + 1] >= 0 ? (int)n : -1; if (s->fdof[f] >= 0) n += 3; }
    for (i64 c = 0; c < m->nc; c++) { s->cdof[c] = (int)n; n += 3; }
    s->n = n;
    s->dkind = malloc(sizeof(int) * (n ? n : 1));
    s->dent = malloc(sizeof(int) * (n ? n : 1));
    s->dsub = malloc(sizeof(int) * (n ? n : 1));
    for (i64 e = 0; e < m->ne; e++)
        if (s->edof[e] >= 0)
            for (int a = 0; a < 2; a++) { s->dkind[s->edof[e] + a] = 1; s->dent[s->edof[e] + a] = (int)e; s->dsub[s->edof[e] + a] = a; }
    for (i64 f = 0; f < m->nfacet; f++) {
        if (s->gdof[f] >= 0)
            for (int a = 0; a < 2; a++) { s->dkind[s->gdof[f] + a] = 4; s->dent[s->gdof[f] + a] = (int)f; s->dsub[s->gdof[f] + a] = a; }
        if (s->fdof[f] >= 0)
            for (int a = 0; a < 3; a++) { s->dkind[s->fdof[f] + a] = 2; s->dent[s->fdof[f] + a] = (int)f; s->dsub[s->fdof[f] + a] = a; }
    }
    for (i64 c = 0; c < m->nc; c++)
        for (int a = 0; a < 3; a++) { s->dkind[s->cdof[c] + a] = 3; s->dent[s->cdof[c] + a] = (int)c; s->dsub[s->cdof[c] + a] = a; }
    return 0;
}

/* k = 2 (NEXT-2; reading R-num2): 2D E-B.  E (CG2): free vertex DoFs in
 * vertex order, then free edge-midpoint DoFs in edge order; B (RT2): 2 DoFs per interior
 * edge (edge order; sub 0/1 = moment against lambda of the lower/higher vertex), then 2
 * DoFs per cell (cell order; sub r = component).  Boundary DoFs removed (R-bc).    */
static int os_build2(OSpace *s, const OMesh *m) {
    s->vdof = malloc(sizeof(int) * m->nv);
    s->edof = malloc(sizeof(int) * m->ne);
    s->fdof = malloc(sizeof(int) * m->nfacet);
    s->cdof = malloc(sizeof(int) * m->nc);
    i64 n = 0;
    for (i64 v = 0; v < m->nv; v++) s->vdof[v] = m->vbnd[v] ? -1 : (int)n++;
    for (i64 e = 0; e < m->ne; e++) s->edof[e] = m->ebnd[e] ? -1 : (int)n++;
    s->nE = n;
    for (i64 f = 0; f < m->nfacet; f++) { s->fdof[f] = m->fcell[2 * f + 1] >= 0 ? (int)n : -1; if (s->fdof[f] >= 0) n += 2; }
    for (i64 c = 0; c < m->nc; c++) { s->cdof[c] = (int)n; n += 2; }
    s->n = n;
    s->dkind = malloc(sizeof(int) * (n ? n : 1));
    s->dent = malloc(sizeof(int) * (n ? n : 1));
    s->dsub = malloc(sizeof(int) * (n ? n : 1));
    for (i64 v = 0; v < m->nv; v++) if (s->vdof[v] >= 0) { s->dkind[s->vdof[v]] = 0; s->dent[s->vdof[v]] = (int)v; s->dsub[s->vdof[v]] = 0; }
    for (i64 e = 0; e < m->ne; e++) if (s->edof[e] >= 0) { s->dkind[s->edof[e]] = 1; s->dent[s->edof[e]] = (int)e; s->dsub[s->edof[e]] = 0; }
    for (i64 f = 0; f < m->nfacet; f++)
        if (s->fdof[f] >= 0)
            for (int a = 0; a < 2; a++) { s->dkind[s->fdof[f] + a] = 2; s->dent[s->fdof[f] + a] = (int)f; s->dsub[s->fdof[f] + a] = a; }
    for (i64 c = 0; c < m->nc; c++)
        for (int a = 0; a < 2; a++) { s->dkind[s->cdof[c] + a] = 3; s->dent[s->cdof[c] + a] = (int)c; s->dsub[s->cdof[c] + a] = a; }
    return 0;
}

int os_build(OSpace *s, const OMesh *m, int block, int degree) {
    memset(s, 0, sizeof(*s));
    s->block = block; s->dim = m->dim; s->degree = degree;
    if (degree == 2) {
        if (m->dim == 3) return block == ORC_EB ? os_build2_eb3(s, m) : os_build2_vel(s, m);
        return block == ORC_EB ? os_build2(s, m) : os_build2_vel(s, m);
    }
    if (degree != 1) return 1;
    s->vdof = malloc(sizeof(int) * m->nv);
    s->edof = malloc(sizeof(int) * m->ne);
    s->fdof = malloc(sizeof(int) * m->nfacet);
    for (i64 v = 0; v < m->nv; v++) s->vdof[v] = -1;
    for (i64 e = 0; e < m->ne; e++) s->edof[e] = -1;
    for (i64 f = 0; f < m->nfacet; f++) s->fdof[f] = -1;
    i64 n = 0;
    if (block == ORC_EB) {
        if (m->dim == 2) {
            for (i64 v = 0; v < m->nv; v++) if (!m->vbnd[v]) s->vdof[v] = (int)n++;
        } else {
            for (i64 e = 0; e < m->ne; e++) if (!m->ebnd[e]) s->edof[e] = (int)n++;
        }
        s->nE = n;
        for (i64 f = 0; f < m->nfacet; f++) if (m->fcell[2 * f + 1] >= 0) s->fdof[f] = (int)n++;
    } else {
        for (i64 f = 0; f < m->nfacet; f++)
            if (m->fcell[2 * f + 1] >= 0) { s->fdof[f] = (int)n; n += m->dim; }
    }
    s->n = n;
    s->dkind = malloc(sizeof(int) * n);
    s->dent = malloc(sizeof(int) * n);
    s->dsub = malloc(sizeof(int) * n);
    for (i64 v = 0; v < m->nv; v++) if (s->vdof[v] >= 0) { s->dkind[s->vdof[v]] = 0; s->dent[s->vdof[v]] = (int)v; s->dsub[s->vdof[v]] = 0; }
    for (i64 e = 0; e < m->ne; e++) if (s->edof[e] >= 0) { s->dkind[s->edof[e]] = 1; s->dent[s->edof[e]] = (int)e; s->dsub[s->edof[e]] = 0; }
    int nsub = block == ORC_VEL ? m->dim : 1;
    for (i64 f = 0; f < m->nfacet; f++)
        if (s->fdof[f] >= 0)
            for (int a = 0; a < nsub; a++) {
                s->dkind[s->fdof[f] + a] = 2; s->dent[s->fdof[f] + a] = (int)f; s->dsub[s->fdof[f] + a] = a;
            }
    return 0;
}

void os_free(OSpace *s) {
    free(s->vdof); free(s->edof); free(s->fdof); free(s->cdof); free(s->gdof); free(s->dkind); free(s->dent);
    free(s->dsub);
    memset(s, 0, sizeof(*s));
}

/* does the entity of free DoF d contain vertex v? */
static int dof_contains_vertex(const OMesh *m, const OSpace *s, int d, int v) {
    int e = s->dent[d];
    switch (s->dkind[d]) {
    case 0: return e == v;
    case 1: return m->ev[2 * e] == v || m->ev[2 * e + 1] == v;
    case 4: return m->fv[3 * e] == v || m->fv[3 * e + 1] == v || m->fv[3 * e + 2] == v;
    case 3: {
        int nvc = m->dim + 1;
        for (int q = 0; q < nvc; q++) if (m->cv[(i64)e * nvc + q] == v) return 1;
        return 0;
    }
    default:
        if (m->dim == 2) return m->ev[2 * e] == v || m->ev[2 * e + 1] == v;
        return m->fv[3 * e] == v || m->fv[3 * e + 1] == v || m->fv[3 * e + 2] == v;
    }
}

static int cmp_int(const void *a, const void *b) {
    int x = *(const int *)a, y = *(const int *)b;
    return x < y ? -1 : x > y;
}

/* Patch of vertex v: every free DoF of every cell of the star of v whose entity
 * contains v.  Built from the vertex -> cells incidence.                 */
int opt_build(OPatches *pt, const OMesh *m, const OSpace *s) {
    memset(pt, 0, sizeof(*pt));
    int nvc = m->dim + 1, nle = om_nle(m->dim);
    /* vertex -> cells */
    i64 *vcp = calloc((size_t)m->nv + 1, sizeof(i64));
    for (i64 c = 0; c < m->nc; c++) for (int q = 0; q < nvc; q++) vcp[m->cv[c * nvc + q] + 1]++;
    for (i64 v = 0; v < m->nv; v++) vcp[v + 1] += vcp[v];
    int *vc = malloc(sizeof(int) * vcp[m->nv]);
    i64 *fill = calloc((size_t)m->nv, sizeof(i64));
    for (i64 c = 0; c < m->nc; c++)
        for (int q = 0; q < nvc; q++) { int v = m->cv[c * nvc + q]; vc[vcp[v] + fill[v]++] = (int)c; }
    free(fill);

    int maxloc = 64 * 24;
    int *buf = malloc(sizeof(int) * maxloc);
    i64 cap = 1024, used = 0;
    pt->dofs = malloc(sizeof(int) * cap);
    pt->vert = malloc(sizeof(int) * m->nv);
    pt->ptr = malloc(sizeof(i64) * (m->nv + 1));
    pt->ptr[0] = 0;
    i64 np = 0;
    for (i64 v = 0; v < m->nv; v++) {
        int nb = 0;
        for (i64 t = vcp[v]; t < vcp[v + 1]; t++) {
            i64 c = vc[t];
            /* all free DoFs of cell c */
            int cand[64]; int nc = 0;
            if (s->degree == 2 && m->dim == 3 && s->block == ORC_EB) {   /* NED1_2 x RT2 (3D) */
                for (int q = 0; q < 6; q++) { int d = s->edof[m->ce[c * 6 + q]]; if (d >= 0) { cand[nc++] = d; cand[nc++] = d + 1; } }
                for (int q = 0; q < 4; q++) {
                    int f = om_facet_of_cell(m, c, q);
                    if (s->gdof[f] >= 0) { cand[nc++] = s->gdof[f]; cand[nc++] = s->gdof[f] + 1; }
                    if (s->fdof[f] >= 0) for (int a = 0; a < 3; a++) cand[nc++] = s->fdof[f] + a;
                }
                for (int a = 0; a < 3; a++) cand[nc++] = s->cdof[c] + a;
            } else if (s->degree == 2 && s->block == ORC_VEL) {   /* BDM2: 3 (2D) / 6 (3D) per facet and cell */
                int per = m->dim == 2 ? 3 : 6;
                for (int q = 0; q < nvc; q++) {
                    int d = s->fdof[om_facet_of_cell(m, c, q)];
                    if (d >= 0) for (int a = 0; a < per; a++) cand[nc++] = d + a;
                }
                for (int a = 0; a < per; a++) cand[nc++] = s->cdof[c] + a;
            } else if (s->degree == 2) {                    /* CG2 x RT2 (2D) */
                for (int q = 0; q < 3; q++) { int d = s->vdof[m->cv[c * 3 + q]]; if (d >= 0) cand[nc++] = d; }
                for (int q = 0; q < 3; q++) { int d = s->edof[m->ce[c * 3 + q]]; if (d >= 0) cand[nc++] = d; }
                for (int q = 0; q < 3; q++) {
                    int d = s->fdof[om_facet_of_cell(m, c, q)];
                    if (d >= 0) { cand[nc++] = d; cand[nc++] = d + 1; }
                }
                cand[nc++] = s->cdof[c]; cand[nc++] = s->cdof[c] + 1;
            } else if (s->block == ORC_EB) {
                if (m->dim == 2) for (int q = 0; q < 3; q++) { int d = s->vdof[m->cv[c * 3 + q]]; if (d >= 0) cand[nc++] = d; }
                else for (int q = 0; q < nle; q++) { int d = s->edof[m->ce[c * nle + q]]; if (d >= 0) cand[nc++] = d; }
                for (int q = 0; q < nvc; q++) { int d = s->fdof[om_facet_of_cell(m, c, q)]; if (d >= 0) cand[nc++] = d; }
            } else {
                for (int q = 0; q < nvc; q++) {
                    int d = s->fdof[om_facet_of_cell(m, c, q)];
                    if (d >= 0) for (int a = 0; a < m->dim; a++) cand[nc++] = d + a;
                }
            }
            for (int u = 0; u < nc; u++)
                if (dof_contains_vertex(m, s, cand[u], (int)v)) buf[nb++] = cand[u];
        }
        qsort(buf, (size_t)nb, sizeof(int), cmp_int);
        int nu = 0;
        for (int u = 0; u < nb; u++) if (u == 0 || buf[u] != buf[u - 1]) buf[nu++] = buf[u];
        if (nu == 0) continue;
        while (used + nu > cap) { cap *= 2; pt->dofs = realloc(pt->dofs, sizeof(int) * cap); }
        memcpy(pt->dofs + used, buf, sizeof(int) * nu);
        used += nu;
        pt->vert[np] = (int)v;
        pt->ptr[++np] = used;
    }
    pt->np = np;
    free(buf); free(vcp); free(vc);
    /* multiplicities and DoF -> slot lists (ascending patch order) */
    i64 n = s->n;
    pt->mult = calloc((size_t)n, sizeof(int));
    for (i64 t = 0; t < used; t++) pt->mult[pt->dofs[t]]++;
    pt->mmax = 0;
    for (i64 d = 0; d < n; d++) if (pt->mult[d] > pt->mmax) pt->mmax = pt->mult[d];
    pt->dptr = calloc((size_t)n + 1, sizeof(i64));
    for (i64 d = 0; d < n; d++) pt->dptr[d + 1] = pt->dptr[d] + pt->mult[d];
    pt->dslot = malloc(sizeof(i64) * (used ? used : 1));
    i64 *f2 = calloc((size_t)n, sizeof(i64));
    for (i64 t = 0; t < used; t++) { int d = pt->dofs[t]; pt->dslot[pt->dptr[d] + f2[d]++] = t; }
    free(f2);
    return 0;
}

void opt_free(OPatches *pt) {
    free(pt->vert); free(pt->ptr); free(pt->dofs); free(pt->mult); free(pt->dptr); free(pt->dslot);
    memset(pt, 0, sizeof(*pt));
}
