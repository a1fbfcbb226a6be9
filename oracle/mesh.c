/*
 * mesh.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Structured triangulations of the unit square / cube and their entities.
 *   - Nested uniform hierarchy: P:572 ("the uniformly-refined mesh hierarchy we
 *     consider is nested").
 *   - 2D: every square split by the same bottom-left -> top-right diagonal
 *     (BASELINE.json config 1 "same diagonal"; reading R-mesh / SURVEY A16).
 *   - 3D: six Kuhn tetrahedra per cube (BASELINE.json configs 4-5 "split into 6
 *     tetrahedra"; reading R-mesh / SURVEY A17).
 *   - Edges / faces are the sorted vertex tuples occurring in cells, numbered in
 *     lexicographic order (reading R-num / SURVEY A15).  Implemented the obvious
 *     way: list every tuple, qsort, unique.
 */
#include <stdlib.h>
#include <string.h>
#include "orc.h"

static int vid(int N, int dim, int i, int j, int k) {
    return dim == 2 ? i + (N + 1) * j : i + (N + 1) * (j + (N + 1) * k);
}

static void sort_small(int *a, int n) {
    for (int i = 1; i < n; i++)
        for (int j = i; j > 0 && a[j - 1] > a[j]; j--) { int t = a[j]; a[j] = a[j - 1]; a[j - 1] = t; }
}

static int cmp2(const void *p, const void *q) {
    const int *a = p, *b = q;
    if (a[0] != b[0]) return a[0] < b[0] ? -1 : 1;
    if (a[1] != b[1]) return a[1] < b[1] ? -1 : 1;
    return 0;
}
static int cmp3(const void *p, const void *q) {
    const int *a = p, *b = q;
    for (int t = 0; t < 3; t++) if (a[t] != b[t]) return a[t] < b[t] ? -1 : 1;
    return 0;
}

int om_nle(int dim) { return dim == 2 ? 3 : 6; }

/* local edges: pairs of local (ascending) vertices in lexicographic order */
static const int LE2[3][2] = {{0, 1}, {0, 2}, {1, 2}};
static const int LE3[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
static const int LF3[4][3] = {{0, 1, 2}, {0, 1, 3}, {0, 2, 3}, {1, 2, 3}};

void om_edge_local_verts(int dim, int q, int *lv) {
    if (dim == 2) { lv[0] = LE2[q][0]; lv[1] = LE2[q][1]; }
    else { lv[0] = LE3[q][0]; lv[1] = LE3[q][1]; }
}

int om_facet_opp(int dim, int q) { return dim == 2 ? 2 - q : 3 - q; }

void om_facet_local_verts(int dim, int q, int *lv) {
    if (dim == 2) { lv[0] = LE2[q][0]; lv[1] = LE2[q][1]; }
    else { lv[0] = LF3[q][0]; lv[1] = LF3[q][1]; lv[2] = LF3[q][2]; }
}

i64 om_find_edge(const OMesh *m, int a, int b) {
    int key[2] = {a < b ? a : b, a < b ? b : a};
    int *r = bsearch(key, m->ev, (size_t)m->ne, 2 * sizeof(int), cmp2);
    return r ? (i64)((r - m->ev) / 2) : -1;
}

i64 om_find_face(const OMesh *m, int a, int b, int c) {
    int key[3] = {a, b, c};
    sort_small(key, 3);
    int *r = bsearch(key, m->fv, (size_t)m->nf, 3 * sizeof(int), cmp3);
    return r ? (i64)((r - m->fv) / 3) : -1;
}

int om_facet_of_cell(const OMesh *m, i64 c, int q) {
    return m->dim == 2 ? m->ce[c * 3 + q] : m->cf[c * 4 + q];
}

int om_build(OMesh *m, int dim, int N) {
    memset(m, 0, sizeof(*m));
    if ((dim != 2 && dim != 3) || N < 1) return 1;
    m->dim = dim; m->N = N;
    i64 np1 = N + 1;
    m->nv = dim == 2 ? np1 * np1 : np1 * np1 * np1;
    m->lat = malloc(sizeof(int) * 3 * m->nv);
    m->x = malloc(sizeof(double) * 3 * m->nv);
    m->vbnd = calloc((size_t)m->nv, 1);
    for (int k = 0; k < (dim == 2 ? 1 : N + 1); k++)
        for (int j = 0; j <= N; j++)
            for (int i = 0; i <= N; i++) {
                int v = vid(N, dim, i, j, k);
                m->lat[3 * v] = i; m->lat[3 * v + 1] = j; m->lat[3 * v + 2] = k;
                m->x[3 * v] = (double)i / N; m->x[3 * v + 1] = (double)j / N;
                m->x[3 * v + 2] = dim == 2 ? 0.0 : (double)k / N;
                int b = i == 0 || i == N || j == 0 || j == N;
                if (dim == 3) b = b || k == 0 || k == N;
                m->vbnd[v] = (unsigned char)b;
            }
    /* cells */
    int nvc = dim + 1;
    if (dim == 2) {
        m->nc = 2LL * N * N;
        m->cv = malloc(sizeof(int) * nvc * m->nc);
        for (int j = 0; j < N; j++)
            for (int i = 0; i < N; i++) {
                i64 s = i + (i64)N * j;
                int *t0 = m->cv + 3 * (2 * s), *t1 = m->cv + 3 * (2 * s + 1);
                /* T[2s] = (v(i,j), v(i+1,j), v(i+1,j+1)); T[2s+1] = (v(i,j), v(i+1,j+1), v(i,j+1)) */
                t0[0] = vid(N, 2, i, j, 0); t0[1] = vid(N, 2, i + 1, j, 0); t0[2] = vid(N, 2, i + 1, j + 1, 0);
                t1[0] = vid(N, 2, i, j, 0); t1[1] = vid(N, 2, i + 1, j + 1, 0); t1[2] = vid(N, 2, i, j + 1, 0);
                sort_small(t0, 3); sort_small(t1, 3);
            }
    } else {
        /* permutations of the axes in lexicographic order: 012 021 102 120 201 210 */
        static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        m->nc = 6LL * N * N * N;
        m->cv = malloc(sizeof(int) * nvc * m->nc);
        for (int k = 0; k < N; k++)
            for (int j = 0; j < N; j++)
                for (int i = 0; i < N; i++) {
                    i64 c = i + (i64)N * (j + (i64)N * k);
                    for (int p = 0; p < 6; p++) {
                        int *t = m->cv + 4 * (6 * c + p);
                        int cur[3] = {i, j, k};
                        t[0] = vid(N, 3, cur[0], cur[1], cur[2]);
                        for (int s = 0; s < 3; s++) {       /* walk x0 -> +e_s0 -> +e_s1 -> +e_s2 */
                            cur[PERM[p][s]] += 1;
                            t[s + 1] = vid(N, 3, cur[0], cur[1], cur[2]);
                        }
                        sort_small(t, 4);
                    }
                }
    }
    /* edges: all sorted pairs from cells, sorted lexicographically, unique */
    int nle = om_nle(dim);
    const int (*LE)[2] = dim == 2 ? LE2 : LE3;
    int *tmp = malloc(sizeof(int) * 2 * nle * m->nc);
    for (i64 c = 0; c < m->nc; c++)
        for (int q = 0; q < nle; q++) {
            tmp[2 * (c * nle + q)] = m->cv[c * nvc + LE[q][0]];
            tmp[2 * (c * nle + q) + 1] = m->cv[c * nvc + LE[q][1]];
        }
    qsort(tmp, (size_t)(nle * m->nc), 2 * sizeof(int), cmp2);
    i64 ne = 0;
    for (i64 t = 0; t < nle * m->nc; t++)
        if (t == 0 || cmp2(tmp + 2 * t, tmp + 2 * (t - 1)) != 0) {
            tmp[2 * ne] = tmp[2 * t]; tmp[2 * ne + 1] = tmp[2 * t + 1]; ne++;
        }
    m->ne = ne;
    m->ev = realloc(tmp, sizeof(int) * 2 * ne);
    m->ce = malloc(sizeof(int) * nle * m->nc);
    for (i64 c = 0; c < m->nc; c++)
        for (int q = 0; q < nle; q++)
            m->ce[c * nle + q] = (int)om_find_edge(m, m->cv[c * nvc + LE[q][0]], m->cv[c * nvc + LE[q][1]]);
    if (dim == 3) {
        int *tf = malloc(sizeof(int) * 3 * 4 * m->nc);
        for (i64 c = 0; c < m->nc; c++)
            for (int q = 0; q < 4; q++)
                for (int t = 0; t < 3; t++) tf[3 * (c * 4 + q) + t] = m->cv[c * 4 + LF3[q][t]];
        qsort(tf, (size_t)(4 * m->nc), 3 * sizeof(int), cmp3);
        i64 nf = 0;
        for (i64 t = 0; t < 4 * m->nc; t++)
            if (t == 0 || cmp3(tf + 3 * t, tf + 3 * (t - 1)) != 0) {
                for (int u = 0; u < 3; u++) tf[3 * nf + u] = tf[3 * t + u];
                nf++;
            }
        m->nf = nf;
        m->fv = realloc(tf, sizeof(int) * 3 * nf);
        m->cf = malloc(sizeof(int) * 4 * m->nc);
        for (i64 c = 0; c < m->nc; c++)
            for (int q = 0; q < 4; q++)
                m->cf[c * 4 + q] = (int)om_find_face(m, m->cv[c * 4 + LF3[q][0]], m->cv[c * 4 + LF3[q][1]],
                                                     m->cv[c * 4 + LF3[q][2]]);
    }
    m->nfacet = dim == 2 ? m->ne : m->nf;
    /* facet -> adjacent cells, ascending cell order */
    m->fcell = malloc(sizeof(int) * 2 * m->nfacet);
    for (i64 f = 0; f < 2 * m->nfacet; f++) m->fcell[f] = -1;
    for (i64 c = 0; c < m->nc; c++)
        for (int q = 0; q < dim + 1; q++) {
            int f = om_facet_of_cell(m, c, q);
            if (m->fcell[2 * f] < 0) m->fcell[2 * f] = (int)c;
            else m->fcell[2 * f + 1] = (int)c;
        }
    /* constrained edges: 2D boundary edges; 3D edges of boundary faces */
    m->ebnd = calloc((size_t)m->ne, 1);
    if (dim == 2) {
        for (i64 e = 0; e < m->ne; e++) m->ebnd[e] = m->fcell[2 * e + 1] < 0;
    } else {
        for (i64 f = 0; f < m->nf; f++)
            if (m->fcell[2 * f + 1] < 0) {
                const int *v = m->fv + 3 * f;
                m->ebnd[om_find_edge(m, v[0], v[1])] = 1;
                m->ebnd[om_find_edge(m, v[0], v[2])] = 1;
                m->ebnd[om_find_edge(m, v[1], v[2])] = 1;
            }
    }
    return 0;
}

void om_free(OMesh *m) {
    free(m->lat); free(m->x); free(m->cv); free(m->ev); free(m->fv); free(m->ce); free(m->cf);
    free(m->fcell); free(m->vbnd); free(m->ebnd);
    memset(m, 0, sizeof(*m));
}
