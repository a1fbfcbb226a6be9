/*
 * orc.h -- internal declarations of the ORACLE.
 *
 * TEST INFRASTRUCTURE ONLY.  The oracle is a plain, slow, single-threaded C
 * implementation of the vertex-star Schwarz smoother and V-cycle of
 * arXiv 2104.14855 (§3.3-§3.5, §4.1).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.  It shares no
 * code, header, table or constant generator with paper_2104_14855_b200/ (the
 * product path), and never reads anything produced by it.
 *
 * Every function cites the PAPER.md passage (P:line) or the DESIGN.md reading
 * (R-xx, which restate SURVEY.md §8(c) readings A1-A26) it follows.
 */
#ifndef ORC_H
#define ORC_H

#include <stddef.h>

typedef long long i64;

/* ---------------- mesh (P:572 nested uniform hierarchy; R-mesh) ---------------- */
typedef struct {
    int dim, N;            /* unit square/cube, N cells per side                     */
    i64 nv, ne, nf, nc;    /* vertices, edges, faces (3D only), cells               */
    i64 nfacet;            /* facets: edges (2D) or faces (3D)                        */
    int *lat;              /* nv*3 integer lattice coordinates (i,j,k)                */
    double *x;             /* nv*3 physical coordinates lat/N                         */
    int *cv;               /* nc*(dim+1) cell vertices, ascending global id           */
    int *ev;               /* ne*2 sorted                                             */
    int *fv;               /* nf*3 sorted (3D)                                        */
    int *ce;               /* nc*nle : local edge -> global edge                      */
    int *cf;               /* nc*4   : local face -> global face (3D)                 */
    int *fcell;            /* nfacet*2 : adjacent cells, [0] < [1], [1] = -1 on bdry   */
    unsigned char *vbnd;   /* nv : vertex on the boundary                              */
    unsigned char *ebnd;   /* ne : edge constrained (2D: boundary edge; 3D: edge of a boundary face) */
} OMesh;

int  om_build(OMesh *m, int dim, int N);
void om_free(OMesh *m);
int  om_nle(int dim);                   /* local edges per cell                    */
int  om_facet_of_cell(const OMesh *m, i64 c, int q);  /* global facet id of local facet q */
/* local facet q of a cell is opposite local vertex opp(q) */
int  om_facet_opp(int dim, int q);
void om_facet_local_verts(int dim, int q, int *lv);  /* the dim local vertices of facet q, ascending */
void om_edge_local_verts(int dim, int q, int *lv);   /* 2 local vertices of local edge q          */
i64  om_find_edge(const OMesh *m, int a, int b);
i64  om_find_face(const OMesh *m, int a, int b, int c);

/* ---------------- spaces / free DoFs (R-dofs) ---------------- */
enum { ORC_EB = 0, ORC_VEL = 1 };

typedef struct {
    int block, dim;
    int degree;            /* k = 1, or 2 (NEXT-2: 2D E-B block, CG2 x RT2, reading R-basis2) */
    i64 n;                 /* free DoFs                                                */
    i64 nE;                /* E-B: number of free E DoFs (they come first)             */
    /* global free index per entity (or -1 if constrained) */
    int *vdof;             /* nv (2D E)                                               */
    int *edof;             /* ne (3D E: NED1)                                          */
    int *fdof;             /* nfacet (B: RT)  or first velocity DoF of the facet (BDM: +0..dim-1);
                              k = 2: first of the 2 RT2 DoFs of the edge                */
    int *cdof;             /* nc (k = 2 only): first interior DoF of the cell (RT2: 2 in 2D, 3 in 3D) */
    int *gdof;             /* nfacet (3D E-B k = 2 only): first of the 2 NED1_2 face DoFs       */
    /* per free DoF: entity kind (0 vertex, 1 edge, 2 facet, 3 cell, 4 facet of the E field
       in 3D k = 2), entity id, sub index                                                 */
    int *dkind, *dent, *dsub;
} OSpace;

int  os_build(OSpace *s, const OMesh *m, int block, int degree);   /* 0, or 1 if unsupported */
void os_free(OSpace *s);

/* ---------------- CSR ---------------- */
typedef struct {
    i64 n, nnz;
    i64 *rp;
    int *ci;
    double *v;
} OCsr;
void oc_free(OCsr *a);
i64  oc_find(const OCsr *a, i64 row, int col);   /* position of (row,col) or -1 */

/* ---------------- parameters ---------------- */
typedef struct {
    double Re, Rem, S, gamma, sigma, mu;
    int nu_pre, nu_post;
    double dt;     /* NEXT-4: > 0 -> transient (eta = 1): (1/dt) mass terms */
    int picard;    /* NEXT-4: 1 -> Picard linearisation (delta = 0): no G~ term    */
    const double *bn;  /* NEXT-4: potential of B^n at this level's vertices (as w, R-w), or NULL:
                          velocity block + S (B^n x (u x B^n), v) = S (u x B^n, v x B^n) */
} OParams;

/* ---------------- operator assembly ---------------- */
/* w: potential of the advecting field at THIS level's vertices (R-w): 2D stream
 * function (1 per vertex), 3D vector potential (3 per vertex). */
int oa_assemble(OCsr *A, const OMesh *m, const OSpace *s, const OParams *p, const double *w);
/* as oa_assemble, but only cells with cmask[c] != 0 (and facets touching one) contribute;
 * rows whose support neighbourhood lies inside the mask are bitwise identical to oa_assemble
 * (the row rounding of R-exact depends on the row only) */
int oa_assemble_masked(OCsr *A, const OMesh *m, const OSpace *s, const OParams *p, const double *w,
                       const unsigned char *cmask);

/* NEXT-3 coupling blocks of the 4x4 system on one mesh (see fem.c) */
int oa_assemble_coupling(OCsr *Bt, OCsr *J, OCsr *Dt, OCsr *G, const OMesh *m, const OSpace *sv, const OSpace *se,
                         const OParams *p, const double *w, const double *bn, const double *floor_u,
                         const double *floor_E);   /* row floors of the grid (R-cgrid), or NULL */

/* quadrature / load / evaluation (manufactured-solution pins only) */
int  oa_ncomp(const OSpace *s);
int  oa_nq(int dim);
void oa_quadrature(const OMesh *m, double *pts, double *wts);
void oa_load(const OMesh *m, const OSpace *s, const double *fv, double *out);
void oa_eval(const OMesh *m, const OSpace *s, const double *coef, double *fv);

double oa_duality_error(const OMesh *m, const OSpace *s);

/* ---------------- prolongation ---------------- */
int op_prolongation(OCsr *P, const OMesh *mf, const OSpace *sf, const OMesh *mc, const OSpace *sc);
int oc_transpose(OCsr *T, const OCsr *A, i64 ncols);

/* ---------------- patches ---------------- */
typedef struct {
    i64 np;                /* patches (non-empty vertex stars, ascending vertex)     */
    int *vert;             /* np : vertex id of the patch                            */
    i64 *ptr;              /* np+1 offsets into dofs                                  */
    int *dofs;             /* ascending global free indices                           */
    int *mult;             /* n : multiplicity m_d                                    */
    int mmax;              /* max_d m_d (R-weights2)                                   */
    /* DoF -> (slot) lists in ascending patch order */
    i64 *dptr;             /* n+1 */
    i64 *dslot;            /* positions into dofs[] (= slot index)                    */
} OPatches;
int  opt_build(OPatches *pt, const OMesh *m, const OSpace *s);
void opt_free(OPatches *pt);

/* ---------------- dense LU (R-lu) ---------------- */
/* a: n*n row-major, in/out. perm[k] = original row now at position k.
 * returns 0, or k+1 if |pivot| <= 1e-14 * amax at step k.                       */
int od_lu(double *a, int n, int *perm, double amax);
void od_lu_solve(const double *lu, int n, const int *perm, const double *r, double *z);
/* R-dot inner product (blocks of 256, fma chains from +0.0, pairwise tree) */
double od_dot(const double *a, const double *b, i64 n);

#endif
