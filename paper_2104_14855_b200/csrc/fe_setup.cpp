// fe_setup.cpp -- host setup stage of libmhdp, product code.
//
// An implementation of the discretisation of arXiv 2104.14855 that is independent of
// the oracle (shares no code, different algorithms):
//   * meshes: structured closed forms.  Edges are the vertex pairs whose lattice
//     difference is a non-zero 0/1 vector (2D: (1,0),(0,1),(1,1); 3D Kuhn: all seven),
//     faces the chains a -> a+e1 -> a+e1+e2 with disjoint e1, e2; both are generated
//     directly in lexicographic order of their sorted vertex ids (R-num), so no sort.
//   * element integrals in closed form with barycentric moments
//     int_K lam_a lam_b = |K|(1+d_ab)/((d+1)(d+2)),  int_F mu_a mu_b = |F|(1+d_ab)/(d(d+1))
//     (every integrand is polynomial because the advecting field is constant per cell,
//     reading R-w), instead of quadrature;
//   * gather-form ("owner computes") assembly: each row block sums the contributions of
//     the cells / facets touching it in ascending order -- rows are independent, so the
//     loop is OpenMP-parallel and deterministic.
//
// Operators (trial j, test i):
//   E-B  (Table 1):
//        [[M_E, G~ - A/Rem], [A^T, C]],  G~_ik = (w x psi_k, phi_i), A_ik = (psi_k, vcurl phi_i),
//        C_kl = (1/Rem)(div psi_l, div psi_k)
//   AL velocity (reading R-vel): (2/Re)(eps u, eps v) + SIPG
//        (sigma = 10, h_F = edge length / longest face edge) - (u, div(v (x) w)) + upwind
//        facet terms with side-own normals + gamma (div u, div v).
// The grad-div / div-div entries use the exact closed form of reading R-gamma:
// (c * m) / d^2 with c = gamma d!N^d (or c = d!N^d / Rem with /1) and m the integer sum
// of orientation-sign products -- single-rounded, so both implementations agree bitwise.
#include <omp.h>

#include <algorithm>
#include <array>
#include <climits>
#include <cmath>
#include <cstring>
#include <numeric>

#include "ddreal.hpp"
#include "setup.hpp"

namespace mhdp {
namespace {

typedef int64_t i64;

// ------------------------------------------------------------------------------------
// structured mesh
// ------------------------------------------------------------------------------------
struct Mesh {
    int dim = 2, N = 1;
    i64 nv = 0, ne = 0, nf = 0, nc = 0, nfacet = 0;
    std::vector<int> ev;          // 2 per edge, sorted
    std::vector<i64> vedge;       // nv+1: edges whose first vertex is v
    std::vector<int> fv;          // 3 per face, sorted
    std::vector<i64> vface;       // nv+1: faces whose first vertex is v
    std::vector<int> cv;          // (dim+1) per cell, sorted ascending
    std::vector<int> cfacet;      // (dim+1) per cell: facet opposite local vertex q
    std::vector<int> cedge;       // 6 per cell (3D): local pairs (0,1)(0,2)(0,3)(1,2)(1,3)(2,3)
    std::vector<int> fcell;       // 2 per facet, ascending, -1 for none

    int side() const { return N + 1; }
    void lat(i64 v, int *ijk) const {
        const i64 s = N + 1;
        ijk[0] = (int)(v % s);
        ijk[1] = (int)((v / s) % s);
        ijk[2] = dim == 3 ? (int)(v / (s * s)) : 0;
    }
    i64 vid(int i, int j, int k) const { return i + (i64)(N + 1) * (j + (i64)(N + 1) * k); }
    bool on_bnd(i64 v) const {
        int p[3];
        lat(v, p);
        for (int a = 0; a < dim; ++a) if (p[a] == 0 || p[a] == N) return true;
        return false;
    }
    // lattice-plane test: do all given vertices lie on one boundary plane/line?
    bool common_bnd(const int *vs, int m) const {
        int p[4][3];
        for (int t = 0; t < m; ++t) lat(vs[t], p[t]);
        for (int a = 0; a < dim; ++a)
            for (int side = 0; side < 2; ++side) {
                const int val = side ? N : 0;
                bool all = true;
                for (int t = 0; t < m; ++t) all = all && p[t][a] == val;
                if (all) return true;
            }
        return false;
    }
    i64 edge_id(int a, int b) const {
        if (a > b) std::swap(a, b);
        for (i64 e = vedge[a]; e < vedge[a + 1]; ++e) if (ev[2 * e + 1] == b) return e;
        return -1;
    }
    i64 face_id(int a, int b, int c) const {
        int s[3] = {a, b, c};
        std::sort(s, s + 3);
        for (i64 f = vface[s[0]]; f < vface[s[0] + 1]; ++f)
            if (fv[3 * f + 1] == s[1] && fv[3 * f + 2] == s[2]) return f;
        return -1;
    }
    bool facet_interior(i64 f) const { return fcell[2 * f + 1] >= 0; }
};

// 0/1 offset vectors in ascending order of their vertex-id offset
static const int OFF2[3][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}};
static const int OFF3[7][3] = {{1, 0, 0}, {0, 1, 0}, {1, 1, 0}, {0, 0, 1}, {1, 0, 1}, {0, 1, 1}, {1, 1, 1}};

void build_mesh(Mesh &m, int dim, int N) {
    m.dim = dim; m.N = N;
    const i64 s = N + 1;
    m.nv = dim == 2 ? s * s : s * s * s;
    const int noff = dim == 2 ? 3 : 7;
    const int (*OFF)[3] = dim == 2 ? OFF2 : OFF3;
    // edges, lexicographic: for a ascending, b = a + off ascending
    m.vedge.assign(m.nv + 1, 0);
    m.ev.clear();
    for (i64 a = 0; a < m.nv; ++a) {
        int p[3];
        m.lat(a, p);
        for (int o = 0; o < noff; ++o) {
            int q[3] = {p[0] + OFF[o][0], p[1] + OFF[o][1], p[2] + OFF[o][2]};
            if (q[0] > N || q[1] > N || (dim == 3 && q[2] > N)) continue;
            m.ev.push_back((int)a);
            m.ev.push_back((int)m.vid(q[0], q[1], q[2]));
        }
        m.vedge[a + 1] = (i64)m.ev.size() / 2;
    }
    m.ne = (i64)m.ev.size() / 2;
    // faces (3D): chains a -> a+e1 -> a+e1+e2, e1 & e2 disjoint, lexicographic
    m.vface.assign(m.nv + 1, 0);
    m.fv.clear();
    if (dim == 3) {
        for (i64 a = 0; a < m.nv; ++a) {
            int p[3];
            m.lat(a, p);
            for (int o1 = 0; o1 < 7; ++o1) {
                const int *e1 = OFF3[o1];
                int q[3] = {p[0] + e1[0], p[1] + e1[1], p[2] + e1[2]};
                if (q[0] > N || q[1] > N || q[2] > N) continue;
                for (int o2 = 0; o2 < 7; ++o2) {
                    const int *e2 = OFF3[o2];
                    if ((e1[0] && e2[0]) || (e1[1] && e2[1]) || (e1[2] && e2[2])) continue;
                    int r[3] = {q[0] + e2[0], q[1] + e2[1], q[2] + e2[2]};
                    if (r[0] > N || r[1] > N || r[2] > N) continue;
                    m.fv.push_back((int)a);
                    m.fv.push_back((int)m.vid(q[0], q[1], q[2]));
                    m.fv.push_back((int)m.vid(r[0], r[1], r[2]));
                }
            }
            m.vface[a + 1] = (i64)m.fv.size() / 3;
        }
    }
    m.nf = (i64)m.fv.size() / 3;
    m.nfacet = dim == 2 ? m.ne : m.nf;
    // cells: 2D T[2s] = (v(i,j), v(i+1,j), v(i+1,j+1)), T[2s+1] = (v(i,j), v(i,j+1), v(i+1,j+1));
    // 3D Kuhn T[6c+p]: chain x0, +e_s0, +e_s1, +e_s2 for the p-th permutation (lexicographic)
    const int nvc = dim + 1;
    if (dim == 2) {
        m.nc = 2LL * N * N;
        m.cv.resize(3 * m.nc);
        for (int j = 0; j < N; ++j)
            for (int i = 0; i < N; ++i) {
                const i64 sq = i + (i64)N * j;
                int *t0 = &m.cv[3 * (2 * sq)], *t1 = &m.cv[3 * (2 * sq + 1)];
                t0[0] = (int)m.vid(i, j, 0); t0[1] = (int)m.vid(i + 1, j, 0); t0[2] = (int)m.vid(i + 1, j + 1, 0);
                t1[0] = (int)m.vid(i, j, 0); t1[1] = (int)m.vid(i, j + 1, 0); t1[2] = (int)m.vid(i + 1, j + 1, 0);
            }
    } else {
        static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
        m.nc = 6LL * N * N * N;
        m.cv.resize(4 * m.nc);
        for (int k = 0; k < N; ++k)
            for (int j = 0; j < N; ++j)
                for (int i = 0; i < N; ++i) {
                    const i64 cube = i + (i64)N * (j + (i64)N * k);
                    for (int p = 0; p < 6; ++p) {
                        int x[3] = {i, j, k};
                        int *t = &m.cv[4 * (6 * cube + p)];
                        t[0] = (int)m.vid(x[0], x[1], x[2]);
                        for (int st = 0; st < 3; ++st) {
                            x[PERM[p][st]] += 1;
                            t[st + 1] = (int)m.vid(x[0], x[1], x[2]);   // chain: ids increase
                        }
                    }
                }
    }
    m.cfacet.resize(nvc * m.nc);
    if (dim == 3) m.cedge.resize(6 * m.nc);
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) {
        const int *v = &m.cv[nvc * c];
        for (int q = 0; q < nvc; ++q) {
            int w[3], t = 0;
            for (int a = 0; a < nvc; ++a) if (a != q) w[t++] = v[a];
            m.cfacet[nvc * c + q] = (int)(dim == 2 ? m.edge_id(w[0], w[1]) : m.face_id(w[0], w[1], w[2]));
        }
        if (dim == 3)
            for (int q = 0; q < 6; ++q) m.cedge[6 * c + q] = (int)m.edge_id(v[LE[q][0]], v[LE[q][1]]);
    }
    m.fcell.assign(2 * m.nfacet, -1);
    for (i64 c = 0; c < m.nc; ++c)
        for (int q = 0; q < nvc; ++q) {
            const int f = m.cfacet[nvc * c + q];
            if (m.fcell[2 * f] < 0) m.fcell[2 * f] = (int)c;
            else m.fcell[2 * f + 1] = (int)c;
        }
}

// ------------------------------------------------------------------------------------
// free DoFs (R-num, R-bc): E-B: free E entities then free facets; velocity: d per facet
// ------------------------------------------------------------------------------------
struct Space {
    int block = 0, dim = 2;
    i64 n = 0, nE = 0;
    std::vector<int> vdof, edof, fdof;   // -1 = constrained
};

void build_space(Space &s, const Mesh &m, int block) {
    s.block = block; s.dim = m.dim;
    s.vdof.assign(m.nv, -1); s.edof.assign(m.ne, -1); s.fdof.assign(m.nfacet, -1);
    i64 n = 0;
    if (block == 0) {
        if (m.dim == 2) {
            for (i64 v = 0; v < m.nv; ++v) if (!m.on_bnd(v)) s.vdof[v] = (int)n++;
        } else {
            for (i64 e = 0; e < m.ne; ++e) if (!m.common_bnd(&m.ev[2 * e], 2)) s.edof[e] = (int)n++;
        }
        s.nE = n;
        for (i64 f = 0; f < m.nfacet; ++f) {
            const int *fvv = m.dim == 2 ? &m.ev[2 * f] : &m.fv[3 * f];
            if (!m.common_bnd(fvv, m.dim)) s.fdof[f] = (int)n++;
        }
    } else {
        for (i64 f = 0; f < m.nfacet; ++f) {
            const int *fvv = m.dim == 2 ? &m.ev[2 * f] : &m.fv[3 * f];
            if (!m.common_bnd(fvv, m.dim)) { s.fdof[f] = (int)n; n += m.dim; }
        }
    }
    s.n = n;
}

// all DoF slots of a cell in local order (-1 = constrained):
//   E-B 2D: vertices 0..2, facets q = 0..2     E-B 3D: edges (LE order), facets q = 0..3
//   velocity: facet q (opposite vertex q), facet-vertex s  ->  index d*q + s
int cell_dofs(const Mesh &m, const Space &s, i64 c, int *out) {
    const int d = m.dim, nvc = d + 1;
    int k = 0;
    if (s.block == 0) {
        if (d == 2) for (int a = 0; a < 3; ++a) out[k++] = s.vdof[m.cv[3 * c + a]];
        else for (int q = 0; q < 6; ++q) out[k++] = s.edof[m.cedge[6 * c + q]];
        for (int q = 0; q < nvc; ++q) out[k++] = s.fdof[m.cfacet[nvc * c + q]];
    } else {
        for (int q = 0; q < nvc; ++q) {
            const int f0 = s.fdof[m.cfacet[nvc * c + q]];
            for (int t = 0; t < d; ++t) out[k++] = f0 < 0 ? -1 : f0 + t;
        }
    }
    return k;
}

// ------------------------------------------------------------------------------------
// cell geometry: barycentric gradients from the lattice (unimodular => exact integers).
// R = dd for the assembly (reading R-exact), R = double for the prolongation, whose
// values are exact dyadic rationals on the lattice (reading R-prol).
// ------------------------------------------------------------------------------------
template <class R>
struct GeoT {
    int d;
    R X[4][3];   // vertex coordinates
    R g[4][3];   // gradients of the barycentric coordinates
    R vol;
    R dvol;      // d |K| = |det| h^d / (d-1)!
    int v[4];
};
typedef GeoT<double> Geo;

// scale = N: physical coordinates X = L/N (gradients x N); scale = 1: lattice units
template <class R>
void geo_from_lattice(int d, const int L[4][3], int scale, GeoT<R> &G) {
    int J[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    for (int a = 1; a <= d; ++a)
        for (int r = 0; r < d; ++r) J[r][a - 1] = L[a][r] - L[0][r];
    long C[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};
    long det;
    if (d == 2) {
        det = (long)J[0][0] * J[1][1] - (long)J[0][1] * J[1][0];
        C[0][0] = J[1][1]; C[0][1] = -J[0][1]; C[1][0] = -J[1][0]; C[1][1] = J[0][0];   // adjugate
    } else {
        long Co[3][3];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) {
                const int r1 = (r + 1) % 3, r2 = (r + 2) % 3, c1 = (c + 1) % 3, c2 = (c + 2) % 3;
                Co[r][c] = (long)J[r1][c1] * J[r2][c2] - (long)J[r1][c2] * J[r2][c1];
            }
        det = J[0][0] * Co[0][0] + J[0][1] * Co[0][1] + J[0][2] * Co[0][2];
        for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) C[r][c] = Co[c][r];
    }
    G.d = d;
    for (int a = 0; a < 4; ++a)
        for (int r = 0; r < 3; ++r) { G.X[a][r] = R(0.0); G.g[a][r] = R(0.0); }
    const R sc((double)scale), rdet((double)det);
    for (int a = 0; a <= d; ++a)
        for (int r = 0; r < d; ++r) G.X[a][r] = R((double)L[a][r]) / sc;
    // gradient of lam_a (a >= 1) = row a-1 of J^-1 = adj/det (times scale)
    for (int a = 1; a <= d; ++a)
        for (int r = 0; r < d; ++r) G.g[a][r] = R((double)C[a - 1][r]) * sc / rdet;
    for (int r = 0; r < d; ++r) {
        R s(0.0);
        for (int a = 1; a <= d; ++a) s += G.g[a][r];
        G.g[0][r] = -s;
    }
    const double adet = (double)(det < 0 ? -det : det);
    const R hd = d == 2 ? sc * sc : sc * sc * sc;
    G.vol = R(adet) / (R(d == 2 ? 2.0 : 6.0) * hd);
    G.dvol = R(adet) / (R(d == 2 ? 1.0 : 2.0) * hd);
}

template <class R>
void cell_geo(const Mesh &m, i64 c, GeoT<R> &G) {
    const int d = m.dim;
    int L[4][3] = {{0}};
    for (int a = 0; a <= d; ++a) {
        G.v[a] = m.cv[(d + 1) * c + a];
        m.lat(G.v[a], L[a]);
    }
    geo_from_lattice(d, L, m.N, G);
}

template <class R>
inline R dot3(const R *a, const R *b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
template <class R>
inline void cross3(const R *a, const R *b, R *c) {
    c[0] = a[1] * b[2] - a[2] * b[1];
    c[1] = a[2] * b[0] - a[0] * b[2];
    c[2] = a[0] * b[1] - a[1] * b[0];
}

// area vector |F| n_F of the facet opposite local vertex q, global orientation (R-orient):
// 2D edge a<b: n = (t_y, -t_x);  3D face a<b<c: (x_b - x_a) x (x_c - x_a) / 2
template <class R>
void facet_area(const GeoT<R> &G, int q, R *A, int *fl) {
    int t = 0;
    for (int a = 0; a <= G.d; ++a) if (a != q) fl[t++] = a;
    A[0] = A[1] = A[2] = R(0.0);
    if (G.d == 2) {
        A[0] = G.X[fl[1]][1] - G.X[fl[0]][1];
        A[1] = -(G.X[fl[1]][0] - G.X[fl[0]][0]);
    } else {
        R u[3], w[3];
        for (int r = 0; r < 3; ++r) { u[r] = G.X[fl[1]][r] - G.X[fl[0]][r]; w[r] = G.X[fl[2]][r] - G.X[fl[0]][r]; }
        cross3(u, w, A);
        for (int r = 0; r < 3; ++r) A[r] = A[r] * R(0.5);
    }
}

// +1 if the global normal of facet q points out of the cell
template <class R>
double facet_sign(const GeoT<R> &G, int q, const R *A, const int *fl) {
    R t[3];
    for (int r = 0; r < 3; ++r) t[r] = G.X[fl[0]][r] - G.X[q][r];
    return to_double(dot3(A, t)) > 0 ? 1.0 : -1.0;
}

// advecting field on the cell (R-w): 2D vcurl of the P1 stream function; 3D curl of the
// NED1 interpolant of the P1 vector potential (edge circulations of A_h)
template <class R>
void cell_wind(const GeoT<R> &G, const double *pot, R *w) {
    w[0] = w[1] = w[2] = R(0.0);
    if (G.d == 2) {
        R gx(0.0), gy(0.0);
        for (int a = 0; a < 3; ++a) { gx += R(pot[G.v[a]]) * G.g[a][0]; gy += R(pot[G.v[a]]) * G.g[a][1]; }
        w[0] = gy; w[1] = -gx;
        return;
    }
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (int e = 0; e < 6; ++e) {
        const int i = LE[e][0], j = LE[e][1];
        R circ(0.0);
        for (int r = 0; r < 3; ++r)
            circ += R(0.5) * (R(pot[3 * (i64)G.v[i] + r]) + R(pot[3 * (i64)G.v[j] + r])) * (G.X[j][r] - G.X[i][r]);
        R cr[3];
        cross3(G.g[i], G.g[j], cr);
        for (int r = 0; r < 3; ++r) w[r] += R(2.0) * circ * cr[r];
    }
}

template <class R>
inline R mass_bary(const GeoT<R> &G, int a, int b) {   // int_K lam_a lam_b
    return G.vol * R(a == b ? 2.0 : 1.0) / R(G.d == 2 ? 12.0 : 20.0);
}

// ------------------------------------------------------------------------------------
// BDM1 flux-nodal basis (R-basis): phi_{q,s} = lam_a v, a = s-th vertex of facet q,
// v orthogonal to the normals of the other facets through a, v . A_q = 1
// ------------------------------------------------------------------------------------
template <class R>
struct VelBasisT {
    int a[12];
    R v[12][3];
    double sg[12];     // orientation sign of the basis function's facet in this cell
};

template <class R>
void vel_basis(const GeoT<R> &G, VelBasisT<R> &B) {
    const int d = G.d;
    for (int q = 0; q <= d; ++q) {
        R A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        const double sgn = facet_sign(G, q, A, fl);
        for (int s = 0; s < d; ++s) {
            const int k = d * q + s, a = fl[s];
            R dir[3] = {R(0.0), R(0.0), R(0.0)};
            if (d == 2) {
                const int b = fl[1 - s];
                dir[0] = -G.g[b][1]; dir[1] = G.g[b][0];
            } else {
                const int b = fl[(s + 1) % 3], c = fl[(s + 2) % 3];
                cross3(G.g[b], G.g[c], dir);
            }
            const R sc = dot3(dir, A);
            B.a[k] = a;
            for (int r = 0; r < 3; ++r) B.v[k][r] = dir[r] / sc;
            B.sg[k] = sgn;
        }
    }
}

// ------------------------------------------------------------------------------------
// CSR pattern: row -> ascending columns
// ------------------------------------------------------------------------------------
struct Pattern {
    std::vector<i64> rp;
    std::vector<int> ci;
};

i64 find_col(const Pattern &P, i64 row, int col) {
    const int *b = P.ci.data() + P.rp[row], *e = P.ci.data() + P.rp[row + 1];
    const int *it = std::lower_bound(b, e, col);
    return (it != e && *it == col) ? (i64)(it - P.ci.data()) : -1;
}

// incidence: entity -> cells (ascending)
void incidence(const Mesh &m, int kind, std::vector<i64> &ptr, std::vector<int> &cells) {
    const int d = m.dim, nvc = d + 1;
    const i64 nent = kind == 0 ? m.nv : (kind == 1 ? m.ne : m.nfacet);
    const int per = kind == 0 ? nvc : (kind == 1 ? 6 : nvc);
    ptr.assign(nent + 1, 0);
    auto ent = [&](i64 c, int t) -> i64 {
        if (kind == 0) return m.cv[nvc * c + t];
        if (kind == 1) return m.cedge[6 * c + t];
        return m.cfacet[nvc * c + t];
    };
    for (i64 c = 0; c < m.nc; ++c) for (int t = 0; t < per; ++t) ptr[ent(c, t) + 1]++;
    for (i64 e = 0; e < nent; ++e) ptr[e + 1] += ptr[e];
    cells.resize(ptr[nent]);
    std::vector<i64> fill(ptr.begin(), ptr.end() - 1);
    for (i64 c = 0; c < m.nc; ++c) for (int t = 0; t < per; ++t) cells[fill[ent(c, t)]++] = (int)c;
}

// R-exact: round the extended-precision entries of one row.  E = exponent of the row's
// largest |entry| (RN53, frexp convention), G = 2^(E-88): each entry is first rounded to
// the nearest multiple of G, then to fp64 (ties to even).  Exact values on the G-grid --
// in particular dyadic values with few significant bits, whose fp64 rounding can be an
// exact tie -- are rounded exactly; exact cancellations become 0.
inline double grid_round(const dd &x, int E) {
    const double H = std::ldexp(x.hi, 88 - E), L = std::ldexp(x.lo, 88 - E);
    const double N = std::nearbyint(H);
    const double k = std::nearbyint((H - N) + L);
    const double v = std::ldexp(N + k, E - 88);
    return v == 0.0 ? 0.0 : v;   // exact cancellation: +0
}

void round_row(const dd *x, i64 len, double *out, double floor = 0.0) {
    double mx = floor;
    for (i64 k = 0; k < len; ++k) mx = std::max(mx, std::fabs(x[k].value()));
    if (mx == 0.0) {
        for (i64 k = 0; k < len; ++k) out[k] = 0.0;
        return;
    }
    int E;
    std::frexp(mx, &E);
    for (i64 k = 0; k < len; ++k) out[k] = grid_round(x[k], E);
}

// ------------------------------------------------------------------------------------
// E-B block, gather form (element data cached per cell, double-double)
// ------------------------------------------------------------------------------------
struct EBLocal {
    int nE, nB;
    int gE[6], gB[4];
    double sB[4];
    dd EE[6][6], EB[6][4], BE[4][6], BB[4][4];
};

void eb_local(const Mesh &m, const Space &s, i64 c, const double *pot, double Rem, double dt, int picard,
              EBLocal &K) {
    GeoT<dd> G;
    cell_geo(m, c, G);
    const int d = m.dim, nvc = d + 1;
    K.nE = d == 2 ? 3 : 6;
    K.nB = nvc;
    dd w[3];
    cell_wind(G, pot, w);
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    dd curlE[6][3];
    for (int a = 0; a < K.nE; ++a) {
        if (d == 2) {
            K.gE[a] = s.vdof[G.v[a]];
            curlE[a][0] = G.g[a][1]; curlE[a][1] = -G.g[a][0]; curlE[a][2] = dd(0.0);
        } else {
            K.gE[a] = s.edof[m.cedge[6 * c + a]];
            cross3(G.g[LE[a][0]], G.g[LE[a][1]], curlE[a]);
            for (int r = 0; r < 3; ++r) curlE[a][r] = curlE[a][r] * dd(2.0);
        }
    }
    // RT basis psi_q = s_q (x - X_q) / (d |K|)
    dd cq[4], cen[3] = {dd(0.0), dd(0.0), dd(0.0)};
    for (int a = 0; a <= d; ++a) for (int r = 0; r < 3; ++r) cen[r] += G.X[a][r];
    for (int r = 0; r < 3; ++r) cen[r] = cen[r] / dd((double)nvc);
    for (int q = 0; q < nvc; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        K.sB[q] = facet_sign(G, q, A, fl);
        cq[q] = dd(K.sB[q]) / G.dvol;
        K.gB[q] = s.fdof[m.cfacet[nvc * c + q]];
    }
    for (int i = 0; i < K.nE; ++i)
        for (int j = 0; j < K.nE; ++j) {
            if (d == 2) K.EE[i][j] = mass_bary(G, i, j);
            else {
                const int a = LE[i][0], b = LE[i][1], p = LE[j][0], q = LE[j][1];
                // (lam_a g_b - lam_b g_a) . (lam_p g_q - lam_q g_p)
                K.EE[i][j] = mass_bary(G, a, p) * dot3(G.g[b], G.g[q]) - mass_bary(G, a, q) * dot3(G.g[b], G.g[p]) -
                             mass_bary(G, b, p) * dot3(G.g[a], G.g[q]) + mass_bary(G, b, q) * dot3(G.g[a], G.g[p]);
            }
        }
    // A_{i,q} = int psi_q . curl phi_i = s_q/d curl phi_i . (centroid - X_q);  G~_{i,q} = int (w x psi_q) . phi_i
    const dd rRem = dd(1.0) / dd(Rem);
    for (int q = 0; q < nvc; ++q) {
        dd dc[3];
        for (int r = 0; r < 3; ++r) dc[r] = cen[r] - G.X[q][r];
        dd wx[4][3];
        for (int b = 0; b <= d; ++b) {
            dd t[3];
            for (int r = 0; r < 3; ++r) t[r] = G.X[b][r] - G.X[q][r];
            if (d == 2) { wx[b][0] = w[0] * t[1] - w[1] * t[0]; wx[b][1] = wx[b][2] = dd(0.0); }
            else cross3(w, t, wx[b]);
        }
        for (int i = 0; i < K.nE; ++i) {
            const dd a_iq = dd(K.sB[q]) * dot3(curlE[i], dc) / dd((double)d);
            dd gt(0.0);
            if (d == 2) {
                for (int b = 0; b <= 2; ++b) gt += mass_bary(G, b, i) * wx[b][0];
            } else {
                const int a = LE[i][0], bb = LE[i][1];
                for (int b = 0; b <= 3; ++b)
                    gt += mass_bary(G, b, a) * dot3(wx[b], G.g[bb]) - mass_bary(G, b, bb) * dot3(wx[b], G.g[a]);
            }
            gt = picard ? dd(0.0) : gt * cq[q];                       // delta = 0: no G~ (NEXT-4)
            K.EB[i][q] = gt - a_iq / dd(Rem);
            K.BE[q][i] = a_iq;
        }
    }
    // transient (eta = 1): (1/dt)(psi_l, psi_k) = (1/dt) c_k c_l sum_ab M_ab (X_a - X_k).(X_b - X_l)
    for (int k = 0; k < nvc; ++k)
        for (int l = 0; l < nvc; ++l) {
            dd acc(0.0);
            if (dt > 0)
                for (int a = 0; a <= d; ++a)
                    for (int b = 0; b <= d; ++b) {
                        dd ta[3], tb[3];
                        for (int r = 0; r < 3; ++r) { ta[r] = G.X[a][r] - G.X[k][r]; tb[r] = G.X[b][r] - G.X[l][r]; }
                        acc += mass_bary(G, a, b) * dot3(ta, tb);
                    }
            K.BB[k][l] = dt > 0 ? acc * cq[k] * cq[l] / dd(dt) : dd(0.0);
        }
    (void)rRem;
}

void assemble_eb(const Mesh &m, const Space &s, const Params &p, const double *pot, Pattern &P,
                 std::vector<double> &val) {
    const int d = m.dim;
    std::vector<i64> vp, ep, fp;
    std::vector<int> vc, ec, fc;
    if (d == 2) incidence(m, 0, vp, vc); else incidence(m, 1, ep, ec);
    incidence(m, 2, fp, fc);
    std::vector<int> dkind(s.n), dent(s.n);
    for (i64 v = 0; v < m.nv; ++v) if (s.vdof[v] >= 0) { dkind[s.vdof[v]] = 0; dent[s.vdof[v]] = (int)v; }
    for (i64 e = 0; e < m.ne; ++e) if (s.edof[e] >= 0) { dkind[s.edof[e]] = 1; dent[s.edof[e]] = (int)e; }
    for (i64 f = 0; f < m.nfacet; ++f) if (s.fdof[f] >= 0) { dkind[s.fdof[f]] = 2; dent[s.fdof[f]] = (int)f; }
    auto cells_of = [&](i64 row, const int *&b, const int *&e) {
        const int k = dkind[row], id = dent[row];
        if (k == 0) { b = vc.data() + vp[id]; e = vc.data() + vp[id + 1]; }
        else if (k == 1) { b = ec.data() + ep[id]; e = ec.data() + ep[id + 1]; }
        else { b = fc.data() + fp[id]; e = fc.data() + fp[id + 1]; }
    };
    // pattern: DoFs of the cells containing the row's entity
    P.rp.assign(s.n + 1, 0);
    std::vector<std::vector<int>> rows(s.n);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        std::vector<int> cols;
        int loc[10];
        for (const int *c = b; c != e; ++c) {
            const int k = cell_dofs(m, s, *c, loc);
            for (int t = 0; t < k; ++t) if (loc[t] >= 0) cols.push_back(loc[t]);
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        rows[r] = std::move(cols);
    }
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] = P.rp[r] + (i64)rows[r].size();
    P.ci.resize(P.rp[s.n]);
    for (i64 r = 0; r < s.n; ++r) std::copy(rows[r].begin(), rows[r].end(), P.ci.begin() + P.rp[r]);
    rows.clear();
    // element data of every cell, once
    std::vector<EBLocal> loc(m.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) eb_local(m, s, c, pot, p.Rem, p.dt, p.picard, loc[c]);
    val.assign(P.rp[s.n], 0.0);
    const double Kinv = d == 2 ? 2.0 * m.N * m.N : 6.0 * m.N * m.N * m.N;   // 1/|K|
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        const i64 base = P.rp[r], len = P.rp[r + 1] - base;
        std::vector<dd> acc(len);
        std::vector<int> cnt(len, 0);
        const bool isB = dkind[r] == 2;
        for (const int *c = b; c != e; ++c) {
            const EBLocal &K = loc[*c];
            int li = -1;
            if (!isB) { for (int a = 0; a < K.nE; ++a) if (K.gE[a] == r) li = a; }
            else { for (int q = 0; q < K.nB; ++q) if (K.gB[q] == r) li = q; }
            auto add = [&](int col, const dd &v) { acc[find_col(P, r, col) - base] += v; };
            if (!isB) {
                for (int j = 0; j < K.nE; ++j) if (K.gE[j] >= 0) add(K.gE[j], K.EE[li][j]);
                for (int q = 0; q < K.nB; ++q) if (K.gB[q] >= 0) add(K.gB[q], K.EB[li][q]);
            } else {
                for (int j = 0; j < K.nE; ++j) if (K.gE[j] >= 0) add(K.gE[j], K.BE[li][j]);
                for (int q = 0; q < K.nB; ++q)
                    if (K.gB[q] >= 0) {
                        cnt[find_col(P, r, K.gB[q]) - base] += (int)(K.sB[li] * K.sB[q]);
                        if (p.dt > 0) add(K.gB[q], K.BB[li][q]);
                    }
            }
        }
        // C = (1/Rem)(div psi_l, div psi_k): exact value Kinv m / Rem (R-gamma)
        for (i64 k = 0; k < len; ++k)
            if (cnt[k]) acc[k] += dd(Kinv * cnt[k]) / dd(p.Rem);
        round_row(acc.data(), len, val.data() + base);
    }
}

// ------------------------------------------------------------------------------------
// AL velocity block, gather form by facet row blocks (element data cached per cell)
// ------------------------------------------------------------------------------------
struct CellVel {
    GeoT<dd> G;
    VelBasisT<dd> B;
    dd w[3];
    dd bn[3];          // B^n on the cell (NEXT-4), zero when absent
    dd eps[12][3][3];
    int gi[12];
};

void cell_vel(const Mesh &m, const Space &s, i64 c, const double *pot, const double *bpot, CellVel &K) {
    cell_geo(m, c, K.G);
    vel_basis(K.G, K.B);
    cell_wind(K.G, pot, K.w);
    K.bn[0] = K.bn[1] = K.bn[2] = dd(0.0);
    if (bpot) cell_wind(K.G, bpot, K.bn);
    const int d = m.dim, nb = d * (d + 1);
    cell_dofs(m, s, c, K.gi);
    for (int k = 0; k < nb; ++k) {
        const dd *g = K.G.g[K.B.a[k]], *v = K.B.v[k];
        for (int l = 0; l < 3; ++l)
            for (int r = 0; r < 3; ++r) K.eps[k][l][r] = dd(0.5) * (v[l] * g[r] + v[r] * g[l]);
    }
}

void assemble_vel(const Mesh &m, const Space &s, const Params &p, const double *pot, const double *bpot, Pattern &P,
                  std::vector<double> &val) {
    const int d = m.dim, nvc = d + 1, nb = d * nvc;
    // row blocks = free facets; pattern from the cells of the facet and their facet neighbours
    std::vector<int> freef;
    for (i64 f = 0; f < m.nfacet; ++f) if (s.fdof[f] >= 0) freef.push_back((int)f);
    const i64 nblk = (i64)freef.size();
    std::vector<std::vector<int>> cols(nblk);
#pragma omp parallel for schedule(dynamic, 128)
    for (i64 t = 0; t < nblk; ++t) {
        const int f = freef[t];
        std::vector<int> cells;
        for (int side = 0; side < 2; ++side) {
            const int c = m.fcell[2 * f + side];
            if (c < 0) continue;
            cells.push_back(c);
            for (int q = 0; q < nvc; ++q) {
                const int g = m.cfacet[nvc * c + q];
                for (int s2 = 0; s2 < 2; ++s2) {
                    const int o = m.fcell[2 * g + s2];
                    if (o >= 0) cells.push_back(o);
                }
            }
        }
        std::vector<int> cl;
        int loc[12];
        for (int c : cells) {
            cell_dofs(m, s, c, loc);
            for (int k = 0; k < nb; ++k) if (loc[k] >= 0) cl.push_back(loc[k]);
        }
        std::sort(cl.begin(), cl.end());
        cl.erase(std::unique(cl.begin(), cl.end()), cl.end());
        cols[t] = std::move(cl);
    }
    P.rp.assign(s.n + 1, 0);
    for (i64 t = 0; t < nblk; ++t)
        for (int a = 0; a < d; ++a) P.rp[s.fdof[freef[t]] + a + 1] = (i64)cols[t].size();
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] += P.rp[r];
    P.ci.resize(P.rp[s.n]);
    for (i64 t = 0; t < nblk; ++t)
        for (int a = 0; a < d; ++a) std::copy(cols[t].begin(), cols[t].end(), P.ci.begin() + P.rp[s.fdof[freef[t]] + a]);
    cols.clear();
    // element data of every cell, once
    std::vector<CellVel> cellv(m.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) cell_vel(m, s, c, pot, bpot, cellv[c]);
    val.assign(P.rp[s.n], 0.0);
    const dd nu2 = dd(2.0) / dd(p.Re);
    const double Kinv = d == 2 ? 2.0 * m.N * m.N : 6.0 * m.N * m.N * m.N;
    const dd fden(d == 2 ? 6.0 : 12.0);   // int_F mu_a mu_b = |F|(1+d_ab)/fden
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 t = 0; t < nblk; ++t) {
        const int f = freef[t];
        const int r0 = s.fdof[f];
        const i64 base = P.rp[r0], len = P.rp[r0 + 1] - base;
        std::vector<dd> acc(d * len);
        std::vector<int> cnt(len, 0);
        auto pos = [&](int col) -> i64 { return find_col(P, r0, col) - base; };
        auto add = [&](int a, int col, const dd &v) { acc[a * len + pos(col)] += v; };
        // ---- cell terms, cells of f ascending ----
        std::vector<int> fcells;
        for (int side = 0; side < 2; ++side) if (m.fcell[2 * f + side] >= 0) fcells.push_back(m.fcell[2 * f + side]);
        for (int c : fcells) {
            const CellVel &K = cellv[c];
            int qf = -1;
            for (int q = 0; q < nvc; ++q) if (m.cfacet[nvc * c + q] == f) qf = q;
            const dd V = K.G.vol, Vn = K.G.vol / dd((double)nvc);
            for (int a = 0; a < d; ++a) {
                const int i = d * qf + a;                  // test function (this row)
                const dd gw = dot3(K.G.g[K.B.a[i]], K.w);
                for (int j = 0; j < nb; ++j) {
                    if (K.gi[j] < 0) continue;
                    dd ee(0.0);
                    for (int l = 0; l < 3; ++l) for (int r = 0; r < 3; ++r) ee += K.eps[j][l][r] * K.eps[i][l][r];
                    dd term = nu2 * V * ee - dot3(K.B.v[j], K.B.v[i]) * gw * Vn;          // viscous - advection
                    if (p.dt > 0)                                                         // (1/dt)(u, v), NEXT-4
                        term += mass_bary(K.G, K.B.a[j], K.B.a[i]) * dot3(K.B.v[j], K.B.v[i]) / dd(p.dt);
                    if (bpot) {                                 // S (u x B^n, v x B^n), NEXT-4
                        dd cj[3], ci[3];
                        if (d == 2) {
                            cj[0] = K.B.v[j][0] * K.bn[1] - K.B.v[j][1] * K.bn[0];
                            ci[0] = K.B.v[i][0] * K.bn[1] - K.B.v[i][1] * K.bn[0];
                            cj[1] = cj[2] = ci[1] = ci[2] = dd(0.0);
                        } else {
                            cross3(K.B.v[j], K.bn, cj);
                            cross3(K.B.v[i], K.bn, ci);
                        }
                        term += dd(p.S) * mass_bary(K.G, K.B.a[j], K.B.a[i]) * dot3(cj, ci);
                    }
                    add(a, K.gi[j], term);
                }
            }
            for (int j = 0; j < nb; ++j)
                if (K.gi[j] >= 0) cnt[pos(K.gi[j])] += (int)(K.B.sg[d * qf] * K.B.sg[j]);
        }
        // ---- facet terms: every facet of the cells of f ----
        std::vector<int> gs;
        for (int c : fcells) for (int q = 0; q < nvc; ++q) gs.push_back(m.cfacet[nvc * c + q]);
        std::sort(gs.begin(), gs.end());
        gs.erase(std::unique(gs.begin(), gs.end()), gs.end());
        for (int g : gs) {
            const int cp = m.fcell[2 * g], cm = m.fcell[2 * g + 1];
            const bool interior = cm >= 0;
            const CellVel &Kp = cellv[cp];
            int qp = -1, qm = -1;
            for (int q = 0; q < nvc; ++q) {
                if (m.cfacet[nvc * cp + q] == g) qp = q;
                if (interior && m.cfacet[nvc * cm + q] == g) qm = q;
            }
            dd A[3];
            int fl[3];
            facet_area(Kp.G, qp, A, fl);
            const dd area = sqrt(dot3(A, A));
            const double sgn = facet_sign(Kp.G, qp, A, fl);
            dd n[3];
            for (int r = 0; r < 3; ++r) n[r] = dd(sgn) * A[r] / area;
            dd hF(0.0);
            if (d == 2) hF = area;
            else
                for (int a = 0; a < 3; ++a)
                    for (int b = a + 1; b < 3; ++b) {
                        dd tt[3];
                        for (int r = 0; r < 3; ++r) tt[r] = Kp.G.X[fl[b]][r] - Kp.G.X[fl[a]][r];
                        const dd l = sqrt(dot3(tt, tt));
                        if (l > hF) hF = l;
                    }
            const dd avg(interior ? 0.5 : 1.0);
            const dd pen = dd(p.sigma) / (dd(p.Re) * hF);
            // Burman stabilisation (reading R-mu): interior facets add
            // mu h_F^2 int_F [grad u]:[grad v]; grad (lam_a v) = v (x) grad lam_a is constant per
            // cell, so [grad phi_I]:[grad phi_J] = J_I J_J (v_I . v_J)(g_I . g_J); h_F^2 exact
            dd hF2(0.0);
            if (d == 2) hF2 = dot3(A, A);
            else
                for (int a = 0; a < 3; ++a)
                    for (int b = a + 1; b < 3; ++b) {
                        dd tt[3];
                        for (int r = 0; r < 3; ++r) tt[r] = Kp.G.X[fl[b]][r] - Kp.G.X[fl[a]][r];
                        if (dot3(tt, tt) > hF2) hF2 = dot3(tt, tt);
                    }
            const dd burman = interior ? dd(p.mu) * hF2 * area : dd(0.0);
            const bool use_burman = interior && p.mu != 0.0;
            const dd wn = dot3(Kp.w, n), awn = fabs(wn);
            const dd upp = dd(0.5) * (wn + awn), upm = dd(-0.5) * (awn - wn);
            const dd intF = area / dd((double)d);
            struct Fn { int side, vtx, gidx; dd v[3], en[3], g[3]; };
            Fn fn[24];
            int nf = 0;
            for (int side = 0; side < (interior ? 2 : 1); ++side) {
                const CellVel &K = side ? cellv[cm] : Kp;
                const int qq = side ? qm : qp;
                for (int k = 0; k < nb; ++k) {
                    Fn &F = fn[nf++];
                    F.side = side ? -1 : 1;
                    F.vtx = K.B.a[k] == qq ? -1 : K.G.v[K.B.a[k]];   // lam_a = 0 on g if a is opposite
                    F.gidx = K.gi[k];
                    for (int r = 0; r < 3; ++r) {
                        F.v[r] = K.B.v[k][r];
                        F.en[r] = K.eps[k][r][0] * n[0] + K.eps[k][r][1] * n[1] + K.eps[k][r][2] * n[2];
                        F.g[r] = K.G.g[K.B.a[k]][r];
                    }
                }
            }
            for (int ti = 0; ti < nf; ++ti) {
                const Fn &I = fn[ti];
                if (I.gidx < r0 || I.gidx >= r0 + d) continue;   // rows of this block only
                const int a = I.gidx - r0;
                const dd Ji((double)I.side);
                for (int tj = 0; tj < nf; ++tj) {
                    const Fn &J = fn[tj];
                    if (J.gidx < 0) continue;
                    const dd Jj((double)J.side);
                    dd term(0.0);
                    if (I.vtx >= 0) term += -(nu2 * avg * Ji * dot3(J.en, I.v) * intF);     // consistency
                    if (J.vtx >= 0) term += -(nu2 * avg * Jj * dot3(J.v, I.en) * intF);     // symmetry
                    if (I.vtx >= 0 && J.vtx >= 0) {
                        const dd vv = dot3(J.v, I.v) * area * dd(I.vtx == J.vtx ? 2.0 : 1.0) / fden;
                        term += pen * Ji * Jj * vv;                                         // penalty
                        if (interior) term += (J.side > 0 ? upp : upm) * vv * Ji;           // upwind
                        else term += upp * vv;
                    }
                    if (use_burman) term += burman * Ji * Jj * dot3(J.v, I.v) * dot3(J.g, I.g);  // Burman
                    add(a, J.gidx, term);
                }
            }
        }
        // ---- gamma (div u, div v) = gamma Kinv m / d^2, exact (R-gamma); rows rounded once (R-exact)
        const double Gk = p.gamma * Kinv;
        for (int a = 0; a < d; ++a) {
            for (i64 k = 0; k < len; ++k)
                if (cnt[k]) acc[a * len + k] += dd(Gk * cnt[k]) / dd((double)(d * d));
            round_row(acc.data() + a * len, len, val.data() + P.rp[r0 + a]);
        }
    }
}

// ------------------------------------------------------------------------------------
// vertex-star patches: per vertex, the free DoFs whose entity contains it
// ------------------------------------------------------------------------------------
void build_patches(const Mesh &m, const Space &s, std::vector<i64> &pptr, std::vector<int> &pdofs, std::vector<int> &pvert) {
    // vertex -> incident edges and facets
    std::vector<std::vector<int>> vlist(m.nv);
    for (i64 v = 0; v < m.nv; ++v) if (s.vdof[v] >= 0) vlist[v].push_back(s.vdof[v]);
    for (i64 e = 0; e < m.ne; ++e)
        if (s.edof[e] >= 0) { vlist[m.ev[2 * e]].push_back(s.edof[e]); vlist[m.ev[2 * e + 1]].push_back(s.edof[e]); }
    const int nfv = m.dim;
    for (i64 f = 0; f < m.nfacet; ++f) {
        if (s.fdof[f] < 0) continue;
        const int *fvv = m.dim == 2 ? &m.ev[2 * f] : &m.fv[3 * f];
        const int k = s.block == 1 ? m.dim : 1;
        for (int t = 0; t < nfv; ++t)
            for (int a = 0; a < k; ++a) vlist[fvv[t]].push_back(s.fdof[f] + a);
    }
    pptr.assign(1, 0);
    pdofs.clear();
    pvert.clear();
    for (i64 v = 0; v < m.nv; ++v) {
        auto &L = vlist[v];
        if (L.empty()) continue;   // empty stars dropped (R-patch)
        std::sort(L.begin(), L.end());
        pdofs.insert(pdofs.end(), L.begin(), L.end());
        pptr.push_back((i64)pdofs.size());
        pvert.push_back((int)v);
    }
}

// ------------------------------------------------------------------------------------
// prolongation: P_IJ = N_I^fine(phi_J^coarse), on the fine lattice (h_f = 1,
// coarse cells of edge 2) where every value is an exact dyadic rational
// ------------------------------------------------------------------------------------
struct Aff { double c[3]; double G[3][3]; };   // f(x) = c + G x   (lattice coordinates)

void aff_eval(const Aff &f, const double *x, double *out) {
    for (int l = 0; l < 3; ++l) out[l] = f.c[l] + f.G[l][0] * x[0] + f.G[l][1] * x[1] + f.G[l][2] * x[2];
}

// barycentric coordinate lam_a as affine function on the lattice: lam_a(x) = 1{a==0} + g_a.(x - X_0)
void bary_aff(const Geo &G, int a, double *c, double *g) {
    for (int r = 0; r < 3; ++r) g[r] = G.g[a][r];
    *c = (a == 0 ? 1.0 : 0.0) - dot3(G.g[a], G.X[0]);
}

void build_prolongation(const Mesh &mf, const Space &sf, const Mesh &mc, const Space &sc, std::vector<i64> &rp,
                        std::vector<int> &ci, std::vector<double> &vv) {
    const int d = mf.dim, nvc = d + 1;
    std::vector<std::vector<std::pair<int, double>>> rows(sf.n);
    std::vector<char> done(sf.n, 0);
    static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    for (i64 c = 0; c < mf.nc; ++c) {
        int loc[12];
        const int k = cell_dofs(mf, sf, c, loc);
        bool any = false;
        for (int t = 0; t < k; ++t) any = any || (loc[t] >= 0 && !done[loc[t]]);
        if (!any) continue;
        // fine cell lattice vertices and its coarse parent
        int Lf[4][3] = {{0}};
        int sum[3] = {0, 0, 0};
        for (int a = 0; a <= d; ++a) {
            mf.lat(mf.cv[nvc * c + a], Lf[a]);
            for (int r = 0; r < d; ++r) sum[r] += Lf[a][r];
        }
        // centroid = sum/(d+1); coarse cube = floor(centroid / 2); relative order inside
        int cube[3] = {0, 0, 0}, rel[3] = {0, 0, 0};
        for (int r = 0; r < d; ++r) { cube[r] = sum[r] / (2 * nvc); rel[r] = sum[r] - 2 * nvc * cube[r]; }
        i64 pc;
        if (d == 2) {
            const i64 sq = cube[0] + (i64)mc.N * cube[1];
            pc = rel[0] > rel[1] ? 2 * sq : 2 * sq + 1;
        } else {
            const i64 cb = cube[0] + (i64)mc.N * (cube[1] + (i64)mc.N * cube[2]);
            pc = -1;
            for (int q = 0; q < 6; ++q)
                if (rel[PERM[q][0]] > rel[PERM[q][1]] && rel[PERM[q][1]] > rel[PERM[q][2]]) pc = 6 * cb + q;
        }
        int Lc[4][3] = {{0}};
        for (int a = 0; a <= d; ++a) {
            mc.lat(mc.cv[nvc * pc + a], Lc[a]);
            for (int r = 0; r < d; ++r) Lc[a][r] *= 2;
        }
        Geo Gc;
        geo_from_lattice(d, Lc, 1, Gc);
        // coarse basis functions as affine fields on the lattice
        Aff F[12];
        int gJ[12];
        int nbc = 0;
        auto coarse_basis = [&](int kind) {
            nbc = 0;
            if (kind == 0) {       // CG1
                for (int a = 0; a < 3; ++a) {
                    Aff &f = F[nbc]; memset(&f, 0, sizeof f);
                    bary_aff(Gc, a, &f.c[0], f.G[0]);
                    gJ[nbc++] = sc.vdof[mc.cv[3 * pc + a]];
                }
            } else if (kind == 1) {  // NED1 Whitney lam_i g_j - lam_j g_i
                for (int e = 0; e < 6; ++e) {
                    Aff &f = F[nbc]; memset(&f, 0, sizeof f);
                    const int i = LE[e][0], j = LE[e][1];
                    double ci_, gi_[3], cj_, gj_[3];
                    bary_aff(Gc, i, &ci_, gi_);
                    bary_aff(Gc, j, &cj_, gj_);
                    for (int l = 0; l < 3; ++l) {
                        f.c[l] = ci_ * Gc.g[j][l] - cj_ * Gc.g[i][l];
                        for (int r = 0; r < 3; ++r) f.G[l][r] = Gc.g[j][l] * gi_[r] - Gc.g[i][l] * gj_[r];
                    }
                    gJ[nbc++] = sc.edof[mc.cedge[6 * pc + e]];
                }
            } else if (kind == 2) {  // RT: s (x - X_q) / (d |K|)
                for (int q = 0; q < nvc; ++q) {
                    Aff &f = F[nbc]; memset(&f, 0, sizeof f);
                    double A[3]; int fl[3];
                    facet_area(Gc, q, A, fl);
                    const double cc = facet_sign(Gc, q, A, fl) / Gc.dvol;
                    for (int l = 0; l < d; ++l) { f.c[l] = -cc * Gc.X[q][l]; f.G[l][l] = cc; }
                    gJ[nbc++] = sc.fdof[mc.cfacet[nvc * pc + q]];
                }
            } else {                 // BDM1: lam_a v
                VelBasisT<double> B;
                vel_basis(Gc, B);
                for (int q = 0; q < nvc; ++q) {
                    const int f0 = sc.fdof[mc.cfacet[nvc * pc + q]];
                    for (int t = 0; t < d; ++t) {
                        Aff &f = F[nbc]; memset(&f, 0, sizeof f);
                        const int kk = d * q + t;
                        double ca, ga[3];
                        bary_aff(Gc, B.a[kk], &ca, ga);
                        for (int l = 0; l < 3; ++l) {
                            f.c[l] = ca * B.v[kk][l];
                            for (int r = 0; r < 3; ++r) f.G[l][r] = B.v[kk][l] * ga[r];
                        }
                        gJ[nbc++] = f0 < 0 ? -1 : f0 + t;
                    }
                }
            }
        };
        Geo Gf;
        geo_from_lattice(d, Lf, 1, Gf);
        int last_kind = -1;
        for (int t = 0; t < k; ++t) {
            const int I = loc[t];
            if (I < 0 || done[I]) continue;
            done[I] = 1;
            // fine DoF entity and functional
            int kind;
            if (sf.block == 1) kind = 3;
            else if (d == 2) kind = t < 3 ? 0 : 2;
            else kind = t < 6 ? 1 : 2;
            if (kind != last_kind) { coarse_basis(kind); last_kind = kind; }
            double val[12];
            for (int b = 0; b < nbc; ++b) {
                double fx[3];
                if (kind == 0) {
                    double x[3] = {(double)Lf[t][0], (double)Lf[t][1], 0.0};
                    aff_eval(F[b], x, fx);
                    val[b] = fx[0];
                } else if (kind == 1) {
                    const int i = LE[t][0], j = LE[t][1];
                    double mid[3], tg[3];
                    for (int r = 0; r < 3; ++r) { mid[r] = 0.5 * (Gf.X[i][r] + Gf.X[j][r]); tg[r] = Gf.X[j][r] - Gf.X[i][r]; }
                    aff_eval(F[b], mid, fx);
                    val[b] = dot3(fx, tg);
                } else {
                    const int q = sf.block == 1 ? t / d : t - (d == 2 ? 3 : 6);
                    double A[3]; int fl[3];
                    facet_area(Gf, q, A, fl);
                    if (kind == 2) {
                        // flux of an affine field = |F| x (mean of its vertex values) . n;
                        // every term is an exact dyadic rational on the lattice
                        double acc = 0;
                        for (int a = 0; a < d; ++a) {
                            aff_eval(F[b], Gf.X[fl[a]], fx);
                            acc += dot3(fx, A);
                        }
                        val[b] = acc / d;
                    } else {
                        aff_eval(F[b], Gf.X[fl[t % d]], fx);
                        val[b] = dot3(fx, A);
                    }
                }
            }
            for (int b = 0; b < nbc; ++b)
                if (gJ[b] >= 0 && val[b] != 0.0) rows[I].push_back({gJ[b], val[b]});
        }
    }
    rp.assign(sf.n + 1, 0);
    for (i64 I = 0; I < sf.n; ++I) {
        std::sort(rows[I].begin(), rows[I].end());
        rp[I + 1] = rp[I] + (i64)rows[I].size();
    }
    ci.resize(rp[sf.n]);
    vv.resize(rp[sf.n]);
    for (i64 I = 0; I < sf.n; ++I)
        for (size_t t = 0; t < rows[I].size(); ++t) { ci[rp[I] + t] = rows[I][t].first; vv[rp[I] + t] = rows[I][t].second; }
}

// ------------------------------------------------------------------------------------
// NEXT-3 coupling blocks (Table 1), gather form, double-double, R-exact rows.
// Closed forms with phi_i = lam_a v (BDM1), psi_k = sum_b lam_b P_b (RT1, P_b =
// c_k (X_b - X_k)), E = lam_e (CG1) or lam_p g_q - lam_q g_p (NED1); u^n = w, B^n
// constant per cell.  2D conventions: u x B = u1 B2 - u2 B1, B x s = (B2 s, -B1 s).
// ------------------------------------------------------------------------------------
inline void xcr(int d, const dd *a, const dd *b, dd *c) {          // vector x vector
    if (d == 2) { c[0] = a[0] * b[1] - a[1] * b[0]; c[1] = c[2] = dd(0.0); }
    else cross3(a, b, c);
}
inline void xsc(int d, const dd *B, const dd *s, dd *c) {          // B x (scalar or vector)
    if (d == 2) { c[0] = B[1] * s[0]; c[1] = -(B[0] * s[0]); c[2] = dd(0.0); }
    else cross3(B, s, c);
}

struct CellCoup {
    GeoT<dd> G;
    VelBasisT<dd> V;
    dd w[3], bn[3];
    dd cq[4];          // RT scale s_q / (d |K|)
    int gv[12], gE[6], gB[4];
};

void cell_coup(const Mesh &m, const Space &sv, const Space &se, i64 c, const double *pot, const double *bpot,
               CellCoup &K) {
    cell_geo(m, c, K.G);
    vel_basis(K.G, K.V);
    cell_wind(K.G, pot, K.w);
    K.bn[0] = K.bn[1] = K.bn[2] = dd(0.0);
    if (bpot) cell_wind(K.G, bpot, K.bn);
    const int d = m.dim, nvc = d + 1;
    cell_dofs(m, sv, c, K.gv);
    int ebd[10];
    cell_dofs(m, se, c, ebd);
    const int nE = d == 2 ? 3 : 6;
    for (int t = 0; t < nE; ++t) K.gE[t] = ebd[t];
    for (int q = 0; q < nvc; ++q) {
        K.gB[q] = ebd[nE + q] < 0 ? -1 : ebd[nE + q] - (int)se.nE;
        dd A[3];
        int fl[3];
        facet_area(K.G, q, A, fl);
        K.cq[q] = dd(facet_sign(K.G, q, A, fl)) / K.G.dvol;
    }
}

// coupling of velocity test function i with the E basis function e / B basis function k
inline dd coup_J(const CellCoup &K, int d, int i, int e) {
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    const int ai = K.V.a[i];
    const dd *v = K.V.v[i];
    if (d == 2) {                                    // (B^n x lam_e) . v = lam_e (B1 v0 - B0 v1)
        return mass_bary(K.G, e, ai) * (K.bn[1] * v[0] - K.bn[0] * v[1]);
    }
    const int p = LE[e][0], q = LE[e][1];
    dd c1[3], c2[3];
    cross3(K.bn, K.G.g[q], c1);
    cross3(K.bn, K.G.g[p], c2);
    return mass_bary(K.G, p, ai) * dot3(c1, v) - mass_bary(K.G, q, ai) * dot3(c2, v);
}
inline dd coup_G(const CellCoup &K, int d, int e, int i) {      // (v_i x B^n, F_e)
    static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};
    const int ai = K.V.a[i];
    dd vb[3];
    xcr(d, K.V.v[i], K.bn, vb);
    if (d == 2) return mass_bary(K.G, ai, e) * vb[0];
    const int p = LE[e][0], q = LE[e][1];
    return mass_bary(K.G, ai, p) * dot3(vb, K.G.g[q]) - mass_bary(K.G, ai, q) * dot3(vb, K.G.g[p]);
}
inline dd coup_D(const CellCoup &K, int d, int i, int k) {      // D~1 + D~2, without S
    const int ai = K.V.a[i];
    dd wb[3];
    xcr(d, K.w, K.bn, wb);                                      // u^n x B^n
    dd acc(0.0);
    for (int b = 0; b <= d; ++b) {
        dd P[3];
        for (int r = 0; r < 3; ++r) P[r] = K.cq[k] * (K.G.X[b][r] - K.G.X[k][r]);
        dd t1[3], ub[3], t2[3];
        xsc(d, P, wb, t1);                                      // B x (u^n x B^n)
        xcr(d, K.w, P, ub);                                     // u^n x B
        xsc(d, K.bn, ub, t2);                                   // B^n x (u^n x B)
        acc += mass_bary(K.G, b, ai) * (dot3(t1, K.V.v[i]) + dot3(t2, K.V.v[i]));
    }
    return acc;
}

}  // namespace

std::string assemble_coupling(int dim, int N, const Params &p, const double *w, const double *bn, const double *floor_u,
                              const double *floor_E, CouplingBlocks &out) {
    Mesh m;
    build_mesh(m, dim, N);
    Space sv, se;
    build_space(sv, m, 1);
    build_space(se, m, 0);
    const int d = dim, nvc = d + 1, nb = d * nvc, nE = d == 2 ? 3 : 6;
    out.nu = sv.n; out.np = m.nc; out.nE = se.nE; out.nB = se.n - se.nE;
    std::vector<CellCoup> cc(m.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) cell_coup(m, sv, se, c, w, bn, cc[c]);
    // ---- u rows (Bt, J, Dt): row block = free facet f, cells of f ascending ----
    std::vector<int> freef;
    for (i64 f = 0; f < m.nfacet; ++f) if (sv.fdof[f] >= 0) freef.push_back((int)f);
    auto init = [](HostCsr &A, i64 n, i64 ncols) { A.n = n; A.ncols = ncols; A.rp.assign(n + 1, 0); };
    init(out.Bt, out.nu, out.np); init(out.J, out.nu, out.nE); init(out.Dt, out.nu, out.nB); init(out.G, out.nE, out.nu);
    struct RowData { std::vector<int> cB, cJ, cD; std::vector<dd> vB, vJ, vD; };
    std::vector<RowData> rows(sv.n);
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 t = 0; t < (i64)freef.size(); ++t) {
        const int f = freef[t], r0 = sv.fdof[f];
        std::vector<int> cells;
        for (int side = 0; side < 2; ++side) if (m.fcell[2 * f + side] >= 0) cells.push_back(m.fcell[2 * f + side]);
        // column sets: union over the cells (sorted unique)
        std::vector<int> colsE, colsB, colsP;
        for (int c : cells) {
            colsP.push_back(c);
            for (int e = 0; e < nE; ++e) if (cc[c].gE[e] >= 0) colsE.push_back(cc[c].gE[e]);
            for (int q = 0; q < nvc; ++q) if (cc[c].gB[q] >= 0) colsB.push_back(cc[c].gB[q]);
        }
        for (auto *v : {&colsE, &colsB, &colsP}) {
            std::sort(v->begin(), v->end());
            v->erase(std::unique(v->begin(), v->end()), v->end());
        }
        for (int a = 0; a < d; ++a) {
            RowData &R = rows[r0 + a];
            R.cB = colsP; R.cJ = colsE; R.cD = colsB;
            R.vB.assign(colsP.size(), dd(0.0)); R.vJ.assign(colsE.size(), dd(0.0)); R.vD.assign(colsB.size(), dd(0.0));
            for (int c : cells) {
                const CellCoup &K = cc[c];
                int li = -1;
                for (int k = 0; k < nb; ++k) if (K.gv[k] == r0 + a) li = k;
                const dd divv = dot3(K.V.v[li], K.G.g[K.V.a[li]]) * K.G.vol;        // int_K div v
                R.vB[std::lower_bound(colsP.begin(), colsP.end(), c) - colsP.begin()] += -divv;
                for (int e = 0; e < nE; ++e)
                    if (K.gE[e] >= 0)
                        R.vJ[std::lower_bound(colsE.begin(), colsE.end(), K.gE[e]) - colsE.begin()] +=
                            dd(p.S) * coup_J(K, d, li, e);
                if (!p.picard)
                    for (int q = 0; q < nvc; ++q)
                        if (K.gB[q] >= 0)
                            R.vD[std::lower_bound(colsB.begin(), colsB.end(), K.gB[q]) - colsB.begin()] +=
                                dd(p.S) * coup_D(K, d, li, q);
            }
        }
    }
    // ---- E rows (G): cells of the E entity ascending ----
    std::vector<i64> ep;
    std::vector<int> ec;
    if (d == 2) incidence(m, 0, ep, ec); else incidence(m, 1, ep, ec);
    std::vector<std::vector<int>> gcols(out.nE);
    std::vector<std::vector<dd>> gvals(out.nE);
    std::vector<int> Eent(out.nE);
    if (d == 2) { for (i64 v = 0; v < m.nv; ++v) if (se.vdof[v] >= 0) Eent[se.vdof[v]] = (int)v; }
    else { for (i64 e = 0; e < m.ne; ++e) if (se.edof[e] >= 0) Eent[se.edof[e]] = (int)e; }
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < out.nE; ++r) {
        const int ent = Eent[r];
        std::vector<int> cl;
        for (i64 t = ep[ent]; t < ep[ent + 1]; ++t)
            for (int k = 0; k < nb; ++k) if (cc[ec[t]].gv[k] >= 0) cl.push_back(cc[ec[t]].gv[k]);
        std::sort(cl.begin(), cl.end());
        cl.erase(std::unique(cl.begin(), cl.end()), cl.end());
        std::vector<dd> vals(cl.size(), dd(0.0));
        for (i64 t = ep[ent]; t < ep[ent + 1]; ++t) {
            const CellCoup &K = cc[ec[t]];
            int le = -1;
            for (int e = 0; e < nE; ++e) if (K.gE[e] == r) le = e;
            for (int k = 0; k < nb; ++k)
                if (K.gv[k] >= 0) vals[std::lower_bound(cl.begin(), cl.end(), K.gv[k]) - cl.begin()] += coup_G(K, d, le, k);
        }
        gcols[r] = std::move(cl);
        gvals[r] = std::move(vals);
    }
    // ---- pack with the row rounding of R-exact, on the grid of the whole Newton row
    // (reading R-cgrid: the grid exponent is floored by the diagonal block's row max) ----
    auto pack = [](HostCsr &A, i64 n, auto colsOf, auto valsOf, const double *floor) {
        for (i64 r = 0; r < n; ++r) A.rp[r + 1] = A.rp[r] + (i64)colsOf(r).size();
        A.ci.resize(A.rp[n]);
        A.v.resize(A.rp[n]);
        for (i64 r = 0; r < n; ++r) {
            const auto &c = colsOf(r);
            std::copy(c.begin(), c.end(), A.ci.begin() + A.rp[r]);
            round_row(valsOf(r).data(), (i64)c.size(), A.v.data() + A.rp[r], floor ? floor[r] : 0.0);
        }
    };
    pack(out.Bt, out.nu, [&](i64 r) -> const std::vector<int> & { return rows[r].cB; },
         [&](i64 r) -> const std::vector<dd> & { return rows[r].vB; }, floor_u);
    pack(out.J, out.nu, [&](i64 r) -> const std::vector<int> & { return rows[r].cJ; },
         [&](i64 r) -> const std::vector<dd> & { return rows[r].vJ; }, floor_u);
    pack(out.Dt, out.nu, [&](i64 r) -> const std::vector<int> & { return rows[r].cD; },
         [&](i64 r) -> const std::vector<dd> & { return rows[r].vD; }, floor_u);
    pack(out.G, out.nE, [&](i64 r) -> const std::vector<int> & { return gcols[r]; },
         [&](i64 r) -> const std::vector<dd> & { return gvals[r]; }, floor_E);
    return "";
}


// ------------------------------------------------------------------------------------
// NEXT-2: element degree k = 2 for the 2D E-B block, E in CG2, B in RT2,
// reading R-basis2 (DoFs: CG2 point values at vertices and edge midpoints; RT2 normal
// moments int_e (B.n_e) lam_s ds against the two P1 functions of each edge, s = lower /
// higher global vertex, and N int_K B_r dx per cell).  Independent of the oracle's
// quadrature: every function is a homogeneous polynomial in the barycentric coordinates
// and every integral is the closed form  int_K lam^alpha = 2|K| alpha! / (|alpha| + 2)!
// (edges: int_e mu^beta = |e| beta! / (|beta| + 1)!).  The RT2 primal basis is
// {lam_a psi_q} (P1 times the RT0 functions psi_q = s_q (x - X_q)/(2|K|); the relation
// sum_q lam_q (x - X_q) = 0 removes (a, q) = (2, 2)), made dual to the DoFs by inverting
// the 8 x 8 DoF matrix in double-double.
// ------------------------------------------------------------------------------------
namespace {

inline double fact(int n) { double r = 1; for (int i = 2; i <= n; ++i) r *= i; return r; }

// int_K lam_i1 ... lam_ik (k = 2, 3, 4) / (2|K|)  =  prod n_j! / (k + 2)!
dd bary_int_eval(const int *idx, int k) {
    int n[3] = {0, 0, 0};
    for (int t = 0; t < k; ++t) n[idx[t]]++;
    return dd(fact(n[0]) * fact(n[1]) * fact(n[2])) / dd(fact(k + 2));
}
struct BaryTables {
    dd t2[9], t3[27], t4[81];
    BaryTables() {
        for (int a = 0; a < 81; ++a) {
            const int idx[4] = {a / 27, (a / 9) % 3, (a / 3) % 3, a % 3};
            t4[a] = bary_int_eval(idx, 4);
            if (a < 27) { const int i3[3] = {a / 9, (a / 3) % 3, a % 3}; t3[a] = bary_int_eval(i3, 3); }
            if (a < 9) { const int i2[2] = {a / 3, a % 3}; t2[a] = bary_int_eval(i2, 2); }
        }
    }
};
const BaryTables &bary_tables() { static const BaryTables T; return T; }
inline const dd &bary_int(const int *idx, int k) {
    const BaryTables &T = bary_tables();
    if (k == 2) return T.t2[3 * idx[0] + idx[1]];
    if (k == 3) return T.t3[9 * idx[0] + 3 * idx[1] + idx[2]];
    return T.t4[27 * idx[0] + 9 * idx[1] + 3 * idx[2] + idx[3]];
}

struct Space2 {
    i64 n = 0, nE = 0;
    std::vector<int> vdof, edof, fdof, cdof;   // edof: CG2 midpoint DoF per edge (2D: edge = facet)
};

// R-num2 (same order as DESIGN.md): free vertices, free edges (CG2); 2 per interior edge,
// then 2 per cell (RT2)
void build_space2(Space2 &s, const Mesh &m) {
    s.vdof.assign(m.nv, -1); s.edof.assign(m.ne, -1); s.fdof.assign(m.nfacet, -1); s.cdof.assign(m.nc, -1);
    i64 n = 0;
    for (i64 v = 0; v < m.nv; ++v) if (!m.on_bnd(v)) s.vdof[v] = (int)n++;
    for (i64 e = 0; e < m.ne; ++e) if (!m.common_bnd(&m.ev[2 * e], 2)) s.edof[e] = (int)n++;
    s.nE = n;
    for (i64 f = 0; f < m.nfacet; ++f) if (!m.common_bnd(&m.ev[2 * f], 2)) { s.fdof[f] = (int)n; n += 2; }
    for (i64 c = 0; c < m.nc; ++c) { s.cdof[c] = (int)n; n += 2; }
    s.n = n;
}

// local order: E: vertices 0..2, edges (0,1) (0,2) (1,2); B: facet q (opposite vertex q)
// x s = 0, 1, then r = 0, 1
static const int E2V[3][2] = {{0, 1}, {0, 2}, {1, 2}};
void cell_dofs2(const Mesh &m, const Space2 &s, i64 c, int *gE, int *gB) {
    for (int a = 0; a < 3; ++a) gE[a] = s.vdof[m.cv[3 * c + a]];
    for (int t = 0; t < 3; ++t) gE[3 + t] = s.edof[m.cfacet[3 * c + (2 - t)]];   // edge (i,j) is opposite 3-i-j
    for (int q = 0; q < 3; ++q) {
        const int f0 = s.fdof[m.cfacet[3 * c + q]];
        gB[2 * q] = f0 < 0 ? -1 : f0;
        gB[2 * q + 1] = f0 < 0 ? -1 : f0 + 1;
    }
    gB[6] = s.cdof[c]; gB[7] = s.cdof[c] + 1;
}

// element of the k = 2 E-B block: CG2 as quadratics sum e[b][d] lam_b lam_d, RT2 as
// sum V[a][b] lam_a lam_b (2-vectors)
struct Elem2 {
    GeoT<dd> G;
    dd e[6][3][3];
    dd V[8][3][3][2];
};

// RT2 functionals (local order) of the field sum V[a][b] lam_a lam_b on cell G
void rt2_dofs(const GeoT<dd> &G, int Ncells, const dd V[3][3][2], dd *out) {
    for (int q = 0; q < 3; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        // int_e (B.A/|e|) mu_s ds = sum_{a,b in e} (V_ab . A) int_e mu_a mu_b mu_s / |e|
        for (int s = 0; s < 2; ++s) {
            dd acc(0.0);
            for (int ia = 0; ia < 2; ++ia)
                for (int ib = 0; ib < 2; ++ib) {
                    const int a = fl[ia], b = fl[ib];
                    int n[2] = {0, 0};
                    n[ia]++; n[ib]++; n[s]++;
                    const dd mom = dd(fact(n[0]) * fact(n[1])) / dd(24.0);     // beta! / 4!
                    acc += (V[a][b][0] * A[0] + V[a][b][1] * A[1]) * mom;
                }
            out[2 * q + s] = acc;
        }
    }
    for (int r = 0; r < 2; ++r) {
        dd acc(0.0);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                const int idx[2] = {a, b};
                acc += V[a][b][r] * bary_int(idx, 2);
            }
        out[6 + r] = acc * dd(2.0) * G.vol * dd((double)Ncells);
    }
}

dd dd_fabs(const dd &x) { return x.hi < 0 ? -x : x; }

void elem2(const Mesh &m, i64 c, Elem2 &K) {
    cell_geo(m, c, K.G);
    const GeoT<dd> &G = K.G;
    memset((void *)K.e, 0, sizeof K.e);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) K.e[a][a][b] = dd(a == b ? 1.0 : -1.0);   // lam_a (2 lam_a - sum lam)
    for (int t = 0; t < 3; ++t) K.e[3 + t][E2V[t][0]][E2V[t][1]] = dd(4.0);
    // primal RT2 functions p_{a,q} = lam_a psi_q, psi_q = c_q sum_b lam_b (X_b - X_q)
    dd cq[3];
    for (int q = 0; q < 3; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        cq[q] = dd(facet_sign(G, q, A, fl)) / G.dvol;
    }
    int np = 0;
    dd Pv[8][3][3][2];
    memset((void *)Pv, 0, sizeof Pv);
    for (int a = 0; a < 3; ++a)
        for (int q = 0; q < 3; ++q) {
            if (a == 2 && q == 2) continue;
            for (int b = 0; b < 3; ++b)
                for (int r = 0; r < 2; ++r) Pv[np][a][b][r] = cq[q] * (G.X[b][r] - G.X[q][r]);
            ++np;
        }
    // DoF matrix M[i][j] = N_i(p_j), Gauss-Jordan in double-double
    dd W[8][16];
    for (int j = 0; j < 8; ++j) {
        dd col[8];
        rt2_dofs(G, m.N, Pv[j], col);
        for (int i = 0; i < 8; ++i) W[i][j] = col[i];
    }
    for (int i = 0; i < 8; ++i) for (int j = 0; j < 8; ++j) W[i][8 + j] = dd(i == j ? 1.0 : 0.0);
    for (int k = 0; k < 8; ++k) {
        int p = k;
        for (int i = k + 1; i < 8; ++i) if (to_double(dd_fabs(W[i][k])) > to_double(dd_fabs(W[p][k]))) p = i;
        if (p != k) for (int j = 0; j < 16; ++j) std::swap(W[k][j], W[p][j]);
        const dd piv = W[k][k];
        for (int j = 0; j < 16; ++j) W[k][j] = W[k][j] / piv;
        for (int i = 0; i < 8; ++i) {
            if (i == k) continue;
            const dd l = W[i][k];
            for (int j = 0; j < 16; ++j) W[i][j] = W[i][j] - l * W[k][j];
        }
    }
    // dual basis phi_j = sum_k Cinv[k][j] p_k
    for (int j = 0; j < 8; ++j)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                for (int r = 0; r < 2; ++r) {
                    dd acc(0.0);
                    for (int k = 0; k < 8; ++k) acc += W[k][8 + j] * Pv[k][a][b][r];
                    K.V[j][a][b][r] = acc;
                }
}

struct EBLocal2 {
    int gE[6], gB[8];
    dd EE[6][6], EB[6][8], BE[8][6], BB[8][8];
};

void eb_local2(const Mesh &m, const Space2 &s, i64 c, const double *pot, const Params &p, EBLocal2 &L) {
    Elem2 K;
    elem2(m, c, K);
    const GeoT<dd> &G = K.G;
    cell_dofs2(m, s, c, L.gE, L.gB);
    dd w[3];
    cell_wind(G, pot, w);
    const dd twoK = dd(2.0) * G.vol;
    // gradient of the CG2 functions: sum_c lam_c Gr[c] ;  vcurl = (Gr_y, -Gr_x)
    dd R[6][3][2];
    for (int i = 0; i < 6; ++i)
        for (int cc = 0; cc < 3; ++cc) {
            dd gx(0.0), gy(0.0);
            for (int d2 = 0; d2 < 3; ++d2) {
                const dd t = K.e[i][cc][d2] + K.e[i][d2][cc];
                gx += t * G.g[d2][0];
                gy += t * G.g[d2][1];
            }
            R[i][cc][0] = gy; R[i][cc][1] = -gx;
        }
    // divergence of the RT2 functions: sum_c lam_c D[c]
    dd D[8][3];
    for (int k = 0; k < 8; ++k)
        for (int cc = 0; cc < 3; ++cc) {
            dd acc(0.0);
            for (int b = 0; b < 3; ++b) {
                acc += G.g[b][0] * K.V[k][cc][b][0] + G.g[b][1] * K.V[k][cc][b][1];
                acc += G.g[b][0] * K.V[k][b][cc][0] + G.g[b][1] * K.V[k][b][cc][1];
            }
            D[k][cc] = acc;
        }
    for (int i = 0; i < 6; ++i)
        for (int j = 0; j < 6; ++j) {
            dd acc(0.0);
            for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b)
                for (int cc = 0; cc < 3; ++cc) for (int d2 = 0; d2 < 3; ++d2) {
                    const int idx[4] = {a, b, cc, d2};
                    acc += K.e[i][a][b] * K.e[j][cc][d2] * bary_int(idx, 4);
                }
            L.EE[i][j] = acc * twoK;
        }
    for (int i = 0; i < 6; ++i)
        for (int k = 0; k < 8; ++k) {
            dd ab(0.0), gt(0.0);
            for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) {
                for (int cc = 0; cc < 3; ++cc) {
                    const int idx[3] = {a, b, cc};
                    ab += (K.V[k][a][b][0] * R[i][cc][0] + K.V[k][a][b][1] * R[i][cc][1]) * bary_int(idx, 3);
                }
                if (!p.picard) {
                    const dd wxb = w[0] * K.V[k][a][b][1] - w[1] * K.V[k][a][b][0];
                    for (int cc = 0; cc < 3; ++cc) for (int d2 = 0; d2 < 3; ++d2) {
                        const int idx[4] = {a, b, cc, d2};
                        gt += wxb * K.e[i][cc][d2] * bary_int(idx, 4);
                    }
                }
            }
            ab = ab * twoK;
            gt = gt * twoK;
            L.EB[i][k] = gt - ab / dd(p.Rem);
            L.BE[k][i] = ab;
        }
    for (int k = 0; k < 8; ++k)
        for (int l = 0; l < 8; ++l) {
            dd dv(0.0);
            for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) {
                const int idx[2] = {a, b};
                dv += D[k][a] * D[l][b] * bary_int(idx, 2);
            }
            dd v = dv * twoK / dd(p.Rem);
            if (p.dt > 0) {
                dd ms(0.0);
                for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b)
                    for (int cc = 0; cc < 3; ++cc) for (int d2 = 0; d2 < 3; ++d2) {
                        const int idx[4] = {a, b, cc, d2};
                        ms += (K.V[k][a][b][0] * K.V[l][cc][d2][0] + K.V[k][a][b][1] * K.V[l][cc][d2][1]) *
                              bary_int(idx, 4);
                    }
                v += ms * twoK / dd(p.dt);
            }
            L.BB[k][l] = v;
        }
}

// gather-form assembly by rows (cells of the row's entity, ascending), R-exact rows
void assemble_eb2(const Mesh &m, const Space2 &s, const Params &p, const double *pot, Pattern &P,
                  std::vector<double> &val) {
    std::vector<i64> vp, fp;
    std::vector<int> vc, fc;
    incidence(m, 0, vp, vc);
    incidence(m, 2, fp, fc);
    std::vector<int> dkind(s.n), dent(s.n);
    for (i64 v = 0; v < m.nv; ++v) if (s.vdof[v] >= 0) { dkind[s.vdof[v]] = 0; dent[s.vdof[v]] = (int)v; }
    for (i64 e = 0; e < m.ne; ++e) if (s.edof[e] >= 0) { dkind[s.edof[e]] = 1; dent[s.edof[e]] = (int)e; }
    for (i64 f = 0; f < m.nfacet; ++f)
        if (s.fdof[f] >= 0) for (int a = 0; a < 2; ++a) { dkind[s.fdof[f] + a] = 1; dent[s.fdof[f] + a] = (int)f; }
    for (i64 c = 0; c < m.nc; ++c) for (int a = 0; a < 2; ++a) { dkind[s.cdof[c] + a] = 2; dent[s.cdof[c] + a] = (int)c; }
    std::vector<int> self(m.nc);
    std::iota(self.begin(), self.end(), 0);
    auto cells_of = [&](i64 row, const int *&b, const int *&e) {
        const int k = dkind[row], id = dent[row];
        if (k == 0) { b = vc.data() + vp[id]; e = vc.data() + vp[id + 1]; }
        else if (k == 1) { b = fc.data() + fp[id]; e = fc.data() + fp[id + 1]; }
        else { b = self.data() + id; e = b + 1; }
    };
    std::vector<EBLocal2> loc(m.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) eb_local2(m, s, c, pot, p, loc[c]);
    P.rp.assign(s.n + 1, 0);
    std::vector<std::vector<int>> rows(s.n);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        std::vector<int> cols;
        for (const int *c = b; c != e; ++c) {
            for (int t = 0; t < 6; ++t) if (loc[*c].gE[t] >= 0) cols.push_back(loc[*c].gE[t]);
            for (int t = 0; t < 8; ++t) if (loc[*c].gB[t] >= 0) cols.push_back(loc[*c].gB[t]);
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        rows[r] = std::move(cols);
    }
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] = P.rp[r] + (i64)rows[r].size();
    P.ci.resize(P.rp[s.n]);
    for (i64 r = 0; r < s.n; ++r) std::copy(rows[r].begin(), rows[r].end(), P.ci.begin() + P.rp[r]);
    rows.clear();
    val.assign(P.rp[s.n], 0.0);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        const i64 base = P.rp[r], len = P.rp[r + 1] - base;
        std::vector<dd> acc(len);
        const bool isB = r >= s.nE;
        for (const int *c = b; c != e; ++c) {
            const EBLocal2 &K = loc[*c];
            int li = -1;
            if (!isB) { for (int a = 0; a < 6; ++a) if (K.gE[a] == r) li = a; }
            else { for (int a = 0; a < 8; ++a) if (K.gB[a] == r) li = a; }
            auto add = [&](int col, const dd &v) { acc[find_col(P, r, col) - base] += v; };
            for (int j = 0; j < 6; ++j) if (K.gE[j] >= 0) add(K.gE[j], isB ? K.BE[li][j] : K.EE[li][j]);
            for (int j = 0; j < 8; ++j) if (K.gB[j] >= 0) add(K.gB[j], isB ? K.BB[li][j] : K.EB[li][j]);
        }
        round_row(acc.data(), len, val.data() + base);
    }
}

void build_patches2(const Mesh &m, const Space2 &s, std::vector<i64> &pptr, std::vector<int> &pdofs, std::vector<int> &pvert) {
    std::vector<std::vector<int>> vlist(m.nv);
    for (i64 v = 0; v < m.nv; ++v) if (s.vdof[v] >= 0) vlist[v].push_back(s.vdof[v]);
    for (i64 e = 0; e < m.ne; ++e)
        for (int t = 0; t < 2; ++t) {
            const int v = m.ev[2 * e + t];
            if (s.edof[e] >= 0) vlist[v].push_back(s.edof[e]);
            if (s.fdof[e] >= 0) { vlist[v].push_back(s.fdof[e]); vlist[v].push_back(s.fdof[e] + 1); }
        }
    for (i64 c = 0; c < m.nc; ++c)
        for (int t = 0; t < 3; ++t) { vlist[m.cv[3 * c + t]].push_back(s.cdof[c]); vlist[m.cv[3 * c + t]].push_back(s.cdof[c] + 1); }
    pptr.assign(1, 0);
    pdofs.clear();
    pvert.clear();
    for (i64 v = 0; v < m.nv; ++v) {
        auto &L = vlist[v];
        if (L.empty()) continue;
        std::sort(L.begin(), L.end());
        pdofs.insert(pdofs.end(), L.begin(), L.end());
        pptr.push_back((i64)pdofs.size());
        pvert.push_back((int)v);
    }
}

// R-prol at k = 2: coarse functions rewritten in the fine cell's barycentrics
// (lam^c_b = sum_a lam^c_b(X^f_a) lam^f_a, exact dyadic weights), fine functionals in
// closed form; rows rounded as R-exact, |x| < 2^-30 max|row| dropped (R-prol2)
void build_prolongation2(const Mesh &mf, const Space2 &sf, const Mesh &mc, const Space2 &sc, std::vector<i64> &rp,
                         std::vector<int> &ci, std::vector<double> &vv) {
    std::vector<std::vector<std::pair<int, dd>>> rows(sf.n);
    // coarse elements once; each fine DoF is computed by its owner, the lowest-index fine
    // cell containing its entity (deterministic under any schedule)
    std::vector<Elem2> ce(mc.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < mc.nc; ++c) elem2(mc, c, ce[c]);
    std::vector<int> owner(sf.n, INT32_MAX);
    for (i64 c = mf.nc - 1; c >= 0; --c) {
        int gE[6], gB[8];
        cell_dofs2(mf, sf, c, gE, gB);
        for (int t = 0; t < 6; ++t) if (gE[t] >= 0) owner[gE[t]] = (int)c;
        for (int t = 0; t < 8; ++t) if (gB[t] >= 0) owner[gB[t]] = (int)c;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 c = 0; c < mf.nc; ++c) {
        int gE[6], gB[8];
        cell_dofs2(mf, sf, c, gE, gB);
        int Lf[4][3] = {{0}};
        int sum[2] = {0, 0};
        for (int a = 0; a < 3; ++a) {
            mf.lat(mf.cv[3 * c + a], Lf[a]);
            for (int r = 0; r < 2; ++r) sum[r] += Lf[a][r];
        }
        int cube[2], rel[2];
        for (int r = 0; r < 2; ++r) { cube[r] = sum[r] / 6; rel[r] = sum[r] - 6 * cube[r]; }
        const i64 sq = cube[0] + (i64)mc.N * cube[1];
        const i64 pc = rel[0] > rel[1] ? 2 * sq : 2 * sq + 1;
        const Elem2 &Kc = ce[pc];
        int cE[6], cB[8];
        cell_dofs2(mc, sc, pc, cE, cB);
        GeoT<dd> Gf;
        cell_geo(mf, c, Gf);
        // T[b][a] = lam^c_b(X^f_a)
        dd T[3][3];
        for (int b = 0; b < 3; ++b)
            for (int a = 0; a < 3; ++a) {
                dd v(b == 0 ? 1.0 : 0.0);
                for (int r = 0; r < 2; ++r) v += Kc.G.g[b][r] * (Gf.X[a][r] - Kc.G.X[0][r]);
                T[b][a] = v;
            }
        auto to_fine = [&](const dd in[3][3], dd out[3][3]) {
            for (int a = 0; a < 3; ++a)
                for (int a2 = 0; a2 < 3; ++a2) {
                    dd acc(0.0);
                    for (int b = 0; b < 3; ++b)
                        for (int d2 = 0; d2 < 3; ++d2) acc += in[b][d2] * T[b][a] * T[d2][a2];
                    out[a][a2] = acc;
                }
        };
        for (int t = 0; t < 6; ++t) {          // E DoFs owned by this fine cell
            const int I = gE[t];
            if (I < 0 || owner[I] != c) continue;
            for (int j = 0; j < 6; ++j) {
                if (cE[j] < 0) continue;
                dd f[3][3];
                to_fine(Kc.e[j], f);
                dd v;
                if (t < 3) v = f[t][t];
                else {
                    const int i = E2V[t - 3][0], k = E2V[t - 3][1];
                    v = (f[i][i] + f[k][k] + f[i][k] + f[k][i]) * dd(0.25);
                }
                rows[I].push_back({cE[j], v});
            }
        }
        bool anyB = false;
        for (int t = 0; t < 8; ++t) anyB = anyB || (gB[t] >= 0 && owner[gB[t]] == c);
        if (!anyB) continue;
        for (int j = 0; j < 8; ++j) {          // B DoFs owned by this fine cell
            if (cB[j] < 0) continue;
            dd F[3][3][2], comp[3][3], fin[3][3];
            for (int r = 0; r < 2; ++r) {
                for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) comp[a][b] = Kc.V[j][a][b][r];
                to_fine(comp, fin);
                for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) F[a][b][r] = fin[a][b];
            }
            dd out[8];
            rt2_dofs(Gf, mf.N, F, out);
            for (int t = 0; t < 8; ++t)
                if (gB[t] >= 0 && owner[gB[t]] == c) rows[gB[t]].push_back({cB[j], out[t]});
        }
    }
    rp.assign(sf.n + 1, 0);
    std::vector<std::vector<std::pair<int, double>>> fin(sf.n);
    for (i64 I = 0; I < sf.n; ++I) {
        auto &R = rows[I];
        std::sort(R.begin(), R.end(), [](const std::pair<int, dd> &x, const std::pair<int, dd> &y) { return x.first < y.first; });
        std::vector<dd> xs(R.size());
        for (size_t t = 0; t < R.size(); ++t) xs[t] = R[t].second;
        std::vector<double> rounded(R.size());
        round_row(xs.data(), (i64)xs.size(), rounded.data());
        double mx = 0;
        for (double v : rounded) mx = std::max(mx, std::fabs(v));
        for (size_t t = 0; t < R.size(); ++t)
            if (rounded[t] != 0.0 && std::fabs(to_double(xs[t])) >= std::ldexp(mx, -30)) fin[I].push_back({R[t].first, rounded[t]});
        rp[I + 1] = rp[I] + (i64)fin[I].size();
    }
    ci.resize(rp[sf.n]);
    vv.resize(rp[sf.n]);
    for (i64 I = 0; I < sf.n; ++I)
        for (size_t t = 0; t < fin[I].size(); ++t) { ci[rp[I] + t] = fin[I][t].first; vv[rp[I] + t] = fin[I][t].second; }
}


// ---------------- k = 2 AL velocity block, BDM2 (R-basis2, R-vel; sigma from the
// parameters, 10 k^2 = 40) -------------------------------------------------------
// DoFs: per facet q (opposite vertex q; vertices fl0 < fl1, area vector A = |f| n_f of the
// global orientation) N_{q,s}(u) = u(x_s) . A at x_0 = X_fl0, x_1 = X_fl1, x_2 = midpoint;
// per cell N_{K,e}(u) = int_K u . (lam_i g_j - lam_j g_i), e = (i<j) in (0,1), (0,2), (1,2).
// Local order: q = 0..2 x s = 0..2, then e = 0..2.  Primal basis lam_a lam_b e_r.
void build_space2_vel(Space2 &s, const Mesh &m) {
    s.vdof.assign(m.nv, -1); s.edof.assign(m.ne, -1); s.fdof.assign(m.nfacet, -1); s.cdof.assign(m.nc, -1);
    i64 n = 0;
    for (i64 f = 0; f < m.nfacet; ++f) if (!m.common_bnd(&m.ev[2 * f], 2)) { s.fdof[f] = (int)n; n += 3; }
    for (i64 c = 0; c < m.nc; ++c) { s.cdof[c] = (int)n; n += 3; }
    s.n = n;
    s.nE = 0;
}

void cell_dofs_v2(const Mesh &m, const Space2 &s, i64 c, int *g) {
    for (int q = 0; q < 3; ++q) {
        const int f0 = s.fdof[m.cfacet[3 * c + q]];
        for (int t = 0; t < 3; ++t) g[3 * q + t] = f0 < 0 ? -1 : f0 + t;
    }
    for (int e = 0; e < 3; ++e) g[9 + e] = s.cdof[c] + e;
}

struct ElemV2 {
    GeoT<dd> G;
    dd V[12][3][3][2];       // basis j = sum V[a][b] lam_a lam_b
    dd Gr[12][3][2][2];      // grad (row l = component, col k = direction) = sum_c lam_c Gr[c]
};

// the 12 BDM2 functionals of cell G applied to sum V[a][b] lam_a lam_b
void bdm2_dofs(const GeoT<dd> &G, const dd V[3][3][2], dd *out) {
    const BaryTables &T = bary_tables();
    for (int q = 0; q < 3; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        for (int s = 0; s < 3; ++s) {
            dd lam[3] = {dd(0.0), dd(0.0), dd(0.0)};
            if (s < 2) lam[fl[s]] = dd(1.0);
            else { lam[fl[0]] = dd(0.5); lam[fl[1]] = dd(0.5); }
            dd u[2] = {dd(0.0), dd(0.0)};
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b) {
                    const dd l2 = lam[a] * lam[b];
                    u[0] += V[a][b][0] * l2;
                    u[1] += V[a][b][1] * l2;
                }
            out[3 * q + s] = u[0] * A[0] + u[1] * A[1];
        }
    }
    for (int e = 0; e < 3; ++e) {
        const int i = E2V[e][0], j = E2V[e][1];
        dd acc(0.0);
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b) {
                const dd vgj = V[a][b][0] * G.g[j][0] + V[a][b][1] * G.g[j][1];
                const dd vgi = V[a][b][0] * G.g[i][0] + V[a][b][1] * G.g[i][1];
                acc += vgj * T.t3[9 * a + 3 * b + i] - vgi * T.t3[9 * a + 3 * b + j];
            }
        out[9 + e] = acc * dd(2.0) * G.vol;
    }
}

void elemv2(const Mesh &m, i64 c, ElemV2 &K) {
    cell_geo(m, c, K.G);
    const GeoT<dd> &G = K.G;
    dd Pv[12][3][3][2];
    memset((void *)Pv, 0, sizeof Pv);
    int np = 0;
    for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b)
            for (int r = 0; r < 2; ++r) Pv[np++][a][b][r] = dd(1.0);
    dd W[12][24];
    for (int j = 0; j < 12; ++j) {
        dd col[12];
        bdm2_dofs(G, Pv[j], col);
        for (int i = 0; i < 12; ++i) W[i][j] = col[i];
    }
    for (int i = 0; i < 12; ++i) for (int j = 0; j < 12; ++j) W[i][12 + j] = dd(i == j ? 1.0 : 0.0);
    for (int k = 0; k < 12; ++k) {
        int p = k;
        for (int i = k + 1; i < 12; ++i) if (to_double(dd_fabs(W[i][k])) > to_double(dd_fabs(W[p][k]))) p = i;
        if (p != k) for (int j = 0; j < 24; ++j) std::swap(W[k][j], W[p][j]);
        const dd piv = W[k][k];
        for (int j = 0; j < 24; ++j) W[k][j] = W[k][j] / piv;
        for (int i = 0; i < 12; ++i) {
            if (i == k) continue;
            const dd l = W[i][k];
            for (int j = 0; j < 24; ++j) W[i][j] = W[i][j] - l * W[k][j];
        }
    }
    for (int j = 0; j < 12; ++j)
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                for (int r = 0; r < 2; ++r) {
                    dd acc(0.0);
                    for (int k = 0; k < 12; ++k) acc += W[k][12 + j] * Pv[k][a][b][r];
                    K.V[j][a][b][r] = acc;
                }
    // gradients: d_k (lam_a lam_b) = lam_b g_a,k + lam_a g_b,k
    for (int j = 0; j < 12; ++j)
        for (int cc = 0; cc < 3; ++cc)
            for (int l = 0; l < 2; ++l)
                for (int k = 0; k < 2; ++k) {
                    dd acc(0.0);
                    for (int b = 0; b < 3; ++b) acc += K.V[j][cc][b][l] * G.g[b][k] + K.V[j][b][cc][l] * G.g[b][k];
                    K.Gr[j][cc][l][k] = acc;
                }
}

// row li of the cell matrix of element K (test li, trial j = 0..11), without 2|K|
void vel2_cell_row(const ElemV2 &K, int li, const dd *w, const dd *bx, bool lorentz, const Params &p, dd *row) {
    const BaryTables &T = bary_tables();
    const dd nu2 = dd(2.0) / dd(p.Re);
    dd epi[3][2][2], gwi[3][2], divi[3];
    for (int cc = 0; cc < 3; ++cc) {
        for (int l = 0; l < 2; ++l)
            for (int k = 0; k < 2; ++k) epi[cc][l][k] = (K.Gr[li][cc][l][k] + K.Gr[li][cc][k][l]) * dd(0.5);
        for (int l = 0; l < 2; ++l) gwi[cc][l] = K.Gr[li][cc][l][0] * w[0] + K.Gr[li][cc][l][1] * w[1];
        divi[cc] = K.Gr[li][cc][0][0] + K.Gr[li][cc][1][1];
    }
    for (int j = 0; j < 12; ++j) {
        dd ee(0.0), dv(0.0), adv(0.0), ms(0.0), lor(0.0);
        for (int c1 = 0; c1 < 3; ++c1) {
            dd epj[2][2];
            for (int l = 0; l < 2; ++l)
                for (int k = 0; k < 2; ++k) epj[l][k] = (K.Gr[j][c1][l][k] + K.Gr[j][c1][k][l]) * dd(0.5);
            const dd divj = K.Gr[j][c1][0][0] + K.Gr[j][c1][1][1];
            for (int c2 = 0; c2 < 3; ++c2) {
                const dd t2 = T.t2[3 * c1 + c2];
                ee += (epj[0][0] * epi[c2][0][0] + epj[0][1] * epi[c2][0][1] + epj[1][0] * epi[c2][1][0] +
                       epj[1][1] * epi[c2][1][1]) * t2;
                dv += divj * divi[c2] * t2;
            }
        }
        for (int a = 0; a < 3; ++a)
            for (int b = 0; b < 3; ++b)
                for (int cc = 0; cc < 3; ++cc)
                    adv += (K.V[j][a][b][0] * gwi[cc][0] + K.V[j][a][b][1] * gwi[cc][1]) * T.t3[9 * a + 3 * b + cc];
        if (p.dt > 0 || lorentz)
            for (int a = 0; a < 3; ++a)
                for (int b = 0; b < 3; ++b)
                    for (int c1 = 0; c1 < 3; ++c1)
                        for (int c2 = 0; c2 < 3; ++c2) {
                            const dd t4 = T.t4[27 * a + 9 * b + 3 * c1 + c2];
                            if (p.dt > 0)
                                ms += (K.V[j][a][b][0] * K.V[li][c1][c2][0] + K.V[j][a][b][1] * K.V[li][c1][c2][1]) * t4;
                            if (lorentz)
                                lor += (K.V[j][a][b][0] * bx[1] - K.V[j][a][b][1] * bx[0]) *
                                       (K.V[li][c1][c2][0] * bx[1] - K.V[li][c1][c2][1] * bx[0]) * t4;
                        }
        dd v = nu2 * ee - adv + dd(p.gamma) * dv;
        if (p.dt > 0) v += ms / dd(p.dt);
        if (lorentz) v += dd(p.S) * lor;
        row[j] = v;
    }
}

// trace of cell-basis data on an edge: lam_c = [c == c0] mu0 + [c == c1] mu1
// quadratic u -> coefficients on mu0^2, mu0 mu1, mu1^2;  linear eps -> on mu0, mu1
struct Trace2 { dd u[3][2]; dd en[2][2]; };   // en = eps(u) (sgn A) at mu0 / mu1

void vel2_trace(const ElemV2 &K, int j, int c0, int c1, const dd *sA, Trace2 &T) {
    for (int r = 0; r < 2; ++r) {
        T.u[0][r] = K.V[j][c0][c0][r];
        T.u[1][r] = K.V[j][c0][c1][r] + K.V[j][c1][c0][r];
        T.u[2][r] = K.V[j][c1][c1][r];
    }
    const int cs[2] = {c0, c1};
    for (int t = 0; t < 2; ++t) {
        const int cc = cs[t];
        for (int l = 0; l < 2; ++l) {
            const dd e0 = K.Gr[j][cc][l][0] + K.Gr[j][cc][0][l];
            const dd e1 = K.Gr[j][cc][l][1] + K.Gr[j][cc][1][l];
            T.en[t][l] = (e0 * sA[0] + e1 * sA[1]) * dd(0.5);
        }
    }
}

// int_0^1 mu0^p mu1^q (edge of unit measure) = p! q! / (p+q+1)!
inline dd emom(int p, int q) { return dd(fact(p) * fact(q)) / dd(fact(p + q + 1)); }

// Q = int u_j . v_i,  E = int (a . b) with a linear, b quadratic  (per unit edge measure)
dd tr_qq(const Trace2 &A, const Trace2 &B) {
    static const int P[3][2] = {{2, 0}, {1, 1}, {0, 2}};
    dd acc(0.0);
    for (int x = 0; x < 3; ++x)
        for (int y = 0; y < 3; ++y)
            acc += (A.u[x][0] * B.u[y][0] + A.u[x][1] * B.u[y][1]) * emom(P[x][0] + P[y][0], P[x][1] + P[y][1]);
    return acc;
}
dd tr_lq(const Trace2 &L, const Trace2 &Q) {       // (eps_L sA) . u_Q
    static const int P[3][2] = {{2, 0}, {1, 1}, {0, 2}};
    dd acc(0.0);
    for (int t = 0; t < 2; ++t)
        for (int y = 0; y < 3; ++y)
            acc += (L.en[t][0] * Q.u[y][0] + L.en[t][1] * Q.u[y][1]) * emom((t == 0) + P[y][0], (t == 1) + P[y][1]);
    return acc;
}

void assemble_vel2(const Mesh &m, const Space2 &s, const Params &p, const double *pot, const double *bpot,
                   Pattern &P, std::vector<double> &val) {
    const i64 nc = m.nc;
    std::vector<ElemV2> el(nc);
    std::vector<std::array<dd, 3>> wind(nc), bwind(nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < nc; ++c) {
        elemv2(m, c, el[c]);
        dd w[3];
        cell_wind(el[c].G, pot, w);
        wind[c] = {w[0], w[1], w[2]};
        dd b[3] = {dd(0.0), dd(0.0), dd(0.0)};
        if (bpot) cell_wind(el[c].G, bpot, b);
        bwind[c] = {b[0], b[1], b[2]};
    }
    // DoF -> entity, support cells
    std::vector<int> dkind(s.n), dent(s.n);
    for (i64 f = 0; f < m.nfacet; ++f)
        if (s.fdof[f] >= 0) for (int a = 0; a < 3; ++a) { dkind[s.fdof[f] + a] = 0; dent[s.fdof[f] + a] = (int)f; }
    for (i64 c = 0; c < nc; ++c) for (int a = 0; a < 3; ++a) { dkind[s.cdof[c] + a] = 1; dent[s.cdof[c] + a] = (int)c; }
    auto support = [&](i64 r, int *cells) -> int {
        if (dkind[r] == 1) { cells[0] = dent[r]; return 1; }
        const int f = dent[r];
        cells[0] = m.fcell[2 * f];
        if (m.fcell[2 * f + 1] >= 0) { cells[1] = m.fcell[2 * f + 1]; return 2; }
        return 1;
    };
    // pattern: DoFs of the support cells and of their facet neighbours
    P.rp.assign(s.n + 1, 0);
    std::vector<std::vector<int>> rows(s.n);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        int sc[2];
        const int ns = support(r, sc);
        std::vector<int> cols;
        for (int t = 0; t < ns; ++t) {
            int nb[4] = {sc[t], -1, -1, -1};
            for (int q = 0; q < 3; ++q) {
                const int f = m.cfacet[3 * sc[t] + q];
                nb[q + 1] = m.fcell[2 * f] == sc[t] ? m.fcell[2 * f + 1] : m.fcell[2 * f];
            }
            for (int u = 0; u < 4; ++u) {
                if (nb[u] < 0) continue;
                int g[12];
                cell_dofs_v2(m, s, nb[u], g);
                for (int k = 0; k < 12; ++k) if (g[k] >= 0) cols.push_back(g[k]);
            }
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        rows[r] = std::move(cols);
    }
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] = P.rp[r] + (i64)rows[r].size();
    P.ci.resize(P.rp[s.n]);
    for (i64 r = 0; r < s.n; ++r) std::copy(rows[r].begin(), rows[r].end(), P.ci.begin() + P.rp[r]);
    rows.clear();
    val.assign(P.rp[s.n], 0.0);
    const dd nu2 = dd(2.0) / dd(p.Re), pen = dd(p.sigma) / dd(p.Re);
#pragma omp parallel for schedule(dynamic, 128)
    for (i64 r = 0; r < s.n; ++r) {
        const i64 base = P.rp[r], len = P.rp[r + 1] - base;
        std::vector<dd> acc(len);
        auto add = [&](int col, const dd &v) { acc[find_col(P, r, col) - base] += v; };
        int sc[2];
        const int ns = support(r, sc);
        // cell terms
        for (int t = 0; t < ns; ++t) {
            const int c = sc[t];
            int g[12];
            cell_dofs_v2(m, s, c, g);
            int li = -1;
            for (int k = 0; k < 12; ++k) if (g[k] == r) li = k;
            dd row[12];
            const dd w[3] = {wind[c][0], wind[c][1], wind[c][2]}, b[3] = {bwind[c][0], bwind[c][1], bwind[c][2]};
            vel2_cell_row(el[c], li, w, b, bpot != nullptr, p, row);
            const dd twoK = dd(2.0) * el[c].G.vol;
            for (int k = 0; k < 12; ++k) if (g[k] >= 0) add(g[k], row[k] * twoK);
        }
        // facet terms of every facet of the support cells (ascending facet id)
        std::vector<int> fs;
        for (int t = 0; t < ns; ++t) for (int q = 0; q < 3; ++q) fs.push_back(m.cfacet[3 * sc[t] + q]);
        std::sort(fs.begin(), fs.end());
        fs.erase(std::unique(fs.begin(), fs.end()), fs.end());
        for (int f : fs) {
            const int cp = m.fcell[2 * f], cm = m.fcell[2 * f + 1];
            const bool interior = cm >= 0;
            const ElemV2 &Kp = el[cp];
            int qf = -1;
            for (int q = 0; q < 3; ++q) if (m.cfacet[3 * cp + q] == f) qf = q;
            dd A[3];
            int fl[3];
            facet_area(Kp.G, qf, A, fl);
            const double sg = facet_sign(Kp.G, qf, A, fl);
            const dd sA[2] = {dd(sg) * A[0], dd(sg) * A[1]};          // |f| n, n outward of K+
            const dd WA = wind[cp][0] * sA[0] + wind[cp][1] * sA[1];   // (w.n)|f|
            const dd aWA = WA.hi < 0 ? -WA : WA;
            const int v0 = m.ev[2 * f], v1 = m.ev[2 * f + 1];
            auto loc_of = [&](const ElemV2 &K, int v) { for (int a = 0; a < 3; ++a) if (K.G.v[a] == v) return a; return -1; };
            const dd avg = interior ? dd(0.5) : dd(1.0);
            const int sides = interior ? 2 : 1;
            const int cells[2] = {cp, cm};
            // test traces: every support cell of r on this facet (both, for r's own facet)
            for (int t = 0; t < ns; ++t) {
                const int ci_ = sc[t];
                if (ci_ != cp && ci_ != cm) continue;
                const int Ji = ci_ == cp ? 1 : -1;
                int gi[12];
                cell_dofs_v2(m, s, ci_, gi);
                int li = -1;
                for (int k = 0; k < 12; ++k) if (gi[k] == r) li = k;
                const ElemV2 &Ki = el[ci_];
                Trace2 Ti;
                vel2_trace(Ki, li, loc_of(Ki, v0), loc_of(Ki, v1), sA, Ti);
                for (int sd = 0; sd < sides; ++sd) {
                    const int cj = cells[sd];
                    const int Jj = sd == 0 ? 1 : -1;
                    const ElemV2 &Kj = el[cj];
                    const int a0 = loc_of(Kj, v0), a1 = loc_of(Kj, v1);
                    int gj[12];
                    cell_dofs_v2(m, s, cj, gj);
                    dd upc;
                    if (interior) upc = Jj > 0 ? (WA + aWA) * dd(0.5) : -((-WA + aWA) * dd(0.5));
                    else upc = (WA + aWA) * dd(0.5);
                    for (int j = 0; j < 12; ++j) {
                        if (gj[j] < 0) continue;
                        Trace2 Tj;
                        vel2_trace(Kj, j, a0, a1, sA, Tj);
                        const dd Q = tr_qq(Tj, Ti);
                        const dd E1 = tr_lq(Tj, Ti);       // (eps_j n) . v_i
                        const dd E2 = tr_lq(Ti, Tj);       // u_j . (eps_i n)
                        dd v = -(nu2 * avg * (dd((double)Ji) * E1 + dd((double)Jj) * E2)) +
                               pen * dd((double)(Jj * Ji)) * Q;
                        v += (interior ? upc * dd((double)Ji) : upc) * Q;
                        add(gj[j], v);
                    }
                }
            }
        }
        round_row(acc.data(), len, val.data() + base);
    }
}

void build_patches2_vel(const Mesh &m, const Space2 &s, std::vector<i64> &pptr, std::vector<int> &pdofs, std::vector<int> &pvert) {
    std::vector<std::vector<int>> vlist(m.nv);
    for (i64 f = 0; f < m.nfacet; ++f)
        if (s.fdof[f] >= 0)
            for (int t = 0; t < 2; ++t)
                for (int a = 0; a < 3; ++a) vlist[m.ev[2 * f + t]].push_back(s.fdof[f] + a);
    for (i64 c = 0; c < m.nc; ++c)
        for (int t = 0; t < 3; ++t)
            for (int a = 0; a < 3; ++a) vlist[m.cv[3 * c + t]].push_back(s.cdof[c] + a);
    pptr.assign(1, 0);
    pdofs.clear();
    pvert.clear();
    for (i64 v = 0; v < m.nv; ++v) {
        auto &L = vlist[v];
        if (L.empty()) continue;
        std::sort(L.begin(), L.end());
        pdofs.insert(pdofs.end(), L.begin(), L.end());
        pptr.push_back((i64)pdofs.size());
        pvert.push_back((int)v);
    }
}

void build_prolongation2_vel(const Mesh &mf, const Space2 &sf, const Mesh &mc, const Space2 &sc,
                             std::vector<i64> &rp, std::vector<int> &ci, std::vector<double> &vv) {
    std::vector<std::vector<std::pair<int, dd>>> rows(sf.n);
    std::vector<ElemV2> ce(mc.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < mc.nc; ++c) elemv2(mc, c, ce[c]);
    std::vector<int> owner(sf.n, INT32_MAX);
    for (i64 c = mf.nc - 1; c >= 0; --c) {
        int g[12];
        cell_dofs_v2(mf, sf, c, g);
        for (int t = 0; t < 12; ++t) if (g[t] >= 0) owner[g[t]] = (int)c;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 c = 0; c < mf.nc; ++c) {
        int g[12];
        cell_dofs_v2(mf, sf, c, g);
        bool any = false;
        for (int t = 0; t < 12; ++t) any = any || (g[t] >= 0 && owner[g[t]] == c);
        if (!any) continue;
        int Lf[4][3] = {{0}};
        int sum[2] = {0, 0};
        for (int a = 0; a < 3; ++a) {
            mf.lat(mf.cv[3 * c + a], Lf[a]);
            for (int r = 0; r < 2; ++r) sum[r] += Lf[a][r];
        }
        int cube[2], rel[2];
        for (int r = 0; r < 2; ++r) { cube[r] = sum[r] / 6; rel[r] = sum[r] - 6 * cube[r]; }
        const i64 sq = cube[0] + (i64)mc.N * cube[1];
        const i64 pc = rel[0] > rel[1] ? 2 * sq : 2 * sq + 1;
        const ElemV2 &Kc = ce[pc];
        int cg[12];
        cell_dofs_v2(mc, sc, pc, cg);
        GeoT<dd> Gf;
        cell_geo(mf, c, Gf);
        dd T[3][3];
        for (int b = 0; b < 3; ++b)
            for (int a = 0; a < 3; ++a) {
                dd v(b == 0 ? 1.0 : 0.0);
                for (int r = 0; r < 2; ++r) v += Kc.G.g[b][r] * (Gf.X[a][r] - Kc.G.X[0][r]);
                T[b][a] = v;
            }
        for (int j = 0; j < 12; ++j) {
            if (cg[j] < 0) continue;
            dd F[3][3][2];
            for (int r = 0; r < 2; ++r)
                for (int a = 0; a < 3; ++a)
                    for (int a2 = 0; a2 < 3; ++a2) {
                        dd acc(0.0);
                        for (int b = 0; b < 3; ++b)
                            for (int d2 = 0; d2 < 3; ++d2) acc += Kc.V[j][b][d2][r] * T[b][a] * T[d2][a2];
                        F[a][a2][r] = acc;
                    }
            dd out[12];
            bdm2_dofs(Gf, F, out);
            for (int t = 0; t < 12; ++t)
                if (g[t] >= 0 && owner[g[t]] == c) rows[g[t]].push_back({cg[j], out[t]});
        }
    }
    rp.assign(sf.n + 1, 0);
    std::vector<std::vector<std::pair<int, double>>> fin(sf.n);
    for (i64 I = 0; I < sf.n; ++I) {
        auto &R = rows[I];
        std::sort(R.begin(), R.end(), [](const std::pair<int, dd> &x, const std::pair<int, dd> &y) { return x.first < y.first; });
        std::vector<dd> xs(R.size());
        for (size_t t = 0; t < R.size(); ++t) xs[t] = R[t].second;
        std::vector<double> rounded(R.size());
        round_row(xs.data(), (i64)xs.size(), rounded.data());
        double mx = 0;
        for (double v : rounded) mx = std::max(mx, std::fabs(v));
        for (size_t t = 0; t < R.size(); ++t)
            if (rounded[t] != 0.0 && std::fabs(to_double(xs[t])) >= std::ldexp(mx, -30)) fin[I].push_back({R[t].first, rounded[t]});
        rp[I + 1] = rp[I] + (i64)fin[I].size();
    }
    ci.resize(rp[sf.n]);
    vv.resize(rp[sf.n]);
    for (i64 I = 0; I < sf.n; ++I)
        for (size_t t = 0; t < fin[I].size(); ++t) { ci[rp[I] + t] = fin[I][t].first; vv[rp[I] + t] = fin[I][t].second; }
}


// ---------------- k = 2 E-B block in 3D: NED1_2 x RT2 (reading R-basis2-3D, NEXT-2) ------
// DoFs: per edge e = (a < b), t_e = x_b - x_a: N_{e,s}(E) = int_e (E.t_e/|e|) lam_s ds
// (lam_0 = lam_a, lam_1 = lam_b); per face f = (a < b < c), t_0 = x_b - x_a, t_1 = x_c - x_a:
// N_{f,s}(E) = N int_f E.t_s dA; RT2: N_{f,s}(B) = int_f (B.n_f) lam_{v_s} dA (n_f of
// R-orient), per cell N_{K,r}(B) = N int_K B_r dx.  Numbering (R-num2): 2 per interior
// edge, 2 per interior face (E), then 3 per interior face, 3 per cell (B).  A field is
// stored as sum_p c_p lam^p over the 10 barycentric pairs p = (a <= b); every integral is
// closed-form: int_K lam^beta = 6|K| beta!/(|beta|+3)!, int_f mu^beta = 2|f| beta!/(|beta|+2)!,
// int_e mu^beta = |e| beta!/(|beta|+1)!.  Primal bases: the Arnold-Falk-Winther sets
// lam_i W_jk (j < k, i >= j; W Whitney 1-forms, 20) and lam_i phi_jkl (i >= j; phi
// Whitney 2-forms, 15), made dual to the DoFs by a double-double Gauss-Jordan.
namespace k2d3 {

static const int PA[10][2] = {{0, 0}, {0, 1}, {0, 2}, {0, 3}, {1, 1}, {1, 2}, {1, 3}, {2, 2}, {2, 3}, {3, 3}};
static const int PID[4][4] = {{0, 1, 2, 3}, {1, 4, 5, 6}, {2, 5, 7, 8}, {3, 6, 8, 9}};
static const int LE[6][2] = {{0, 1}, {0, 2}, {0, 3}, {1, 2}, {1, 3}, {2, 3}};

struct Q { dd c[10][3]; };     // vector field sum_p c_p lam^p

inline double bfact(std::initializer_list<int> idx) {   // beta! of a multiset of indices
    int n[4] = {0, 0, 0, 0};
    for (int i : idx) n[i]++;
    return fact(n[0]) * fact(n[1]) * fact(n[2]) * fact(n[3]);
}

struct Tabs {   // int_K lam^beta / (6|K|) = beta! / (|beta|+3)!
    dd m4[10][10], m3[10][4], m2[4][4];
    Tabs() {
        for (int p = 0; p < 10; ++p) {
            for (int q = 0; q < 10; ++q)
                m4[p][q] = dd(bfact({PA[p][0], PA[p][1], PA[q][0], PA[q][1]})) / dd(fact(7));
            for (int c = 0; c < 4; ++c) m3[p][c] = dd(bfact({PA[p][0], PA[p][1], c})) / dd(fact(6));
        }
        for (int a = 0; a < 4; ++a)
            for (int b = 0; b < 4; ++b) m2[a][b] = dd(bfact({a, b})) / dd(fact(5));
    }
};
const Tabs &tabs() { static const Tabs T; return T; }

struct Space3 {
    i64 n = 0, nE = 0;
    std::vector<int> edof, gdof, fdof, cdof;
};

void build_space3(Space3 &s, const Mesh &m) {
    s.edof.assign(m.ne, -1); s.gdof.assign(m.nf, -1); s.fdof.assign(m.nf, -1); s.cdof.assign(m.nc, -1);
    i64 n = 0;
    for (i64 e = 0; e < m.ne; ++e) if (!m.common_bnd(&m.ev[2 * e], 2)) { s.edof[e] = (int)n; n += 2; }
    for (i64 f = 0; f < m.nf; ++f) if (!m.common_bnd(&m.fv[3 * f], 3)) { s.gdof[f] = (int)n; n += 2; }
    s.nE = n;
    for (i64 f = 0; f < m.nf; ++f) if (!m.common_bnd(&m.fv[3 * f], 3)) { s.fdof[f] = (int)n; n += 3; }
    for (i64 c = 0; c < m.nc; ++c) { s.cdof[c] = (int)n; n += 3; }
    s.n = n;
}

// local order: E: edge q (LE order) x s, then face q (opposite vertex q) x s;
//              B: face q x s, then r
void cell_dofs3(const Mesh &m, const Space3 &s, i64 c, int *gE, int *gB) {
    for (int q = 0; q < 6; ++q) {
        const int e0 = s.edof[m.cedge[6 * c + q]];
        for (int t = 0; t < 2; ++t) gE[2 * q + t] = e0 < 0 ? -1 : e0 + t;
    }
    for (int q = 0; q < 4; ++q) {
        const int f = m.cfacet[4 * c + q], g0 = s.gdof[f], f0 = s.fdof[f];
        for (int t = 0; t < 2; ++t) gE[12 + 2 * q + t] = g0 < 0 ? -1 : g0 + t;
        for (int t = 0; t < 3; ++t) gB[3 * q + t] = f0 < 0 ? -1 : f0 + t;
    }
    for (int r = 0; r < 3; ++r) gB[12 + r] = s.cdof[c] + r;
}

inline void face_verts(int q, int *fl) { int t = 0; for (int a = 0; a < 4; ++a) if (a != q) fl[t++] = a; }

// the 20 NED1_2 functionals of F on cell G (farea[q] = |face q|)
void ned_fun(const GeoT<dd> &G, int Ncells, const dd *farea, const Q &F, dd *out) {
    for (int q = 0; q < 6; ++q) {
        const int v[2] = {LE[q][0], LE[q][1]};
        dd t[3];
        for (int r = 0; r < 3; ++r) t[r] = G.X[v[1]][r] - G.X[v[0]][r];
        for (int s = 0; s < 2; ++s) {
            dd acc(0.0);
            for (int x = 0; x < 2; ++x)
                for (int y = x; y < 2; ++y)
                    acc += dot3(F.c[PID[v[x]][v[y]]], t) * dd(bfact({v[x], v[y], v[s]}));
            out[2 * q + s] = acc / dd(24.0);
        }
    }
    for (int q = 0; q < 4; ++q) {
        int fl[3];
        face_verts(q, fl);
        dd t[2][3];
        for (int r = 0; r < 3; ++r) {
            t[0][r] = G.X[fl[1]][r] - G.X[fl[0]][r];
            t[1][r] = G.X[fl[2]][r] - G.X[fl[0]][r];
        }
        for (int s = 0; s < 2; ++s) {
            dd acc(0.0);
            for (int x = 0; x < 3; ++x)
                for (int y = x; y < 3; ++y) acc += dot3(F.c[PID[fl[x]][fl[y]]], t[s]) * dd(bfact({fl[x], fl[y]}));
            out[12 + 2 * q + s] = acc * dd((double)Ncells) * farea[q] / dd(12.0);
        }
    }
}

// the 15 RT2 functionals of F on cell G
void rt_fun(const GeoT<dd> &G, int Ncells, const Q &F, dd *out) {
    for (int q = 0; q < 4; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        for (int s = 0; s < 3; ++s) {
            dd acc(0.0);
            for (int x = 0; x < 3; ++x)
                for (int y = x; y < 3; ++y) acc += dot3(F.c[PID[fl[x]][fl[y]]], A) * dd(bfact({fl[x], fl[y], fl[s]}));
            out[3 * q + s] = acc / dd(60.0);
        }
    }
    for (int r = 0; r < 3; ++r) {
        dd acc(0.0);
        for (int p = 0; p < 10; ++p) acc += F.c[p][r] * dd(bfact({PA[p][0], PA[p][1]}));
        out[12 + r] = acc * dd((double)Ncells) * G.vol / dd(20.0);
    }
}

void add_pair(Q &F, int a, int b, const dd *v, double sgn) {
    dd *c = F.c[PID[a][b]];
    for (int r = 0; r < 3; ++r) c[r] += v[r] * dd(sgn);
}

// dual basis: B_j = sum_k Minv[k][j] p_k, M[i][j] = N_i(p_j)
template <int NB, class Fun>
void dualize(const Q *p, Fun fun, Q *B) {
    dd W[NB][2 * NB];
    for (int j = 0; j < NB; ++j) {
        dd col[NB];
        fun(p[j], col);
        for (int i = 0; i < NB; ++i) { W[i][j] = col[i]; W[i][NB + j] = dd(i == j ? 1.0 : 0.0); }
    }
    for (int k = 0; k < NB; ++k) {
        int piv = k;
        for (int i = k + 1; i < NB; ++i) if (std::fabs(W[i][k].hi) > std::fabs(W[piv][k].hi)) piv = i;
        if (piv != k) for (int j = 0; j < 2 * NB; ++j) std::swap(W[k][j], W[piv][j]);
        const dd d = W[k][k];
        for (int j = 0; j < 2 * NB; ++j) W[k][j] = W[k][j] / d;
        for (int i = 0; i < NB; ++i) {
            if (i == k) continue;
            const dd l = W[i][k];
            if (l.hi == 0.0 && l.lo == 0.0) continue;
            for (int j = 0; j < 2 * NB; ++j) W[i][j] = W[i][j] - l * W[k][j];
        }
    }
    for (int j = 0; j < NB; ++j) {
        memset((void *)&B[j], 0, sizeof(Q));
        for (int k = 0; k < NB; ++k)
            for (int pp = 0; pp < 10; ++pp)
                for (int r = 0; r < 3; ++r) B[j].c[pp][r] += W[k][NB + j] * p[k].c[pp][r];
    }
}

struct Elem3 {
    GeoT<dd> G;
    dd farea[4];
    Q E[20], B[15];
};

void elem3(const Mesh &m, i64 c, Elem3 &K) {
    cell_geo(m, c, K.G);
    const GeoT<dd> &G = K.G;
    for (int q = 0; q < 4; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        K.farea[q] = sqrt(dot3(A, A));
    }
    Q p[20];
    memset((void *)p, 0, sizeof p);
    int n = 0;
    for (int e = 0; e < 6; ++e) {                 // lam_i W_jk = lam_i lam_j g_k - lam_i lam_k g_j
        const int j = LE[e][0], k = LE[e][1];
        for (int i = j; i < 4; ++i, ++n) { add_pair(p[n], i, j, G.g[k], 1.0); add_pair(p[n], i, k, G.g[j], -1.0); }
    }
    dualize<20>(p, [&](const Q &F, dd *out) { ned_fun(G, m.N, K.farea, F, out); }, K.E);
    memset((void *)p, 0, sizeof p);
    n = 0;
    for (int q = 3; q >= 0; --q) {                // faces (j < k < l); lam_i phi_jkl, i >= j
        int fl[3];
        face_verts(q, fl);
        const int j = fl[0], k = fl[1], l = fl[2];
        dd kl[3], jl[3], jk[3];
        cross3(G.g[k], G.g[l], kl); cross3(G.g[j], G.g[l], jl); cross3(G.g[j], G.g[k], jk);
        for (int i = j; i < 4; ++i, ++n) {
            add_pair(p[n], i, j, kl, 1.0); add_pair(p[n], i, k, jl, -1.0); add_pair(p[n], i, l, jk, 1.0);
        }
    }
    dualize<15>(p, [&](const Q &F, dd *out) { rt_fun(G, m.N, F, out); }, K.B);
}

struct EBLocal3 {
    int gE[20], gB[15];
    dd EE[20][20], EB[20][15], BE[15][20], BB[15][15];
};

void eb_local3(const Mesh &m, const Space3 &s, i64 c, const double *pot, const Params &p, EBLocal3 &L) {
    Elem3 K;
    elem3(m, c, K);
    const GeoT<dd> &G = K.G;
    const Tabs &T = tabs();
    cell_dofs3(m, s, c, L.gE, L.gB);
    dd w[3];
    cell_wind(G, pot, w);
    const dd sixK = dd(6.0) * G.vol;
    // curl E_i = sum_c lam_c C[i][c]; div B_k = sum_c lam_c D[k][c]
    dd C[20][4][3], D[15][4];
    memset((void *)C, 0, sizeof C);
    memset((void *)D, 0, sizeof D);
    for (int pp = 0; pp < 10; ++pp) {
        const int a = PA[pp][0], b = PA[pp][1];
        for (int i = 0; i < 20; ++i) {
            dd ca[3], cb[3];
            cross3(G.g[a], K.E[i].c[pp], ca);
            cross3(G.g[b], K.E[i].c[pp], cb);
            for (int r = 0; r < 3; ++r) { C[i][b][r] += ca[r]; C[i][a][r] += cb[r]; }
        }
        for (int k = 0; k < 15; ++k) {
            D[k][b] += dot3(G.g[a], K.B[k].c[pp]);
            D[k][a] += dot3(G.g[b], K.B[k].c[pp]);
        }
    }
    // mass-weighted coefficients WE_i,p = sum_q m4[p][q] E_i,q (same for B); CW_i,p = sum_c m3[p][c] C_i,c
    static thread_local dd WE[20][10][3], WB[15][10][3], CW[20][10][3];
    for (int pp = 0; pp < 10; ++pp)
        for (int r = 0; r < 3; ++r) {
            for (int i = 0; i < 20; ++i) {
                dd acc(0.0), acc2(0.0);
                for (int qq = 0; qq < 10; ++qq) acc += T.m4[pp][qq] * K.E[i].c[qq][r];
                for (int cc = 0; cc < 4; ++cc) acc2 += T.m3[pp][cc] * C[i][cc][r];
                WE[i][pp][r] = acc;
                CW[i][pp][r] = acc2;
            }
            for (int k = 0; k < 15; ++k) {
                dd acc(0.0);
                for (int qq = 0; qq < 10; ++qq) acc += T.m4[pp][qq] * K.B[k].c[qq][r];
                WB[k][pp][r] = acc;
            }
        }
    for (int i = 0; i < 20; ++i)
        for (int j = 0; j < 20; ++j) {
            dd acc(0.0);
            for (int pp = 0; pp < 10; ++pp) acc += dot3(K.E[i].c[pp], WE[j][pp]);
            L.EE[i][j] = acc * sixK;
        }
    for (int k = 0; k < 15; ++k)
        for (int i = 0; i < 20; ++i) {
            dd ab(0.0), gt(0.0);
            for (int pp = 0; pp < 10; ++pp) {
                ab += dot3(K.B[k].c[pp], CW[i][pp]);
                if (!p.picard) {
                    dd wb[3];
                    cross3(w, K.B[k].c[pp], wb);
                    gt += dot3(wb, WE[i][pp]);
                }
            }
            ab = ab * sixK;
            gt = gt * sixK;
            L.BE[k][i] = ab;
            L.EB[i][k] = gt - ab / dd(p.Rem);
        }
    for (int k = 0; k < 15; ++k)
        for (int l = 0; l < 15; ++l) {
            dd dv(0.0);
            for (int a = 0; a < 4; ++a)
                for (int b = 0; b < 4; ++b) dv += D[k][a] * D[l][b] * T.m2[a][b];
            dd v = dv * sixK / dd(p.Rem);
            if (p.dt > 0) {
                dd ms(0.0);
                for (int pp = 0; pp < 10; ++pp) ms += dot3(K.B[k].c[pp], WB[l][pp]);
                v += ms * sixK / dd(p.dt);
            }
            L.BB[k][l] = v;
        }
}

// gather-form assembly by rows (cells of the row's entity, ascending), R-exact rows
void assemble_eb3(const Mesh &m, const Space3 &s, const Params &p, const double *pot, Pattern &P,
                  std::vector<double> &val) {
    std::vector<i64> ep, fp;
    std::vector<int> ec, fc;
    incidence(m, 1, ep, ec);
    incidence(m, 2, fp, fc);
    std::vector<int> dkind(s.n), dent(s.n);
    for (i64 e = 0; e < m.ne; ++e)
        if (s.edof[e] >= 0) for (int a = 0; a < 2; ++a) { dkind[s.edof[e] + a] = 1; dent[s.edof[e] + a] = (int)e; }
    for (i64 f = 0; f < m.nf; ++f) {
        if (s.gdof[f] >= 0) for (int a = 0; a < 2; ++a) { dkind[s.gdof[f] + a] = 2; dent[s.gdof[f] + a] = (int)f; }
        if (s.fdof[f] >= 0) for (int a = 0; a < 3; ++a) { dkind[s.fdof[f] + a] = 2; dent[s.fdof[f] + a] = (int)f; }
    }
    for (i64 c = 0; c < m.nc; ++c) for (int a = 0; a < 3; ++a) { dkind[s.cdof[c] + a] = 3; dent[s.cdof[c] + a] = (int)c; }
    std::vector<int> self(m.nc);
    std::iota(self.begin(), self.end(), 0);
    auto cells_of = [&](i64 row, const int *&b, const int *&e) {
        const int k = dkind[row], id = dent[row];
        if (k == 1) { b = ec.data() + ep[id]; e = ec.data() + ep[id + 1]; }
        else if (k == 2) { b = fc.data() + fp[id]; e = fc.data() + fp[id + 1]; }
        else { b = self.data() + id; e = b + 1; }
    };
    std::vector<EBLocal3> loc(m.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < m.nc; ++c) eb_local3(m, s, c, pot, p, loc[c]);
    P.rp.assign(s.n + 1, 0);
    std::vector<std::vector<int>> rows(s.n);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        std::vector<int> cols;
        for (const int *c = b; c != e; ++c) {
            for (int t = 0; t < 20; ++t) if (loc[*c].gE[t] >= 0) cols.push_back(loc[*c].gE[t]);
            for (int t = 0; t < 15; ++t) if (loc[*c].gB[t] >= 0) cols.push_back(loc[*c].gB[t]);
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        rows[r] = std::move(cols);
    }
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] = P.rp[r] + (i64)rows[r].size();
    P.ci.resize(P.rp[s.n]);
    for (i64 r = 0; r < s.n; ++r) std::copy(rows[r].begin(), rows[r].end(), P.ci.begin() + P.rp[r]);
    rows.clear();
    rows.shrink_to_fit();
    val.assign(P.rp[s.n], 0.0);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        const int *b, *e;
        cells_of(r, b, e);
        const i64 base = P.rp[r], len = P.rp[r + 1] - base;
        std::vector<dd> acc(len);
        const bool isB = r >= s.nE;
        for (const int *c = b; c != e; ++c) {
            const EBLocal3 &K = loc[*c];
            int li = -1;
            if (!isB) { for (int a = 0; a < 20; ++a) if (K.gE[a] == r) li = a; }
            else { for (int a = 0; a < 15; ++a) if (K.gB[a] == r) li = a; }
            auto add = [&](int col, const dd &v) { acc[find_col(P, r, col) - base] += v; };
            for (int j = 0; j < 20; ++j) if (K.gE[j] >= 0) add(K.gE[j], isB ? K.BE[li][j] : K.EE[li][j]);
            for (int j = 0; j < 15; ++j) if (K.gB[j] >= 0) add(K.gB[j], isB ? K.BB[li][j] : K.EB[li][j]);
        }
        round_row(acc.data(), len, val.data() + base);
    }
}

// vertex stars: DoFs of the edges, faces and cells containing the vertex, ascending
void build_patches3(const Mesh &m, const Space3 &s, std::vector<i64> &pptr, std::vector<int> &pdofs, std::vector<int> &pvert) {
    std::vector<std::vector<int>> vlist(m.nv);
    for (i64 e = 0; e < m.ne; ++e)
        if (s.edof[e] >= 0)
            for (int t = 0; t < 2; ++t) for (int a = 0; a < 2; ++a) vlist[m.ev[2 * e + t]].push_back(s.edof[e] + a);
    for (i64 f = 0; f < m.nf; ++f)
        for (int t = 0; t < 3; ++t) {
            auto &L = vlist[m.fv[3 * f + t]];
            if (s.gdof[f] >= 0) for (int a = 0; a < 2; ++a) L.push_back(s.gdof[f] + a);
            if (s.fdof[f] >= 0) for (int a = 0; a < 3; ++a) L.push_back(s.fdof[f] + a);
        }
    for (i64 c = 0; c < m.nc; ++c)
        for (int t = 0; t < 4; ++t) for (int a = 0; a < 3; ++a) vlist[m.cv[4 * c + t]].push_back(s.cdof[c] + a);
    pptr.assign(1, 0);
    pdofs.clear();
    pvert.clear();
    for (i64 v = 0; v < m.nv; ++v) {
        auto &L = vlist[v];
        if (L.empty()) continue;
        std::sort(L.begin(), L.end());
        pdofs.insert(pdofs.end(), L.begin(), L.end());
        pptr.push_back((i64)pdofs.size());
        pvert.push_back((int)v);
    }
}

// R-prol at k = 2 in 3D: coarse functions rewritten in the fine cell's barycentrics
// (lam^c_b = sum_a lam^c_b(X^f_a) lam^f_a), fine functionals in closed form; each fine DoF
// is computed by its owner (the lowest-index fine cell containing its entity); rows
// rounded as R-exact, |x| < 2^-30 max|row| dropped (R-prol2)
void build_prolongation3(const Mesh &mf, const Space3 &sf, const Mesh &mc, const Space3 &sc, std::vector<i64> &rp,
                         std::vector<int> &ci, std::vector<double> &vv) {
    static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    std::vector<std::vector<std::pair<int, dd>>> rows(sf.n);
    std::vector<Elem3> ce(mc.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < mc.nc; ++c) elem3(mc, c, ce[c]);
    std::vector<int> owner(sf.n, INT32_MAX);
    for (i64 c = mf.nc - 1; c >= 0; --c) {
        int gE[20], gB[15];
        cell_dofs3(mf, sf, c, gE, gB);
        for (int t = 0; t < 20; ++t) if (gE[t] >= 0) owner[gE[t]] = (int)c;
        for (int t = 0; t < 15; ++t) if (gB[t] >= 0) owner[gB[t]] = (int)c;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 c = 0; c < mf.nc; ++c) {
        int gE[20], gB[15];
        cell_dofs3(mf, sf, c, gE, gB);
        bool any = false;
        for (int t = 0; t < 20; ++t) any = any || (gE[t] >= 0 && owner[gE[t]] == c);
        for (int t = 0; t < 15; ++t) any = any || (gB[t] >= 0 && owner[gB[t]] == c);
        if (!any) continue;
        int Lf[4][3] = {{0}};
        int sum[3] = {0, 0, 0};
        for (int a = 0; a < 4; ++a) {
            mf.lat(mf.cv[4 * c + a], Lf[a]);
            for (int r = 0; r < 3; ++r) sum[r] += Lf[a][r];
        }
        int cube[3], rel[3];
        for (int r = 0; r < 3; ++r) { cube[r] = sum[r] / 8; rel[r] = sum[r] - 8 * cube[r]; }
        const i64 cb = cube[0] + (i64)mc.N * (cube[1] + (i64)mc.N * cube[2]);
        i64 pc = -1;
        for (int q = 0; q < 6; ++q)
            if (rel[PERM[q][0]] > rel[PERM[q][1]] && rel[PERM[q][1]] > rel[PERM[q][2]]) pc = 6 * cb + q;
        const Elem3 &Kc = ce[pc];
        int cE[20], cB[15];
        cell_dofs3(mc, sc, pc, cE, cB);
        GeoT<dd> Gf;
        cell_geo(mf, c, Gf);
        dd fa[4];
        for (int q = 0; q < 4; ++q) {
            dd A[3];
            int fl[3];
            facet_area(Gf, q, A, fl);
            fa[q] = sqrt(dot3(A, A));
        }
        dd T[4][4];                                 // T[b][a] = lam^c_b(X^f_a)
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a) {
                dd v(b == 0 ? 1.0 : 0.0);
                for (int r = 0; r < 3; ++r) v += Kc.G.g[b][r] * (Gf.X[a][r] - Kc.G.X[0][r]);
                T[b][a] = v;
            }
        auto to_fine = [&](const Q &in, Q &out) {
            memset((void *)&out, 0, sizeof(Q));
            for (int pp = 0; pp < 10; ++pp) {
                const int b = PA[pp][0], d2 = PA[pp][1];
                for (int a = 0; a < 4; ++a)
                    for (int a2 = 0; a2 < 4; ++a2) {
                        const dd tt = T[b][a] * T[d2][a2];
                        if (tt.hi == 0.0) continue;
                        dd *o = out.c[PID[a][a2]];
                        for (int r = 0; r < 3; ++r) o[r] += in.c[pp][r] * tt;
                    }
            }
        };
        for (int j = 0; j < 20; ++j) {
            if (cE[j] < 0) continue;
            Q F;
            to_fine(Kc.E[j], F);
            dd out[20];
            ned_fun(Gf, mf.N, fa, F, out);
            for (int t = 0; t < 20; ++t)
                if (gE[t] >= 0 && owner[gE[t]] == c) rows[gE[t]].push_back({cE[j], out[t]});
        }
        for (int j = 0; j < 15; ++j) {
            if (cB[j] < 0) continue;
            Q F;
            to_fine(Kc.B[j], F);
            dd out[15];
            rt_fun(Gf, mf.N, F, out);
            for (int t = 0; t < 15; ++t)
                if (gB[t] >= 0 && owner[gB[t]] == c) rows[gB[t]].push_back({cB[j], out[t]});
        }
    }
    rp.assign(sf.n + 1, 0);
    std::vector<std::vector<std::pair<int, double>>> fin(sf.n);
#pragma omp parallel for schedule(dynamic, 1024)
    for (i64 I = 0; I < sf.n; ++I) {
        auto &R = rows[I];
        std::sort(R.begin(), R.end(), [](const std::pair<int, dd> &x, const std::pair<int, dd> &y) { return x.first < y.first; });
        std::vector<dd> xs(R.size());
        for (size_t t = 0; t < R.size(); ++t) xs[t] = R[t].second;
        std::vector<double> rounded(R.size());
        round_row(xs.data(), (i64)xs.size(), rounded.data());
        double mx = 0;
        for (double v : rounded) mx = std::max(mx, std::fabs(v));
        for (size_t t = 0; t < R.size(); ++t)
            if (rounded[t] != 0.0 && std::fabs(to_double(xs[t])) >= std::ldexp(mx, -30)) fin[I].push_back({R[t].first, rounded[t]});
    }
    for (i64 I = 0; I < sf.n; ++I) rp[I + 1] = rp[I] + (i64)fin[I].size();
    ci.resize(rp[sf.n]);
    vv.resize(rp[sf.n]);
    for (i64 I = 0; I < sf.n; ++I)
        for (size_t t = 0; t < fin[I].size(); ++t) { ci[rp[I] + t] = fin[I][t].first; vv[rp[I] + t] = fin[I][t].second; }
}


// ---------------- k = 2 AL velocity block in 3D: BDM2 (R-basis2-vel in 3D, NEXT-2) ---------
// DoFs: per face f (vertices a < b < c, area vector A of R-orient) N_{f,s}(u) = u(x_s) . A
// at the P2 nodes x_0..2 = x_a, x_b, x_c, x_3 = mid(a,b), x_4 = mid(a,c), x_5 = mid(b,c);
// per cell N_{K,e}(u) = int_K u . (lam_i g_j - lam_j g_i), e = (i < j) in LE order.
// Free DoFs: 6 per interior face (face order), then 6 per cell.  Primal basis
// lam_a lam_b e_r (30), dual by the double-double Gauss-Jordan.  Forms of R-vel with
// closed-form cell (6|K| beta!/(|beta|+3)!) and face (2|f| beta!/(|beta|+2)!) moments;
// h_F = longest face edge, as the k = 1 3D assembly.
struct SpaceV3 {
    i64 n = 0;
    std::vector<int> fdof, cdof;
};

void build_space_v3(SpaceV3 &s, const Mesh &m) {
    s.fdof.assign(m.nf, -1); s.cdof.assign(m.nc, -1);
    i64 n = 0;
    for (i64 f = 0; f < m.nf; ++f) if (!m.common_bnd(&m.fv[3 * f], 3)) { s.fdof[f] = (int)n; n += 6; }
    for (i64 c = 0; c < m.nc; ++c) { s.cdof[c] = (int)n; n += 6; }
    s.n = n;
}

// local order: face q (opposite vertex q) x s = 0..5, then e = 0..5
void cell_dofs_v3(const Mesh &m, const SpaceV3 &s, i64 c, int *g) {
    for (int q = 0; q < 4; ++q) {
        const int f0 = s.fdof[m.cfacet[4 * c + q]];
        for (int t = 0; t < 6; ++t) g[6 * q + t] = f0 < 0 ? -1 : f0 + t;
    }
    for (int e = 0; e < 6; ++e) g[24 + e] = s.cdof[c] + e;
}

static const int FP[6][2] = {{0, 0}, {0, 1}, {0, 2}, {1, 1}, {1, 2}, {2, 2}};   // face pairs
static const int NODE[6][2] = {{0, 0}, {1, 1}, {2, 2}, {0, 1}, {0, 2}, {1, 2}};  // P2 face nodes

void bdm3_fun(const GeoT<dd> &G, const Q &F, dd *out) {
    const Tabs &T = tabs();
    for (int q = 0; q < 4; ++q) {
        dd A[3];
        int fl[3];
        facet_area(G, q, A, fl);
        for (int s = 0; s < 6; ++s) {
            const int x = fl[NODE[s][0]], y = fl[NODE[s][1]];
            dd u[3];
            if (x == y) for (int r = 0; r < 3; ++r) u[r] = F.c[PID[x][x]][r];
            else
                for (int r = 0; r < 3; ++r) u[r] = (F.c[PID[x][x]][r] + F.c[PID[x][y]][r] + F.c[PID[y][y]][r]) * dd(0.25);
            out[6 * q + s] = dot3(u, A);
        }
    }
    for (int e = 0; e < 6; ++e) {
        const int i = LE[e][0], j = LE[e][1];
        dd acc(0.0);
        for (int p = 0; p < 10; ++p)
            acc += dot3(F.c[p], G.g[j]) * T.m3[p][i] - dot3(F.c[p], G.g[i]) * T.m3[p][j];
        out[24 + e] = acc * dd(6.0) * G.vol;
    }
}

struct ElemV3 {
    GeoT<dd> G;
    Q V[30];
    dd Gr[30][4][3][3];      // grad (row l = component, col k = direction) = sum_c lam_c Gr[c]
};

void elemv3(const Mesh &m, i64 c, ElemV3 &K) {
    cell_geo(m, c, K.G);
    const GeoT<dd> &G = K.G;
    Q p[30];
    memset((void *)p, 0, sizeof p);
    for (int pp = 0; pp < 10; ++pp)
        for (int r = 0; r < 3; ++r) p[3 * pp + r].c[pp][r] = dd(1.0);
    dualize<30>(p, [&](const Q &F, dd *out) { bdm3_fun(G, F, out); }, K.V);
    memset((void *)K.Gr, 0, sizeof K.Gr);
    for (int j = 0; j < 30; ++j)
        for (int pp = 0; pp < 10; ++pp) {
            const int a = PA[pp][0], b = PA[pp][1];
            for (int l = 0; l < 3; ++l)
                for (int k = 0; k < 3; ++k) {
                    K.Gr[j][b][l][k] += K.V[j].c[pp][l] * G.g[a][k];
                    K.Gr[j][a][l][k] += K.V[j].c[pp][l] * G.g[b][k];
                }
        }
}

// row li of the cell matrix (test li, trial j = 0..29), without 6|K|
void vel3_cell_row(const ElemV3 &K, int li, const dd *w, const dd *bx, bool lorentz, const Params &p, dd *row) {
    const Tabs &T = tabs();
    const dd nu2 = dd(2.0) / dd(p.Re);
    dd epi[4][3][3], gwi[4][3], divi[4];
    for (int cc = 0; cc < 4; ++cc) {
        for (int l = 0; l < 3; ++l)
            for (int k = 0; k < 3; ++k) epi[cc][l][k] = (K.Gr[li][cc][l][k] + K.Gr[li][cc][k][l]) * dd(0.5);
        for (int l = 0; l < 3; ++l) gwi[cc][l] = K.Gr[li][cc][l][0] * w[0] + K.Gr[li][cc][l][1] * w[1] + K.Gr[li][cc][l][2] * w[2];
        divi[cc] = K.Gr[li][cc][0][0] + K.Gr[li][cc][1][1] + K.Gr[li][cc][2][2];
    }
    // test side contracted with the moment tables once per row
    dd Me[4][3][3], Md[4], Ga[10][3], Mv[10][3], Mb[10][3];
    for (int c1 = 0; c1 < 4; ++c1) {
        dd d(0.0);
        for (int c2 = 0; c2 < 4; ++c2) d += T.m2[c1][c2] * divi[c2];
        Md[c1] = d;
        for (int l = 0; l < 3; ++l)
            for (int k = 0; k < 3; ++k) {
                dd e(0.0);
                for (int c2 = 0; c2 < 4; ++c2) e += T.m2[c1][c2] * epi[c2][l][k];
                Me[c1][l][k] = e;
            }
    }
    dd vxb_i[10][3];
    if (lorentz) for (int q = 0; q < 10; ++q) cross3(K.V[li].c[q], bx, vxb_i[q]);
    for (int pp = 0; pp < 10; ++pp)
        for (int r = 0; r < 3; ++r) {
            dd a(0.0), mv(0.0), mb(0.0);
            for (int cc = 0; cc < 4; ++cc) a += T.m3[pp][cc] * gwi[cc][r];
            for (int q = 0; q < 10; ++q) {
                mv += T.m4[pp][q] * K.V[li].c[q][r];
                if (lorentz) mb += T.m4[pp][q] * vxb_i[q][r];
            }
            Ga[pp][r] = a; Mv[pp][r] = mv; Mb[pp][r] = mb;
        }
    for (int j = 0; j < 30; ++j) {
        dd ee(0.0), dv(0.0), adv(0.0), ms(0.0), lor(0.0);
        for (int c1 = 0; c1 < 4; ++c1) {
            const dd divj = K.Gr[j][c1][0][0] + K.Gr[j][c1][1][1] + K.Gr[j][c1][2][2];
            for (int l = 0; l < 3; ++l)
                for (int k = 0; k < 3; ++k) ee += (K.Gr[j][c1][l][k] + K.Gr[j][c1][k][l]) * dd(0.5) * Me[c1][l][k];
            dv += divj * Md[c1];
        }
        for (int pp = 0; pp < 10; ++pp) {
            adv += dot3(K.V[j].c[pp], Ga[pp]);
            if (p.dt > 0) ms += dot3(K.V[j].c[pp], Mv[pp]);
            if (lorentz) {
                dd vxb_j[3];
                cross3(K.V[j].c[pp], bx, vxb_j);
                lor += dot3(vxb_j, Mb[pp]);
            }
        }
        dd v = nu2 * ee - adv + dd(p.gamma) * dv;
        if (p.dt > 0) v += ms / dd(p.dt);
        if (lorentz) v += dd(p.S) * lor;
        row[j] = v;
    }
}

// trace of basis function j of K on a face with cell-local vertices a[0..2] (ascending
// global id): quadratic u on the 6 face pairs, linear eps(u) sA on the 3 face vertices
struct Trace3 { dd u[6][3]; dd en[3][3]; };

void vel3_trace(const ElemV3 &K, int j, const int *a, const dd *sA, Trace3 &T) {
    for (int x = 0; x < 6; ++x)
        for (int r = 0; r < 3; ++r) T.u[x][r] = K.V[j].c[PID[a[FP[x][0]]][a[FP[x][1]]]][r];
    for (int t = 0; t < 3; ++t)
        for (int l = 0; l < 3; ++l) {
            dd acc(0.0);
            for (int k = 0; k < 3; ++k) acc += (K.Gr[j][a[t]][l][k] + K.Gr[j][a[t]][k][l]) * sA[k];
            T.en[t][l] = acc * dd(0.5);
        }
}

// int_f mu^beta / |f| = 2 beta! / (|beta| + 2)!
inline dd fmom(int n0, int n1, int n2) {
    return dd(2.0 * fact(n0) * fact(n1) * fact(n2)) / dd(fact(n0 + n1 + n2 + 2));
}
struct FaceTabs {      // fmom of (pair x, pair y) and of (vertex t, pair y)
    dd qq[6][6], lq[3][6];
    FaceTabs() {
        for (int x = 0; x < 6; ++x)
            for (int y = 0; y < 6; ++y) {
                int n[3] = {0, 0, 0};
                n[FP[x][0]]++; n[FP[x][1]]++; n[FP[y][0]]++; n[FP[y][1]]++;
                qq[x][y] = fmom(n[0], n[1], n[2]);
                if (x < 3) {
                    int k[3] = {0, 0, 0};
                    k[x]++; k[FP[y][0]]++; k[FP[y][1]]++;
                    lq[x][y] = fmom(k[0], k[1], k[2]);
                }
            }
    }
};
const FaceTabs &face_tabs() { static const FaceTabs T; return T; }
dd tr3_qq(const Trace3 &A, const Trace3 &B) {
    const FaceTabs &T = face_tabs();
    dd acc(0.0);
    for (int x = 0; x < 6; ++x)
        for (int y = 0; y < 6; ++y) acc += dot3(A.u[x], B.u[y]) * T.qq[x][y];
    return acc;
}
dd tr3_lq(const Trace3 &L, const Trace3 &Qt) {       // (eps_L sA) . u_Q
    const FaceTabs &T = face_tabs();
    dd acc(0.0);
    for (int t = 0; t < 3; ++t)
        for (int y = 0; y < 6; ++y) acc += dot3(L.en[t], Qt.u[y]) * T.lq[t][y];
    return acc;
}

void assemble_vel3(const Mesh &m, const SpaceV3 &s, const Params &p, const double *pot, const double *bpot, Pattern &P,
                   std::vector<double> &val) {
    const i64 nc = m.nc;
    std::vector<ElemV3> el(nc);
    std::vector<std::array<dd, 3>> wind(nc), bwind(nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < nc; ++c) {
        elemv3(m, c, el[c]);
        dd w[3];
        cell_wind(el[c].G, pot, w);
        wind[c] = {w[0], w[1], w[2]};
        dd b[3] = {dd(0.0), dd(0.0), dd(0.0)};
        if (bpot) cell_wind(el[c].G, bpot, b);
        bwind[c] = {b[0], b[1], b[2]};
    }
    std::vector<int> dkind(s.n), dent(s.n);
    for (i64 f = 0; f < m.nf; ++f)
        if (s.fdof[f] >= 0) for (int a = 0; a < 6; ++a) { dkind[s.fdof[f] + a] = 0; dent[s.fdof[f] + a] = (int)f; }
    for (i64 c = 0; c < nc; ++c) for (int a = 0; a < 6; ++a) { dkind[s.cdof[c] + a] = 1; dent[s.cdof[c] + a] = (int)c; }
    auto support = [&](i64 r, int *cells) -> int {
        if (dkind[r] == 1) { cells[0] = dent[r]; return 1; }
        const int f = dent[r];
        cells[0] = m.fcell[2 * f];
        if (m.fcell[2 * f + 1] >= 0) { cells[1] = m.fcell[2 * f + 1]; return 2; }
        return 1;
    };
    P.rp.assign(s.n + 1, 0);
    std::vector<std::vector<int>> rows(s.n);
#pragma omp parallel for schedule(dynamic, 256)
    for (i64 r = 0; r < s.n; ++r) {
        int sc[2];
        const int ns = support(r, sc);
        std::vector<int> cols;
        for (int t = 0; t < ns; ++t) {
            int nb[5] = {sc[t], -1, -1, -1, -1};
            for (int q = 0; q < 4; ++q) {
                const int f = m.cfacet[4 * sc[t] + q];
                nb[q + 1] = m.fcell[2 * f] == sc[t] ? m.fcell[2 * f + 1] : m.fcell[2 * f];
            }
            for (int u = 0; u < 5; ++u) {
                if (nb[u] < 0) continue;
                int g[30];
                cell_dofs_v3(m, s, nb[u], g);
                for (int k = 0; k < 30; ++k) if (g[k] >= 0) cols.push_back(g[k]);
            }
        }
        std::sort(cols.begin(), cols.end());
        cols.erase(std::unique(cols.begin(), cols.end()), cols.end());
        rows[r] = std::move(cols);
    }
    for (i64 r = 0; r < s.n; ++r) P.rp[r + 1] = P.rp[r] + (i64)rows[r].size();
    P.ci.resize(P.rp[s.n]);
    for (i64 r = 0; r < s.n; ++r) std::copy(rows[r].begin(), rows[r].end(), P.ci.begin() + P.rp[r]);
    rows.clear();
    rows.shrink_to_fit();
    val.assign(P.rp[s.n], 0.0);
    const dd nu2 = dd(2.0) / dd(p.Re);
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 r = 0; r < s.n; ++r) {
        const i64 base = P.rp[r], len = P.rp[r + 1] - base;
        std::vector<dd> acc(len);
        auto add = [&](int col, const dd &v) { acc[find_col(P, r, col) - base] += v; };
        int sc[2];
        const int ns = support(r, sc);
        for (int t = 0; t < ns; ++t) {
            const int c = sc[t];
            int g[30];
            cell_dofs_v3(m, s, c, g);
            int li = -1;
            for (int k = 0; k < 30; ++k) if (g[k] == r) li = k;
            dd row[30];
            const dd w[3] = {wind[c][0], wind[c][1], wind[c][2]}, b[3] = {bwind[c][0], bwind[c][1], bwind[c][2]};
            vel3_cell_row(el[c], li, w, b, bpot != nullptr, p, row);
            const dd sixK = dd(6.0) * el[c].G.vol;
            for (int k = 0; k < 30; ++k) if (g[k] >= 0) add(g[k], row[k] * sixK);
        }
        std::vector<int> fs;
        for (int t = 0; t < ns; ++t) for (int q = 0; q < 4; ++q) fs.push_back(m.cfacet[4 * sc[t] + q]);
        std::sort(fs.begin(), fs.end());
        fs.erase(std::unique(fs.begin(), fs.end()), fs.end());
        for (int f : fs) {
            const int cp = m.fcell[2 * f], cm = m.fcell[2 * f + 1];
            const bool interior = cm >= 0;
            const ElemV3 &Kp = el[cp];
            int qf = -1;
            for (int q = 0; q < 4; ++q) if (m.cfacet[4 * cp + q] == f) qf = q;
            dd A[3];
            int fl[3];
            facet_area(Kp.G, qf, A, fl);
            const double sg = facet_sign(Kp.G, qf, A, fl);
            const dd sA[3] = {dd(sg) * A[0], dd(sg) * A[1], dd(sg) * A[2]};   // |f| n, n outward of K+
            const dd WA = wind[cp][0] * sA[0] + wind[cp][1] * sA[1] + wind[cp][2] * sA[2];
            const dd aWA = WA.hi < 0 ? -WA : WA;
            dd hF(0.0);
            for (int x = 0; x < 3; ++x)
                for (int y = x + 1; y < 3; ++y) {
                    dd t[3];
                    for (int k = 0; k < 3; ++k) t[k] = Kp.G.X[fl[y]][k] - Kp.G.X[fl[x]][k];
                    const dd l = sqrt(dot3(t, t));
                    if (hF < l) hF = l;
                }
            const dd pen = dd(p.sigma) / dd(p.Re) * sqrt(dot3(A, A)) / hF;     // sigma/(Re h_F) |f|
            const int fvv[3] = {m.fv[3 * f], m.fv[3 * f + 1], m.fv[3 * f + 2]};
            auto locs = [&](const ElemV3 &K, int *a) {
                for (int t = 0; t < 3; ++t) for (int b = 0; b < 4; ++b) if (K.G.v[b] == fvv[t]) a[t] = b;
            };
            const dd avg = interior ? dd(0.5) : dd(1.0);
            const int sides = interior ? 2 : 1;
            const int cells[2] = {cp, cm};
            for (int t = 0; t < ns; ++t) {
                const int ci_ = sc[t];
                if (ci_ != cp && ci_ != cm) continue;
                const int Ji = ci_ == cp ? 1 : -1;
                int gi[30];
                cell_dofs_v3(m, s, ci_, gi);
                int li = -1;
                for (int k = 0; k < 30; ++k) if (gi[k] == r) li = k;
                const ElemV3 &Ki = el[ci_];
                int ai[3];
                locs(Ki, ai);
                Trace3 Ti;
                vel3_trace(Ki, li, ai, sA, Ti);
                // test side contracted once: Q = sum_x u_j[x].Wq[x], E1 = sum_t en_j[t].Zl[t],
                // E2 = sum_y u_j[y].Yl[y]  (tr3_qq(Tj, Ti), tr3_lq(Tj, Ti), tr3_lq(Ti, Tj))
                const FaceTabs &FT = face_tabs();
                dd Wq[6][3], Zl[3][3], Yl[6][3];
                for (int x = 0; x < 6; ++x)
                    for (int r2 = 0; r2 < 3; ++r2) {
                        dd a1(0.0), a2(0.0);
                        for (int y = 0; y < 6; ++y) a1 += FT.qq[x][y] * Ti.u[y][r2];
                        for (int t2 = 0; t2 < 3; ++t2) a2 += FT.lq[t2][x] * Ti.en[t2][r2];
                        Wq[x][r2] = a1;
                        Yl[x][r2] = a2;
                    }
                for (int t2 = 0; t2 < 3; ++t2)
                    for (int r2 = 0; r2 < 3; ++r2) {
                        dd a1(0.0);
                        for (int y = 0; y < 6; ++y) a1 += FT.lq[t2][y] * Ti.u[y][r2];
                        Zl[t2][r2] = a1;
                    }
                for (int sd = 0; sd < sides; ++sd) {
                    const int cj = cells[sd];
                    const int Jj = sd == 0 ? 1 : -1;
                    const ElemV3 &Kj = el[cj];
                    int aj[3];
                    locs(Kj, aj);
                    int gj[30];
                    cell_dofs_v3(m, s, cj, gj);
                    dd upc;
                    if (interior) upc = Jj > 0 ? (WA + aWA) * dd(0.5) : -((-WA + aWA) * dd(0.5));
                    else upc = (WA + aWA) * dd(0.5);
                    for (int j = 0; j < 30; ++j) {
                        if (gj[j] < 0) continue;
                        Trace3 Tj;
                        vel3_trace(Kj, j, aj, sA, Tj);
                        dd Qv(0.0), E1(0.0), E2(0.0);
                        for (int y = 0; y < 6; ++y) { Qv += dot3(Tj.u[y], Wq[y]); E2 += dot3(Tj.u[y], Yl[y]); }
                        for (int t2 = 0; t2 < 3; ++t2) E1 += dot3(Tj.en[t2], Zl[t2]);
                        dd v = -(nu2 * avg * (dd((double)Ji) * E1 + dd((double)Jj) * E2)) + pen * dd((double)(Jj * Ji)) * Qv;
                        v += (interior ? upc * dd((double)Ji) : upc) * Qv;
                        add(gj[j], v);
                    }
                }
            }
        }
        round_row(acc.data(), len, val.data() + base);
    }
}

void build_patches_v3(const Mesh &m, const SpaceV3 &s, std::vector<i64> &pptr, std::vector<int> &pdofs, std::vector<int> &pvert) {
    std::vector<std::vector<int>> vlist(m.nv);
    for (i64 f = 0; f < m.nf; ++f)
        if (s.fdof[f] >= 0)
            for (int t = 0; t < 3; ++t) for (int a = 0; a < 6; ++a) vlist[m.fv[3 * f + t]].push_back(s.fdof[f] + a);
    for (i64 c = 0; c < m.nc; ++c)
        for (int t = 0; t < 4; ++t) for (int a = 0; a < 6; ++a) vlist[m.cv[4 * c + t]].push_back(s.cdof[c] + a);
    pptr.assign(1, 0);
    pdofs.clear();
    pvert.clear();
    for (i64 v = 0; v < m.nv; ++v) {
        auto &L = vlist[v];
        if (L.empty()) continue;
        std::sort(L.begin(), L.end());
        pdofs.insert(pdofs.end(), L.begin(), L.end());
        pptr.push_back((i64)pdofs.size());
        pvert.push_back((int)v);
    }
}

void build_prolongation_v3(const Mesh &mf, const SpaceV3 &sf, const Mesh &mc, const SpaceV3 &sc, std::vector<i64> &rp,
                           std::vector<int> &ci, std::vector<double> &vv) {
    static const int PERM[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
    std::vector<std::vector<std::pair<int, dd>>> rows(sf.n);
    std::vector<ElemV3> ce(mc.nc);
#pragma omp parallel for schedule(static)
    for (i64 c = 0; c < mc.nc; ++c) elemv3(mc, c, ce[c]);
    std::vector<int> owner(sf.n, INT32_MAX);
    for (i64 c = mf.nc - 1; c >= 0; --c) {
        int g[30];
        cell_dofs_v3(mf, sf, c, g);
        for (int t = 0; t < 30; ++t) if (g[t] >= 0) owner[g[t]] = (int)c;
    }
#pragma omp parallel for schedule(dynamic, 64)
    for (i64 c = 0; c < mf.nc; ++c) {
        int g[30];
        cell_dofs_v3(mf, sf, c, g);
        bool any = false;
        for (int t = 0; t < 30; ++t) any = any || (g[t] >= 0 && owner[g[t]] == c);
        if (!any) continue;
        int Lf[4][3] = {{0}};
        int sum[3] = {0, 0, 0};
        for (int a = 0; a < 4; ++a) {
            mf.lat(mf.cv[4 * c + a], Lf[a]);
            for (int r = 0; r < 3; ++r) sum[r] += Lf[a][r];
        }
        int cube[3], rel[3];
        for (int r = 0; r < 3; ++r) { cube[r] = sum[r] / 8; rel[r] = sum[r] - 8 * cube[r]; }
        const i64 cb = cube[0] + (i64)mc.N * (cube[1] + (i64)mc.N * cube[2]);
        i64 pc = -1;
        for (int q = 0; q < 6; ++q)
            if (rel[PERM[q][0]] > rel[PERM[q][1]] && rel[PERM[q][1]] > rel[PERM[q][2]]) pc = 6 * cb + q;
        const ElemV3 &Kc = ce[pc];
        int cg[30];
        cell_dofs_v3(mc, sc, pc, cg);
        GeoT<dd> Gf;
        cell_geo(mf, c, Gf);
        dd T[4][4];
        for (int b = 0; b < 4; ++b)
            for (int a = 0; a < 4; ++a) {
                dd v(b == 0 ? 1.0 : 0.0);
                for (int r = 0; r < 3; ++r) v += Kc.G.g[b][r] * (Gf.X[a][r] - Kc.G.X[0][r]);
                T[b][a] = v;
            }
        for (int j = 0; j < 30; ++j) {
            if (cg[j] < 0) continue;
            Q F;
            memset((void *)&F, 0, sizeof(Q));
            for (int pp = 0; pp < 10; ++pp) {
                const int b = PA[pp][0], d2 = PA[pp][1];
                for (int a = 0; a < 4; ++a)
                    for (int a2 = 0; a2 < 4; ++a2) {
                        const dd tt = T[b][a] * T[d2][a2];
                        if (tt.hi == 0.0) continue;
                        for (int r = 0; r < 3; ++r) F.c[PID[a][a2]][r] += Kc.V[j].c[pp][r] * tt;
                    }
            }
            dd out[30];
            bdm3_fun(Gf, F, out);
            for (int t = 0; t < 30; ++t)
                if (g[t] >= 0 && owner[g[t]] == c) rows[g[t]].push_back({cg[j], out[t]});
        }
    }
    rp.assign(sf.n + 1, 0);
    std::vector<std::vector<std::pair<int, double>>> fin(sf.n);
#pragma omp parallel for schedule(dynamic, 1024)
    for (i64 I = 0; I < sf.n; ++I) {
        auto &R = rows[I];
        std::sort(R.begin(), R.end(), [](const std::pair<int, dd> &x, const std::pair<int, dd> &y) { return x.first < y.first; });
        std::vector<dd> xs(R.size());
        for (size_t t = 0; t < R.size(); ++t) xs[t] = R[t].second;
        std::vector<double> rounded(R.size());
        round_row(xs.data(), (i64)xs.size(), rounded.data());
        double mx = 0;
        for (double v : rounded) mx = std::max(mx, std::fabs(v));
        for (size_t t = 0; t < R.size(); ++t)
            if (rounded[t] != 0.0 && std::fabs(to_double(xs[t])) >= std::ldexp(mx, -30)) fin[I].push_back({R[t].first, rounded[t]});
    }
    for (i64 I = 0; I < sf.n; ++I) rp[I + 1] = rp[I] + (i64)fin[I].size();
    ci.resize(rp[sf.n]);
    vv.resize(rp[sf.n]);
    for (i64 I = 0; I < sf.n; ++I)
        for (size_t t = 0; t < fin[I].size(); ++t) { ci[rp[I] + t] = fin[I][t].first; vv[rp[I] + t] = fin[I][t].second; }
}

}  // namespace k2d3

}  // namespace

std::string assemble_hierarchy(int block, int dim, int N, int nlev, const Params &p, const double *w,
                               const double *bn, std::vector<HostLevel> &out) {
    if ((block != 0 && block != 1) || (dim != 2 && dim != 3) || N < 1 || nlev < 1) return "bad arguments";
    if (N % (1 << (nlev - 1))) return "N not divisible by 2^(nlev-1)";
    if (p.degree != 1 && p.degree != 2) return "degree must be 1 or 2";
    out.assign(nlev, HostLevel());
    if (p.degree == 2 && dim == 3 && block == 1) {
        std::vector<Mesh> meshes(nlev);
        std::vector<k2d3::SpaceV3> spaces(nlev);
        for (int l = nlev - 1; l >= 0; --l) {
            const int Nl = N >> (nlev - 1 - l), step = 1 << (nlev - 1 - l);
            Mesh &m = meshes[l];
            build_mesh(m, dim, Nl);
            k2d3::build_space_v3(spaces[l], m);
            std::vector<double> pot(3 * m.nv), bpot(bn ? 3 * m.nv : 0);
            for (i64 v = 0; v < m.nv; ++v) {
                int q[3];
                m.lat(v, q);
                const i64 fv = q[0] * step + (i64)(N + 1) * (q[1] * step + (i64)(N + 1) * (q[2] * step));
                for (int t = 0; t < 3; ++t) pot[3 * v + t] = w[3 * fv + t];
                if (bn) for (int t = 0; t < 3; ++t) bpot[3 * v + t] = bn[3 * fv + t];
            }
            Pattern P;
            std::vector<double> val;
            k2d3::assemble_vel3(m, spaces[l], p, pot.data(), bn ? bpot.data() : nullptr, P, val);
            HostLevel &H = out[l];
            H.n = spaces[l].n;
            H.rp = std::move(P.rp);
            H.ci = std::move(P.ci);
            H.v = std::move(val);
            if (l > 0) k2d3::build_patches_v3(m, spaces[l], H.pptr, H.pdofs, H.pvert);
        }
        for (int l = 1; l < nlev; ++l) {
            k2d3::build_prolongation_v3(meshes[l], spaces[l], meshes[l - 1], spaces[l - 1], out[l].prp, out[l].pci,
                                        out[l].pv);
            out[l].n_coarser = spaces[l - 1].n;
        }
        return "";
    }
    if (p.degree == 2 && dim == 3) {
        std::vector<Mesh> meshes(nlev);
        std::vector<k2d3::Space3> spaces(nlev);
        for (int l = nlev - 1; l >= 0; --l) {
            const int Nl = N >> (nlev - 1 - l), step = 1 << (nlev - 1 - l);
            Mesh &m = meshes[l];
            build_mesh(m, dim, Nl);
            k2d3::build_space3(spaces[l], m);
            std::vector<double> pot(3 * m.nv);
            for (i64 v = 0; v < m.nv; ++v) {
                int q[3];
                m.lat(v, q);
                const i64 fv = q[0] * step + (i64)(N + 1) * (q[1] * step + (i64)(N + 1) * (q[2] * step));
                for (int t = 0; t < 3; ++t) pot[3 * v + t] = w[3 * fv + t];
            }
            Pattern P;
            std::vector<double> val;
            k2d3::assemble_eb3(m, spaces[l], p, pot.data(), P, val);
            HostLevel &H = out[l];
            H.n = spaces[l].n;
            H.rp = std::move(P.rp);
            H.ci = std::move(P.ci);
            H.v = std::move(val);
            if (l > 0) k2d3::build_patches3(m, spaces[l], H.pptr, H.pdofs, H.pvert);
        }
        for (int l = 1; l < nlev; ++l) {
            k2d3::build_prolongation3(meshes[l], spaces[l], meshes[l - 1], spaces[l - 1], out[l].prp, out[l].pci,
                                      out[l].pv);
            out[l].n_coarser = spaces[l - 1].n;
        }
        return "";
    }
    if (p.degree == 2) {
        std::vector<Mesh> meshes(nlev);
        std::vector<Space2> spaces(nlev);
        for (int l = nlev - 1; l >= 0; --l) {
            const int Nl = N >> (nlev - 1 - l), step = 1 << (nlev - 1 - l);
            Mesh &m = meshes[l];
            build_mesh(m, dim, Nl);
            if (block == 0) build_space2(spaces[l], m);
            else build_space2_vel(spaces[l], m);
            std::vector<double> pot(m.nv), bpot(bn ? m.nv : 0);
            for (i64 v = 0; v < m.nv; ++v) {
                int q[3];
                m.lat(v, q);
                pot[v] = w[q[0] * step + (i64)(N + 1) * (q[1] * step)];
                if (bn) bpot[v] = bn[q[0] * step + (i64)(N + 1) * (q[1] * step)];
            }
            Pattern P;
            std::vector<double> val;
            if (block == 0) assemble_eb2(m, spaces[l], p, pot.data(), P, val);
            else assemble_vel2(m, spaces[l], p, pot.data(), bn ? bpot.data() : nullptr, P, val);
            HostLevel &H = out[l];
            H.n = spaces[l].n;
            H.rp = std::move(P.rp);
            H.ci = std::move(P.ci);
            H.v = std::move(val);
            if (l > 0) {
                if (block == 0) build_patches2(m, spaces[l], H.pptr, H.pdofs, H.pvert);
                else build_patches2_vel(m, spaces[l], H.pptr, H.pdofs, H.pvert);
            }
        }
        for (int l = 1; l < nlev; ++l) {
            if (block == 0)
                build_prolongation2(meshes[l], spaces[l], meshes[l - 1], spaces[l - 1], out[l].prp, out[l].pci, out[l].pv);
            else
                build_prolongation2_vel(meshes[l], spaces[l], meshes[l - 1], spaces[l - 1], out[l].prp, out[l].pci,
                                        out[l].pv);
            out[l].n_coarser = spaces[l - 1].n;
        }
        return "";
    }
    std::vector<Mesh> meshes(nlev);
    std::vector<Space> spaces(nlev);
    const int ncomp = dim == 2 ? 1 : 3;
    for (int l = nlev - 1; l >= 0; --l) {
        const int Nl = N >> (nlev - 1 - l), step = 1 << (nlev - 1 - l);
        Mesh &m = meshes[l];
        build_mesh(m, dim, Nl);
        build_space(spaces[l], m, block);
        // potential on this level: injection of the finest vertex values (R-w)
        std::vector<double> pot(ncomp * m.nv), bpot(bn ? ncomp * m.nv : 0);
        for (i64 v = 0; v < m.nv; ++v) {
            int q[3];
            m.lat(v, q);
            const i64 fv = q[0] * step + (i64)(N + 1) * (q[1] * step + (i64)(N + 1) * (q[2] * step));
            for (int t = 0; t < ncomp; ++t) pot[ncomp * v + t] = w[ncomp * fv + t];
            if (bn)
                for (int t = 0; t < ncomp; ++t) bpot[ncomp * v + t] = bn[ncomp * fv + t];
        }
        Pattern P;
        std::vector<double> val;
        if (block == 0) assemble_eb(m, spaces[l], p, pot.data(), P, val);
        else assemble_vel(m, spaces[l], p, pot.data(), bn ? bpot.data() : nullptr, P, val);
        HostLevel &H = out[l];
        H.n = spaces[l].n;
        H.rp = std::move(P.rp);
        H.ci = std::move(P.ci);
        H.v = std::move(val);
        if (l > 0) build_patches(m, spaces[l], H.pptr, H.pdofs, H.pvert);
    }
    for (int l = 1; l < nlev; ++l) {
        build_prolongation(meshes[l], spaces[l], meshes[l - 1], spaces[l - 1], out[l].prp, out[l].pci, out[l].pv);
        out[l].n_coarser = spaces[l - 1].n;
    }
    return "";
}

}  // namespace mhdp
