/*
 * solve.c -- ORACLE (test infrastructure only; see orc.h).
 *
 * Dense LU with partial pivoting (reading R-lu; the paper names PCPATCH local
 * solves and MUMPS, without stating the factorisation), the
 * vertex-star parallel subspace correction sweep (P:529-538 eq. decomp), the
 * V-cycle and right-preconditioned GMRES.
 *
 * Rounding order is pinned (reading R-order): every reduction is an
 * fma chain in a stated index order, so that any implementation honouring the
 * same per-element operation sequence reproduces these results bit for bit.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>
#include "orc.h"

/* Unblocked right-looking LU with partial pivoting (R-lu):
 *   k = 0..n-1: p = argmax_{i>=k} |a_ik| (ties -> smallest i); swap rows k,p;
 *   singular if |a_kk| <= 1e-14 * amax;  l_ik = a_ik / a_kk;
 *   a_ij <- fma(-l_ik, a_kj, a_ij) for i,j > k.                                  */
int od_lu(double *a, int n, int *perm, double amax) {
    for (int i = 0; i < n; i++) perm[i] = i;
    for (int k = 0; k < n; k++) {
        int p = k;
        double best = fabs(a[(i64)k * n + k]);
        for (int i = k + 1; i < n; i++)
            if (fabs(a[(i64)i * n + k]) > best) { best = fabs(a[(i64)i * n + k]); p = i; }
        if (p != k) {
            for (int j = 0; j < n; j++) {
                double t = a[(i64)k * n + j]; a[(i64)k * n + j] = a[(i64)p * n + j]; a[(i64)p * n + j] = t;
            }
            int t = perm[k]; perm[k] = perm[p]; perm[p] = t;
        }
        double piv = a[(i64)k * n + k];
        if (!(fabs(piv) > 1e-14 * amax)) return k + 1;
        for (int i = k + 1; i < n; i++) {
            double l = a[(i64)i * n + k] / piv;
            a[(i64)i * n + k] = l;
            for (int j = k + 1; j < n; j++) a[(i64)i * n + j] = fma(-l, a[(i64)k * n + j], a[(i64)i * n + j]);
        }
    }
    return 0;
}

/* z = U^-1 L^-1 P r:  z_k = r[perm[k]];  forward z_i <- fma(-l_ij, z_j, z_i) (j ascending);
 * back: z_j <- z_j / u_jj, then z_i <- fma(-u_ij, z_j, z_i) for i < j (j descending)    */
void od_lu_solve(const double *lu, int n, const int *perm, const double *r, double *z) {
    for (int k = 0; k < n; k++) z[k] = r[perm[k]];
    for (int j = 0; j < n; j++)
        for (int i = j + 1; i < n; i++) z[i] = fma(-lu[(i64)i * n + j], z[j], z[i]);
    for (int j = n - 1; j >= 0; j--) {
        z[j] = z[j] / lu[(i64)j * n + j];
        for (int i = 0; i < j; i++) z[i] = fma(-lu[(i64)i * n + j], z[j], z[i]);
    }
}
