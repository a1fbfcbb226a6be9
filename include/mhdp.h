/*
 * mhdp.h -- C-ABI of the B200-native vertex-star Schwarz smoother / V-cycle
 * library (libmhdp.so) for the two specialised multigrid solvers of
 * arXiv 2104.14855 (PAPER.md = P:line; SURVEY.md §8(b) = the call list):
 *
 *   - the augmented-Lagrangian H(div) velocity-block multigrid   (§3.4)
 *   - the monolithic E-B block multigrid                          (§3.5)
 *
 * The smoother is the parallel subspace correction of P:529-538 (eq. decomp) over
 * the vertex-star decomposition of P:567-571 (eq. stardecomp); the hierarchy is the
 * nested uniform refinement with the FE-induced prolongation of P:572; the cycle is
 * the V-cycle of P:643 with Richardson Schwarz sweeps instead of GMRES(6) (DESIGN.md
 * reading R-smoother).
 *
 * Conventions (all entry points)
 *   - Every function returns an mhdp_status; nothing throws across the ABI.
 *   - Levels are numbered 0 = coarsest .. n_levels-1 = finest.
 *   - "_dev" pointers are CUDA device pointers of fp64 vectors of the level's length n
 *     (contiguous, owned by the CALLER, on the context's device). "_host" pointers are
 *     host memory owned by the caller. The context owns every internal store.
 *   - Device work is stream-ordered on the context's stream and does not synchronise
 *     the host, except where a function says "synchronises".
 *   - A context is not thread-safe; distinct contexts are independent.
 *   - On error the context keeps a message (mhdp_last_error).
 */
#ifndef MHDP_H
#define MHDP_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
    MHDP_OK = 0,
    MHDP_EINVAL = 1,     /* bad argument: null pointer, bad sizes, bad mesh/params          */
    MHDP_ENOMEM = 2,     /* host or device allocation failed                                */
    MHDP_ECUDA = 3,      /* CUDA runtime error, or a device call on a host-only context      */
    MHDP_ESINGULAR = 4,  /* zero pivot (|pivot| <= 1e-14 max|A_i|) in a patch or coarse LU  */
    MHDP_ESTATE = 5,     /* call out of order (e.g. smooth before setup)                    */
    MHDP_ENOCONV = 6     /* GMRES reached maxit (not fatal: x holds the last iterate)       */
} mhdp_status;

typedef enum {
    MHDP_BLOCK_EB = 0,    /* E-B block  [[M_E, G~ - A/Rem], [A^T, C]]  */
    MHDP_BLOCK_ALVEL = 1  /* AL velocity block: (2/Re) eps-form SIPG + upwind advection
                             + gamma grad-div on BDM1   */
} mhdp_block;

typedef struct {
    int dim;       /* 2 (unit square, triangles) or 3 (unit cube, 6 Kuhn tets per cube)      */
    int n_fine;    /* cells per side on the finest level; n_fine % 2^(n_levels-1) == 0       */
    int n_levels;  /* >= 1; level l has n_fine >> (n_levels-1-l) cells per side     */
} mhdp_mesh;

typedef struct {
    double Re, Rem, S, gamma; /* P:20-35. S is accepted and unused by both blocks
                                 (reading R-S); Re/gamma used by ALVEL, Rem by EB; > 0      */
    double sigma;             /* SIPG penalty sigma = 10 k^2 = 10                    */
    double mu_stab;           /* Burman stabilisation mu >= 0 of the velocity
                                 block: every interior facet adds mu h_F^2 int_F [grad u] :
                                 [grad v] (reading R-mu); 0 for the BASELINE configs; k = 1
                                 only (EINVAL with degree 2); unused by the E-B block        */
    double theta;             /* outer damping of the additive update (R-weights), 1.0       */
    int nu_pre, nu_post;      /* smoothing sweeps per level in the V-cycle (R-nu)             */
    int smoother;             /* 0: nu_pre / nu_post Richardson Schwarz sweeps (north star);
                                 1: GMRES(smoother_its) left-preconditioned by the Schwarz
                                 operator, once before and once after the coarse correction
                                 -- the paper's relaxation, P:643 (R-gmres6)                  */
    int smoother_its;         /* GMRES iterations of the smoother (6), 1..32           */
    double dt;                /* NEXT-4: 0 = stationary (eta = 0); > 0 = one implicit step
                                 (eta = 1): (1/dt)(B, C) in the E-B block, (1/dt)(u, v) in the
                                 velocity block                            */
    int picard;               /* NEXT-4: 0 = Newton (delta = 1), 1 = Picard (delta = 0): the
                                 E-B block loses G~                        */
    int degree;               /* NEXT-2: element degree k.  0 or 1: k = 1 (the
                                 BASELINE configs); 2: k = 2 for both blocks in 2D and 3D --
                                 E-B CG2 x RT2 (2D) / NED1_2 x RT2 (3D, 280-DoF stars), AL
                                 velocity BDM2 (36 / 360-DoF stars); readings R-basis2,
                                 R-basis2-vel, R-basis2-3D.  Other values -> MHDP_EINVAL       */
    int weights_mode;         /* update weights w_i of P:538 "sum_i w_i du_i": 0 = by degree
                                 (k = 1: 1; k = 2: 2), 1 = per-DoF partition of unity
                                 theta / m_d (SURVEY A2, R-weights), 2 = the uniform
                                 per-subspace damping theta / max_d m_d (R-weights2)           */
    int newton_reaction;      /* 0 = Oseen (default); 1 = add the Newton reaction
                                 (u . grad u^n, v) of Table 1 row F.  With the
                                 advecting field of reading R-w (constant on every cell) the
                                 cellwise term is identically zero, so both values assemble
                                 the same operator (reading R-newton)                        */
} mhdp_params;

typedef struct mhdp_ctx mhdp_ctx;

typedef struct {
    long long n;          /* free DoFs of the level                                         */
    long long nnz;        /* operator nonzeros (CSR, structural)                             */
    long long npatch;     /* vertex-star patches (non-empty stars, ascending vertex)         */
    long long sum_n;      /* sum_i n_i  (patch slots)                                         */
    long long sum_n2;     /* sum_i n_i^2 (factor doubles, unpadded)                           */
    long long max_n;      /* largest patch                                                   */
    long long p_nnz;      /* nonzeros of the prolongation from level-1 (0 on level 0)        */
    long long bytes_operator, bytes_factors, bytes_transfer; /* device bytes of each store  */
} mhdp_level_info;

/* ---- lifecycle ---------------------------------------------------------------------- */

/* Create a context on CUDA device `cuda_device` issuing work on `cuda_stream` (a
 * cudaStream_t; NULL = the legacy default stream).  cuda_device = -1 creates a
 * HOST-ONLY context: mhdp_assemble/mhdp_load_level and the export calls work, every
 * device call returns MHDP_ECUDA (used by the CPU test-suite to check host setup).   */
mhdp_status mhdp_create(mhdp_ctx **out, int cuda_device, void *cuda_stream);
void        mhdp_destroy(mhdp_ctx *ctx);

/* Assemble every level of the hierarchy on the host (setup stage a0/a1 of SURVEY §8(a)):
 * structured nested meshes, canonical numbering, free DoFs, vertex-star patches
 * (P:567-571), the level operators by rediscretisation (R-coarse) and the exact
 * prolongations.  w_vertex_host: potential of the advecting field at the
 * finest-level vertices in vertex order i+(N+1)(j+(N+1)k) (R-w): 2D stream function
 * psi (1 double per vertex, field = vcurl psi_h), 3D vector potential A (3 doubles per
 * vertex, field = curl of the NED1 interpolant of A_h).  Coarser levels inject it.
 * Errors: EINVAL (dims, divisibility, non-positive Re/Rem/gamma, mu_stab != 0, NULL). */
mhdp_status mhdp_assemble(mhdp_ctx *ctx, mhdp_block block, const mhdp_mesh *mesh,
                          const mhdp_params *params, const double *w_vertex_host);
/* As mhdp_assemble, plus the linearised Lorentz force of the velocity block (NEXT-4,
 * Table 1 row D): S (B^n x (u x B^n), v) = S (u x B^n, v x B^n), with B^n given
 * like the advecting field by its potential at the finest vertices (bn_vertex_host, same
 * layout as w_vertex_host; NULL = no Lorentz term).  EINVAL for the E-B block.         */
mhdp_status mhdp_assemble_lorentz(mhdp_ctx *ctx, mhdp_block block, const mhdp_mesh *mesh,
                                  const mhdp_params *params, const double *w_vertex_host,
                                  const double *bn_vertex_host);

/* Algebraic entry (the PCPATCH-style interface): install level `level` of an
 * n_levels hierarchy from caller data instead of mhdp_assemble.  Host arrays, copied:
 *   rowptr[n+1] (int64), col[nnz] (int32, ascending within a row), val[nnz]      A_l
 *   pptr[npatch+1] (int64), pdofs[pptr[npatch]] (int32, ascending within a patch) patches
 *   prow[n+1], pcol, pval: prolongation from level-1 (n x n_{l-1}); NULL on level 0.
 * Call mhdp_begin_levels first.  Errors: EINVAL (sizes, unsorted, out of range).     */
mhdp_status mhdp_begin_levels(mhdp_ctx *ctx, int n_levels, const mhdp_params *params);
mhdp_status mhdp_load_level(mhdp_ctx *ctx, int level, long long n,
                            const long long *rowptr, const int *col, const double *val,
                            long long npatch, const long long *pptr, const int *pdofs,
                            const long long *prow, const int *pcol, const double *pval);

/* Upload the stores and factor them on the device (synchronises): batched patch LU with
 * partial pivoting for every level >= 1 (kernel K6) and the dense
 * coarse LU of level 0 (K7; stand-in for MUMPS) and, from its factors, the
 * K8 substitution tiles (k8_coarse.cu).  Errors: ESINGULAR for a singular
 * star names its mesh vertex (mhdp_last_error's `where` = the vertex id,
 * the message names the level), or the patch index for operators installed by
 * mhdp_load_level; `where` = -1 for a singular coarse operator.                        */
mhdp_status mhdp_setup(mhdp_ctx *ctx);
/* Timings of the last mhdp_setup (diagnostics; len >= 3 + n_levels): out[0] = K7 dense
 * coarse LU (device ms), out[1] = K8 tile packing (ms), out[2] = wall time of the whole
 * setup (s: host packing, uploads and kernels), out[3 + l] = K6 batched patch LU of level
 * l (ms; 0 for level 0); if len >= 9 + n_levels, out[3 + n_levels + k] = host wall s of
 * the stages k = 0 operator stores, 1 patch stores, 2 transfers, 3 K6 incl. its CSR
 * upload, 4 lane groups, 5 coarse (dense build, upload, K7, K8 pack).  ESTATE before setup. */
mhdp_status mhdp_setup_timings(const mhdp_ctx *ctx, double *out, int len);

/* SURVEY 8(b) names this call mhdp_level_info, but that is also the name of the struct
 * typedef (one C identifier namespace), so the call carries a get_ prefix.             */
mhdp_status mhdp_get_level_info(const mhdp_ctx *ctx, int level, mhdp_level_info *out);
int         mhdp_num_levels(const mhdp_ctx *ctx);

/* ---- hot path (device pointers, stream-ordered, no host synchronisation) ----------- */

/* y = A_l x                                                   (operator application)   */
mhdp_status mhdp_spmv(mhdp_ctx *ctx, int level, const double *x_dev, double *y_dev);
/* r = b - A_l x   (K1; "(f,v_i) - a(u^k,v_i)")                                     */
mhdp_status mhdp_residual(mhdp_ctx *ctx, int level, const double *b_dev, const double *x_dev,
                          double *r_dev);
/* K2 alone: y_i = A_i^{-1} R_i r for every patch into the context's slot buffer
 * (exposed for timing/tests; the slot buffer is read back with mhdp_export_slots).     */
mhdp_status mhdp_patch_apply(mhdp_ctx *ctx, int level, const double *r_dev);
/* K3 alone: x_d <- fma(theta/m_d, sum_{i ∋ d} y_i[k_i(d)], x_d) from the slot buffer.  */
mhdp_status mhdp_patch_update(mhdp_ctx *ctx, int level, double *x_dev);
/* nsweeps Schwarz sweeps S(x; b) in place on level >= 1:
 *   r = b - A x;  y_i = A_i^{-1} R_i r;  x_d <- fma(theta w_d, sum_i y_i[k_i(d)], x_d).
 * x_is_zero != 0 declares x = 0 on entry: sweep 1 then skips the SpMV (x is written). */
mhdp_status mhdp_smooth(mhdp_ctx *ctx, int level, int nsweeps, int x_is_zero,
                        const double *b_dev, double *x_dev);
/* rc = P_l^T r   (K4, restriction to level-1)                                         */
mhdp_status mhdp_restrict(mhdp_ctx *ctx, int level, const double *r_dev, double *rc_dev);
/* x <- x + P_l ec (K5, prolongation from level-1)                                      */
mhdp_status mhdp_prolong_add(mhdp_ctx *ctx, int level, const double *ec_dev, double *x_dev);
/* x = A_0^{-1} b (K8): the coarse LU solve of SURVEY 8(c.8) (stand-in for MUMPS)
 * -- z = P b, forward z_i <- fma(-l_ij, z_j, z_i) (j ascending), back z_j <- z_j / u_jj,
 * z_i <- fma(-u_ij, z_j, z_i) (j descending), c.6 -- bit-identical to that unblocked
 * sequence.  b and x are device vectors of n_0 doubles; they may alias (b is copied).   */
mhdp_status mhdp_coarse_solve(mhdp_ctx *ctx, const double *b_dev, double *x_dev);
/* Diagnostics: one mhdp_coarse_solve (b, x must not alias) with K8's per-block
 * globaltimer stamps (ns) written to trace_host[(pass * nb + block) * 5 + k], nb =
 * ceil(n_0 / 32), pass 0 forward / 1 back, k = 0 claim start, 1 claim done, 2 chain
 * start, 3 chain done (chain CTA), 4 far-warp hand-off.  Synchronises.                 */
mhdp_status mhdp_coarse_solve_trace(mhdp_ctx *ctx, const double *b_dev, double *x_dev,
                                    long long *trace_host);
/* x = V_l(b) with zero initial guess on level `level` (finest: n_levels-1), P:643:
 * nu_pre sweeps, residual, restrict, recurse, prolong-add, nu_post sweeps.  Repeated
 * calls with the same (level, b, x) replay a CUDA graph of the cycle (captured on the
 * second call; env MHDP_NO_GRAPH disables this).                                       */
mhdp_status mhdp_vcycle(mhdp_ctx *ctx, int level, const double *b_dev, double *x_dev);
/* number of captured V-cycle graphs currently held (diagnostics)                       */
int         mhdp_vcycle_graphs_active(const mhdp_ctx *ctx);
/* enable = 0: mhdp_vcycle launches its kernels directly instead of replaying a captured
 * CUDA graph (diagnostics / profiling); 1 (default): graphs.                         */
mhdp_status mhdp_set_graphs(mhdp_ctx *ctx, int enable);
/* End-to-end variant for callers holding host data: copies b (host, n doubles) to the
 * device, runs mhdp_vcycle on the finest level and copies x back (synchronises).       */
mhdp_status mhdp_vcycle_host(mhdp_ctx *ctx, const double *b_host, double *x_host);
/* Batched end-to-end V-cycles (one preconditioner application per right-hand
 * side): b_host holds nrhs right-hand sides of n doubles each (row k = b_k, host,
 * caller-owned, ideally pinned), x_host receives the nrhs results in the same layout.
 * The upload of b_{k+1} and the download of x_{k-1} overlap the V-cycle of b_k (two
 * device slots, two context-owned copy streams); every x_k is bit-identical to
 * mhdp_vcycle_host(b_k).  Synchronises.  nrhs = 0 is a no-op; nrhs < 0 or NULL
 * buffers -> MHDP_EINVAL.                                                              */
mhdp_status mhdp_vcycle_host_batch(mhdp_ctx *ctx, int nrhs, const double *b_host, double *x_host);
/* Smoother sweeps with host buffers (b, x in/out; synchronises).                       */
mhdp_status mhdp_smooth_host(mhdp_ctx *ctx, int level, int nsweeps, int x_is_zero,
                             const double *b_host, double *x_host);
/* Right-preconditioned GMRES with the V-cycle on the finest level (P:625,
 * P:654): x0 = 0, modified Gram-Schmidt (w <- fma(-h, v, w)), v = w / |w|, Givens
 * rotations, no restart; inner products in the pinned order of reading R-dot, so the
 * iteration is the oracle's step for step.  Stops when the residual estimate |g_k| <=
 * max(rtol |b|, atol).  its_out = iterations, relres_out = |g_its| / |b|, hist_out
 * (optional, host, maxit + 1 doubles) = the residual history |g_k|, k = 0..its
 * (compared when either side does not converge).  1 <= maxit <= 2000.
 * Synchronises every iteration.  Returns ENOCONV at maxit (x holds the iterate).        */
mhdp_status mhdp_gmres(mhdp_ctx *ctx, const double *b_dev, double *x_dev, double rtol,
                       double atol, int maxit, int *its_out, double *relres_out,
                       double *hist_out);

/* Switch the V-cycle smoother (see mhdp_params.smoother / smoother_its); may be called
 * before or after mhdp_setup (the GMRES workspace is allocated on demand).             */
mhdp_status mhdp_set_smoother(mhdp_ctx *ctx, int smoother, int smoother_its);
/* Flexible GMRES with the current V-cycle as a variable right preconditioner on
 * the finest level (required when the smoother is GMRES, which makes the V-cycle
 * nonlinear); x0 = 0; inner products in the pinned order of reading R-dot; stops when
 * the residual estimate <= max(rtol |b|, atol).  Synchronises every iteration. */
mhdp_status mhdp_fgmres(mhdp_ctx *ctx, const double *b_dev, double *x_dev, double rtol,
                        double atol, int maxit, int *its_out, double *relres_out,
                        double *hist_out);   /* as mhdp_gmres (same iteration) */
/* The pinned inner product of reading R-dot of two device vectors (synchronises; n = 0
 * gives +0.0 and the pointers may then be NULL).                                       */
mhdp_status mhdp_dot(mhdp_ctx *ctx, const double *a_dev, const double *b_dev, long long n,
                     double *out_host);

/* ---- export for parity checks (host buffers, caller-allocated, sizes from info) ----- */
mhdp_status mhdp_export_csr(const mhdp_ctx *ctx, int level, long long *rowptr, int *col,
                            double *val);
mhdp_status mhdp_export_patches(const mhdp_ctx *ctx, int level, long long *pptr, int *pdofs);
/* verts[i] = the mesh vertex whose star is patch i (R-patch: non-empty stars in vertex
 * order); npatch ints.  ESTATE for levels installed by mhdp_load_level.          */
mhdp_status mhdp_export_patch_vertices(const mhdp_ctx *ctx, int level, int *verts);
mhdp_status mhdp_export_prolongation(const mhdp_ctx *ctx, int level, long long *prow,
                                     int *pcol, double *pval);
/* Patch `patch` of `level` after setup (synchronises): its LU factors, row-major n_i x n_i
 * (unit L below the diagonal, U on and above), and perm[k] = original row at position k. */
mhdp_status mhdp_export_patch_lu(mhdp_ctx *ctx, int level, long long patch, double *lu,
                                 int *perm);
/* The slot buffer y (sum_n doubles) of the last patch apply on `level` (synchronises).   */
mhdp_status mhdp_export_slots(mhdp_ctx *ctx, int level, double *y);

/* ---- diagnostics --------------------------------------------------------------------- */
mhdp_status mhdp_synchronize(mhdp_ctx *ctx);
/* Last error message (NUL-terminated, truncated to len) and its location (see setup). */
mhdp_status mhdp_last_error(const mhdp_ctx *ctx, char *buf, int len, long long *where);
/* Number of kernels this context has launched since creation (bench gpu_launches).    */
long long   mhdp_launch_count(const mhdp_ctx *ctx);

/* ---- NEXT-3: the coupled Newton system and the paper's outer solver ----------------- */
/* The 4x4 linearised system (Table 1) over x = [u | p | E | B]
 * (velocity BDM1 free DoFs, pressure DG0 one per cell in cell order, E and B in the E-B
 * numbering) on the finest mesh: [[F+D, B^T, J, J~+D~1+D~2], [B, 0, 0, 0],
 * [G, 0, M_E, G~ - A/Rem], [0, 0, A^T, C]] with u^n = the advecting field, B^n given by
 * its potential (bn_vertex_host, may be NULL: B^n = 0) and E^n = 0 (so J~ = 0; reading
 * R-coupled).  The object owns both multigrid hierarchies (velocity and E-B) and every
 * device store; the caller owns the device vectors it passes (fp64, length n_u + n_p +
 * n_E + n_B, on the object's device), calls are ordered on cuda_stream.
 * cuda_device = -1: host-only (assembly and export; device calls return MHDP_ECUDA).
 * Errors: MHDP_EINVAL for bad arguments or params->degree = 2 (the k = 2 coupling blocks
 * are not built); the failing stage's status otherwise (ESINGULAR for a singular patch or
 * coarse operator).  *out is set whenever memory was allocated -- destroy it also on
 * failure; mhdp_coupled_last_error returns the message.                               */
typedef struct mhdp_coupled mhdp_coupled;
mhdp_status mhdp_coupled_create(mhdp_coupled **out, int cuda_device, void *cuda_stream,
                                const mhdp_mesh *mesh, const mhdp_params *params,
                                const double *w_vertex_host, const double *bn_vertex_host);
void        mhdp_coupled_destroy(mhdp_coupled *c);
/* out[5] = n_u, n_p, n_E, n_B, nnz of the coupled operator                             */
mhdp_status mhdp_coupled_sizes(const mhdp_coupled *c, long long *out);
mhdp_status mhdp_coupled_export_csr(const mhdp_coupled *c, long long *rowptr, int *col, double *val);
/* y = A x (device vectors of length n_u + n_p + n_E + n_B)                              */
mhdp_status mhdp_coupled_apply(mhdp_coupled *c, const double *x_dev, double *y_dev);
/* y = P r, the block upper-triangular preconditioner: two FGMRES iterations
 * on the E-B block with its V-cycle, z_u = r_u - K y_EB, two FGMRES iterations on the
 * (u,p) block preconditioned by y_p = -(1/Re+gamma) M_p^-1 s_p, y_u = V_u(s_u - B^T y_p) */
mhdp_status mhdp_coupled_precondition(mhdp_coupled *c, const double *r_dev, double *y_dev);
/* outermost flexible GMRES with P, x0 = 0, stop at max(rtol|b|, atol);
 * 1 <= maxit <= 500; MHDP_ENOCONV when maxit is reached (x_dev holds that iterate).
 * The pressure is determined up to a constant (Q = L^2_0): b must have
 * mean-zero pressure rows for the system to be consistent.                              */
mhdp_status mhdp_coupled_fgmres(mhdp_coupled *c, const double *b_dev, double *x_dev, double rtol,
                                double atol, int maxit, int *its_out, double *relres_out);
mhdp_status mhdp_coupled_set_smoother(mhdp_coupled *c, int smoother, int smoother_its);
mhdp_status mhdp_coupled_last_error(const mhdp_coupled *c, char *buf, int len);

#ifdef __cplusplus
}
#endif
#endif /* MHDP_H */
