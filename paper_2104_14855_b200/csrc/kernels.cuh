// kernels.cuh -- launchers of the sm_100a kernels of the vertex-star Schwarz
// smoother / V-cycle.  Every reduction follows the pinned
// per-element operation order of DESIGN.md reading R-order, so that
// results do not depend on how the work is parallelised.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace mhdp {

// Sliced ELLPACK (SELL-32) operator store: slice s = rows 32s..32s+31; entry k of row
// 32s+l at sptr[s] + 32k + l.  Rows keep their ascending column order (R-order).
struct DevSell {
    int64_t n = 0, nslices = 0, stored = 0;
    int64_t *sptr = nullptr;   // nslices+1
    int *rlen = nullptr;       // n
    int *col = nullptr;        // stored
    double *val = nullptr;     // stored
};

// 3x3-block SELL store for operators whose DoFs come in aligned triples sharing one
// column pattern (3D BDM1 velocity: the 3 DoFs of a face).  Block-row R = DoFs 3R..3R+2;
// slice s = block rows 32s..32s+31; block entry e = sptr[s]+32k+l of block row 32s+l:
// column block index col[e], its 3x3 values (row-major m = 3a+b) at val[m*stored + e].
struct DevBSell3 {
    int64_t nb = 0, nslices = 0, stored = 0;
    int64_t *sptr = nullptr;
    int *rlen = nullptr;       // per block row
    int *col = nullptr;        // block column index
    double *val = nullptr;     // planes == 1: 9 planes of `stored` doubles; planes == 0 (default):
                               // per slice s and block column k the 9 x 32 values contiguous,
                               // entry m of lane l at val[9 sptr[s] + (9 k + m) 32 + l]
    int planes = 0;
};

struct DevCsr {
    int64_t n = 0, nnz = 0;
    int *rp = nullptr;         // n+1 (int32 offsets; transfer operators are small)
    int *ci = nullptr;
    double *v = nullptr;
};

// star sizes: K6 keeps the patch matrix in shared memory up to K6_SMEM_MAX DoFs, in a
// global scratch above; K2 and K6 support stars up to K2_MAX_N DoFs (3D k = 2 sizes)
static constexpr int K6_SMEM_MAX = 160;
static constexpr int K2_MAX_N = 384;

struct DevPatches {
    int64_t np = 0, sum_n = 0, fac_doubles = 0;
    int max_n = 0;
    int *pn = nullptr;         // np   patch sizes
    int64_t *poff = nullptr;   // np   slot offset (= pptr[i])
    int64_t *foff = nullptr;   // np   factor offset in doubles (16-double aligned)
    // the same three arrays with the patches in size-descending (stable) order: the order in
    // which the persistent warp kernels walk them (patches are independent; the last,
    // partial round of the round-robin gets the smallest stars -- load balance)
    int *pn_o = nullptr;
    int64_t *poff_o = nullptr, *foff_o = nullptr;
    int *pdofs = nullptr;      // sum_n ascending DoFs of each patch
    int *gidx = nullptr;       // sum_n pivot-folded gather list  gidx[k] = pdofs[perm[k]]
    int *perm = nullptr;       // sum_n LU row permutation (export only)
    double *fac = nullptr;     // packed LU factors, column-major per patch
    int *dptr = nullptr;       // n+1  DoF -> slot list
    int *dslot = nullptr;      // sum_n slots of each DoF, ascending patch order
    double *wd = nullptr;      // n    theta * (1/m_d)
    bool triples = false;      // DoFs 3R..3R+2 share one slot list at consecutive slots (K3 per triple)
    double *y = nullptr;       // sum_n slot buffer
    // small stars (every patch size in LR_SIZES): thread-per-patch K2 on lane-interleaved
    // factors streamed through TMA rings.
    // Patches grouped 32 at a time by size; element e of lane l of group g at
    // facI[gbase[g] + 32 e + l]; gpatch[32 g + l] = patch or -1 (padding, zero factors).
    int64_t ng = 0;
    int *gn = nullptr;         // ng   common size of the group
    int64_t *gbase = nullptr;  // ng   offset in facI (doubles)
    int *gpatch = nullptr;     // 32 ng
    double *facI = nullptr;
};
// the patch sizes the small-star K2 kernel is instantiated for (2D k = 1 and k = 2 stars)
bool lring_size_supported(int n);
// copy the packed factors into the lane-interleaved layout (setup)
void launch_interleave(const DevPatches &P, cudaStream_t s);
// K2 on the lane-interleaved factors (k2_small.cu)
void apply_lring(const DevPatches &P, const double *r, cudaStream_t s);

// counts every launch made through these wrappers (bench "gpu_launches")
extern long long g_launches;

// K1: r = b - A x (or y = A x when b == nullptr)
void launch_residual(const DevSell &A, const double *b, const double *x, double *r, cudaStream_t s);
void launch_residual_b3(const DevBSell3 &A, const double *b, const double *x, double *r, cudaStream_t s);
// fill the 3x3-block SELL store (col, val: zero-initialised) from the level's device CSR (setup)
void launch_build_b3(const DevBSell3 &A, const int64_t *rp, const int *ci, const double *v, cudaStream_t s);
// K6: batched patch LU (gather from the CSR on the device, partial pivoting)
// rowptr (int64) / col / val: the level operator in CSR; status[0] = first singular patch+1
int64_t patch_lu_scratch_doubles(const DevPatches &P);
void launch_patch_lu(const DevPatches &P, const int64_t *rowptr, const int *col, const double *val, int *status,
                     double *scratch, cudaStream_t s);
// K6 for stars of 33..128 DoFs (k6_patch_lu.cu): column-major, look-ahead panel warp
bool patch_lu_cm_supported(int max_n);
void launch_patch_lu_cm(const DevPatches &P, const int64_t *rowptr, const int *col, const double *val, int *status,
                        cudaStream_t s);
// K2: y_i = A_i^-1 R_i r for every patch
void launch_patch_apply(const DevPatches &P, const double *r, cudaStream_t s);
// K3: x_d <- fma(w_d, sum y, x_d)    (x_is_zero: x_d <- fma(w_d, sum y, 0.0))
void launch_patch_update(const DevPatches &P, int64_t n, double *x, int x_is_zero, cudaStream_t s);
// K4: rc = PT r  (PT: coarse rows);  K5: x <- x + P ec  (P: fine rows)
void launch_restrict(const DevCsr &PT, const double *r, double *rc, cudaStream_t s);
void launch_prolong_add(const DevCsr &P, const double *ec, double *x, cudaStream_t s);
// K7: dense LU with partial pivoting of the row-major n x n matrix a (in place)
// perm[n]; status[0] = 0 or (step+1) of the first singular pivot; amax = max|a|
void launch_dense_lu(double *a, int n, int *perm, int *status, double *scratch, cudaStream_t s);
int k7_max_n();   // largest n whose panel slices fit the cluster's shared memory
// K8 coarse solve (k8_coarse.cu): R-lu forward/back substitution, bit-identical to the
// unblocked c.6 solve.  Tiles/records from the row-major factors (setup); solve: b != x.
int k8_max_n();
int64_t k8_tile_doubles(int n);
int64_t k8_sync_words(int n);
int64_t k8_rec_doubles(int n);
void launch_k8_pack(const double *lu_rowmajor, int n, double *tiles, double *rec, cudaStream_t s);
cudaError_t launch_k8_solve(const double *tiles, const double *rec, const int *perm, int n, const double *b,
                            double *x, double *zf, double *hacc, unsigned long long *sync, cudaStream_t s,
                            long long *trace = nullptr);   // trace: diagnostics, 5 stamps per (pass, block)
// K9 vector ops (deterministic reductions)
void launch_dot(const double *a, const double *b, int64_t n, double *partials, double *out, cudaStream_t s);
void launch_axpy(double *y, double alpha, const double *x, int64_t n, cudaStream_t s);   // y = fma(alpha, x, y)
void launch_scale(double *y, const double *x, double alpha, int64_t n, cudaStream_t s);   // y = x * alpha
void launch_fill(double *y, double v, int64_t n, cudaStream_t s);

// NEXT-1 Krylov pieces (R-dot pinned inner products; explicitly rounded scalar steps)
// part: 2 * ceil(n/256) doubles of scratch; *out = a.b (or sqrt(a.b))
void launch_dot_pinned(const double *a, const double *b, int64_t n, double *part, double *out, int do_sqrt,
                       cudaStream_t s);
void launch_axpy_negdev(double *w, const double *h, const double *v, int64_t n, cudaStream_t s);  // w -= h[0] v
void launch_div_dev(double *y, const double *x, const double *d, int64_t n, cudaStream_t s);       // y = x / d[0]
// kk_dev (optional): device Krylov dimension, set by launch_krylov_init / launch_givens
void launch_krylov_init(const double *g, int m, int *kk, cudaStream_t s);
void launch_givens(double *H, int m, double *cs, double *sn, double *g, const double *hn, int k, int *kk_dev,
                   cudaStream_t s);
void launch_backsub(const double *H, int m, const double *g, int kk, const int *kk_dev, double *y, cudaStream_t s);
void launch_basis_update(double *x, const double *V, int64_t ldv, const double *y, int kk, const int *kk_dev,
                         int64_t n, cudaStream_t s);

// NEXT-3: out = b - A x (CSR, int64 row pointer, ascending fma chains); y = (c s) kinv
void launch_csr_sub(int64_t n, const int64_t *rp, const int *ci, const double *v, const double *x, const double *b,
                    double *out, cudaStream_t s);
void launch_scale2(double *y, const double *s, double c, double kinv, int64_t n, cudaStream_t st);

}  // namespace mhdp
