// k7_dense_lu.cu -- K7: dense LU with partial pivoting of the coarsest operator (setup;
// the stand-in for MUMPS), reading R-lu / SURVEY 8(c.6): unblocked right-looking
// LU, p = first index of max |a_ik|, whole-row swaps, singular if !(|a_kk| > 1e-14 max|A|),
// l_ik = a_ik / a_kk, a_ij <- fma(-l_ik, a_kj, a_ij).  Blocked so that every element still
// receives its updates at k = 0, 1, 2, ... in order (R-order):
//   * panel (NB = 32 columns, all rows below k0) factored by ONE thread-block cluster of
//     16 CTAs: each CTA holds a contiguous slice of the panel's rows in shared memory (row
//     stride 33 doubles: with 32, the column walks of the pivot search and of the row-per-thread
//     update were 32-way bank conflicts, which bounded the panel), the
//     pivot candidates meet in CTA 0 over distributed shared memory, the pivot row is read
//     remotely, two cluster barriers per column (round 1 factored the panel with one CTA
//     walking the row-major matrix in global memory: 583 ms of the c5 setup);
//   * the panel's row swaps applied to the other columns afterwards, in order (laswp);
//   * block row U12 by forward substitution (TRSM), trailing matrix by fma chains over
//     the panel's k ascending (64 x 64 tiles).
// Row-major storage (row i at a + i n).
#include <cooperative_groups.h>

#include <climits>
#include <cstdint>

#include "k2_common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace mhdp {

namespace {

constexpr int LU_NB = 32;     // panel width
constexpr int LU_LD = LU_NB + 1;   // row stride of a panel slice in shared memory (odd: a column walk is conflict-free)
constexpr int CL = 16;        // CTAs in the panel cluster (non-portable cluster size)
constexpr int PT = 256;       // threads per panel CTA

// max |a| over the matrix (NaN ignored, as the oracle's `if (|v| > amax)`): the bit
// pattern of a non-negative double orders like the value, so atomicMax on it is exact
__global__ void k_absmax_grid(const double *__restrict__ a, int64_t m, unsigned long long *out) {
    __shared__ unsigned long long red[PT / 32];
    unsigned long long mx = 0;
    for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += (int64_t)gridDim.x * blockDim.x) {
        const double v = fabs(a[e]);
        if (v == v) {
            const unsigned long long b = (unsigned long long)__double_as_longlong(v);
            mx = b > mx ? b : mx;
        }
    }
    for (int o = 16; o; o >>= 1) {
        const unsigned long long t = __shfl_xor_sync(FULL, mx, o);
        mx = t > mx ? t : mx;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = red[w] > mx ? red[w] : mx;
        mx = red[0] > mx ? red[0] : mx;
        atomicMax(out, mx);
    }
}

__global__ void k_iota(int *p, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = i;
}

// candidate of one CTA: (|value|, row) with the oracle's order -- larger value wins, equal
// values go to the smaller row
__device__ __forceinline__ bool better(double v, int i, double bv, int bi) { return v > bv || (v == bv && i < bi); }

// Panel k0 .. k0+kb-1 over rows k0 .. n-1, one cluster of CL CTAs.  CTA `rank` owns rows
// row0 = k0 + rank R .. +R-1 (R = ceil((n - k0) / CL)), kept in shared memory as sp[lr NB + c].
// swaps[j] = the pivot row chosen at step k0 + j (for laswp).
__global__ void __launch_bounds__(PT) k_lu_panel_cl(double *__restrict__ a, int n, int k0, int kb,
                                                    int *__restrict__ perm, int *__restrict__ status,
                                                    const unsigned long long *__restrict__ amaxbits,
                                                    int *__restrict__ swaps) {
    extern __shared__ __align__(16) double sp[];
    __shared__ double cand_v[CL];
    __shared__ int cand_i[CL];
    __shared__ int cand_nan[CL];
    __shared__ double red_v[PT / 32];
    __shared__ int red_i[PT / 32];
    __shared__ double prow[LU_NB], sbuf[LU_NB];
    __shared__ int s_p;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = (int)cluster.block_rank();
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    const int m = n - k0, R = (m + CL - 1) / CL;
    const int row0 = k0 + rank * R;
    const int nr = max(0, min(R, m - rank * R));
    const bool dead = *status != 0;          // uniform: an earlier panel was singular
    if (!dead)
        for (int e = tid; e < nr * LU_NB; e += PT) {
            const int lr = e / LU_NB, c = e % LU_NB;
            sp[lr * LU_LD + c] = c < kb ? a[(int64_t)(row0 + lr) * n + k0 + c] : 0.0;
        }
    const double thr = 1e-14 * __longlong_as_double((long long)amaxbits[0]);
    cluster.sync();
    if (dead) return;
    auto owner = [&](int gi) { return (gi - k0) / R; };
    for (int j = 0; j < kb; ++j) {
        const int gj = k0 + j;
        // ---- local pivot candidate over owned rows i >= gj ----
        double bv = -1.0;
        int bi = INT_MAX;
        for (int lr = tid; lr < nr; lr += PT) {
            const int i = row0 + lr;
            if (i < gj) continue;
            const double v = fabs(sp[lr * LU_LD + j]);
            if (v == v && better(v, i, bv, bi)) { bv = v; bi = i; }
        }
        for (int o = 16; o; o >>= 1) {
            const double ov = __shfl_xor_sync(FULL, bv, o);
            const int oi = __shfl_xor_sync(FULL, bi, o);
            if (better(ov, oi, bv, bi)) { bv = ov; bi = oi; }
        }
        if (lane == 0) { red_v[wid] = bv; red_i[wid] = bi; }
        __syncthreads();
        if (tid == 0) {
            for (int w2 = 1; w2 < PT / 32; ++w2)
                if (better(red_v[w2], red_i[w2], bv, bi)) { bv = red_v[w2]; bi = red_i[w2]; }
            double *cv = cluster.map_shared_rank(cand_v, 0);
            int *ci = cluster.map_shared_rank(cand_i, 0);
            int *cn = cluster.map_shared_rank(cand_nan, 0);
            cv[rank] = bv;
            ci[rank] = bi;
            // the oracle keeps row k when a_kk is NaN (no |a_ik| compares greater)
            cn[rank] = (gj >= row0 && gj < row0 + nr) ? (sp[(gj - row0) * LU_LD + j] != sp[(gj - row0) * LU_LD + j]) : 0;
        }
        cluster.sync();                                    // #1: candidates in CTA 0
        if (tid == 0) {
            const double *cv = cluster.map_shared_rank(cand_v, 0);
            const int *ci = cluster.map_shared_rank(cand_i, 0);
            const int *cn = cluster.map_shared_rank(cand_nan, 0);
            double v = -1.0;
            int p = INT_MAX, diag_nan = 0;
            for (int r = 0; r < CL; ++r) {
                diag_nan |= cn[r];
                if (better(cv[r], ci[r], v, p)) { v = cv[r]; p = ci[r]; }
            }
            s_p = (diag_nan || p == INT_MAX) ? gj : p;
        }
        __syncthreads();
        const int p = s_p;
        // ---- every CTA reads the new pivot row (old row p); owner(p) also reads old row gj ----
        if (tid < LU_NB) {
            const double *src = cluster.map_shared_rank(sp, owner(p)) + (int64_t)(p - (k0 + owner(p) * R)) * LU_LD;
            prow[tid] = src[tid];
            if (p != gj && owner(p) == rank) {
                const double *sg = cluster.map_shared_rank(sp, owner(gj)) + (int64_t)(gj - (k0 + owner(gj) * R)) * LU_LD;
                sbuf[tid] = sg[tid];
            }
        }
        cluster.sync();                                    // #2: all remote reads done
        if (tid < LU_NB) {
            if (owner(gj) == rank) sp[(gj - row0) * LU_LD + tid] = prow[tid];
            if (p != gj && owner(p) == rank) sp[(p - row0) * LU_LD + tid] = sbuf[tid];
        }
        const double piv = prow[j];
        if (rank == 0 && tid == 0) {
            swaps[j] = p;
            if (p != gj) { const int t = perm[gj]; perm[gj] = perm[p]; perm[p] = t; }
            if (!(fabs(piv) > thr)) *status = gj + 1;
        }
        if (!(fabs(piv) > thr)) return;                    // uniform over the cluster
        __syncthreads();
        // ---- multipliers and the panel update of owned rows below the pivot ----
        const PivotDiv dv(piv);   // IEEE quotients without the slow path of '/' on zero numerators
        for (int lr = tid; lr < nr; lr += PT) {
            const int i = row0 + lr;
            if (i <= gj) continue;
            double *ri = sp + lr * LU_LD;
            const double l = dv(ri[j]);
            ri[j] = l;
            for (int c = j + 1; c < kb; ++c) ri[c] = fma(-l, prow[c], ri[c]);
        }
        __syncthreads();
    }
    cluster.sync();
    for (int e = tid; e < nr * LU_NB; e += PT) {
        const int lr = e / LU_NB, c = e % LU_NB;
        if (c < kb) a[(int64_t)(row0 + lr) * n + k0 + c] = sp[lr * LU_LD + c];
    }
}

// the panel's row swaps (in order) on every column outside the panel
__global__ void k_lu_laswp(double *__restrict__ a, int n, int k0, int kb, const int *__restrict__ swaps,
                           const int *__restrict__ status) {
    if (*status) return;
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n || (c >= k0 && c < k0 + kb)) return;
    for (int j = 0; j < kb; ++j) {
        const int p = swaps[j];
        if (p == k0 + j) continue;
        const int64_t x = (int64_t)(k0 + j) * n + c, y = (int64_t)p * n + c;
        const double t = a[x];
        a[x] = a[y];
        a[y] = t;
    }
}

__global__ void k_lu_trsm(double *__restrict__ a, int n, int k0, int kb, const int *__restrict__ status) {
    if (*status) return;
    const int c = k0 + kb + blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= n) return;
    for (int j = k0 + 1; j < k0 + kb; ++j) {
        double acc = a[(int64_t)j * n + c];
        for (int k = k0; k < j; ++k) acc = fma(-a[(int64_t)j * n + k], a[(int64_t)k * n + c], acc);
        a[(int64_t)j * n + c] = acc;
    }
}

// trailing update of the columns [cbeg, cend): 64x64 output tile per 256-thread CTA, 4x4 per thread
__global__ void __launch_bounds__(256) k_lu_gemm(double *__restrict__ a, int n, int k0, int kb, int cbeg, int cend,
                                                 const int *__restrict__ status) {
    __shared__ double Ls[64][LU_NB + 1];
    __shared__ double Us[LU_NB][64 + 1];
    if (*status) return;
    const int r0 = k0 + kb + blockIdx.y * 64, c0 = cbeg + blockIdx.x * 64;
    const int tid = threadIdx.x;
    for (int e = tid; e < 64 * LU_NB; e += 256) {
        const int rr = e / LU_NB, kk = e % LU_NB;
        const int gr = r0 + rr;
        Ls[rr][kk] = (gr < n && kk < kb) ? a[(int64_t)gr * n + k0 + kk] : 0.0;
    }
    for (int e = tid; e < 64 * LU_NB; e += 256) {
        const int kk = e / 64, cc = e % 64;
        const int gc = c0 + cc;
        Us[kk][cc] = (gc < cend && kk < kb) ? a[(int64_t)(k0 + kk) * n + gc] : 0.0;
    }
    __syncthreads();
    const int ty = tid / 16, tx = tid % 16;
    double acc[4][4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int gr = r0 + ty + 16 * u, gc = c0 + tx + 16 * v;
            acc[u][v] = (gr < n && gc < cend) ? a[(int64_t)gr * n + gc] : 0.0;
        }
    for (int kk = 0; kk < kb; ++kk) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const double l = Ls[ty + 16 * u][kk];
#pragma unroll
            for (int v = 0; v < 4; ++v) acc[u][v] = fma(-l, Us[kk][tx + 16 * v], acc[u][v]);
        }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int v = 0; v < 4; ++v) {
            const int gr = r0 + ty + 16 * u, gc = c0 + tx + 16 * v;
            if (gr < n && gc < cend) a[(int64_t)gr * n + gc] = acc[u][v];
        }
}


}  // namespace

int k7_max_n() {
    // shared memory of a panel CTA: ceil(n / CL) rows x NB doubles within 227 KB
    return (227 * 1024 / (8 * LU_LD) - 4) * CL;
}

// scratch: >= 2 doubles (amax bits) + 2 * 32 ints (two swap lists) of device memory
void launch_dense_lu(double *a, int n, int *perm, int *status, double *scratch, cudaStream_t s) {
    if (n == 0) return;
    unsigned long long *amax = reinterpret_cast<unsigned long long *>(scratch);
    int *swaps = reinterpret_cast<int *>(scratch + 2);
    cudaMemsetAsync(amax, 0, sizeof(unsigned long long), s);
    k_iota<<<grid_for(n, 256), 256, 0, s>>>(perm, n);
    k_absmax_grid<<<sm_count() * 4, PT, 0, s>>>(a, (int64_t)n * n, amax);
    g_launches += 2;
    const int Rmax = (n + CL - 1) / CL;
    const size_t smem = sizeof(double) * (size_t)Rmax * LU_LD;
    static unsigned long long init = 0;
    if (first_use_on_device(init)) cudaFuncSetAttribute(k_lu_panel_cl, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_lu_panel_cl, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    // Look-ahead: the trailing update of panel k is split at the next panel's columns.  Once
    // those 32 columns are updated, panel k+1 is factored on a second (high-priority) stream by
    // its 16-CTA cluster while the other SMs update the remaining columns; the two touch
    // disjoint columns, and the swaps / substitution / update of panel k+1 follow after both.
    cudaStream_t sa = nullptr;
    cudaEvent_t e1 = nullptr, e2 = nullptr;
    int plo = 0, phi = 0;
    cudaDeviceGetStreamPriorityRange(&plo, &phi);
    const bool la = cudaStreamCreateWithPriority(&sa, cudaStreamNonBlocking, phi) == cudaSuccess &&
                    cudaEventCreateWithFlags(&e1, cudaEventDisableTiming) == cudaSuccess &&
                    cudaEventCreateWithFlags(&e2, cudaEventDisableTiming) == cudaSuccess;
    auto panel = [&](int k0, cudaStream_t st) {
        const int kb = n - k0 < LU_NB ? n - k0 : LU_NB;
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(CL);
        cfg.blockDim = dim3(PT);
        cfg.dynamicSmemBytes = sizeof(double) * (size_t)((n - k0 + CL - 1) / CL) * LU_LD;
        cfg.stream = st;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = CL;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaLaunchKernelEx(&cfg, k_lu_panel_cl, a, n, k0, kb, perm, status,
                           (const unsigned long long *)amax, swaps + (k0 / LU_NB & 1) * LU_NB);
        ++g_launches;
    };
    panel(0, s);
    for (int k0 = 0; k0 < n; k0 += LU_NB) {
        const int kb = n - k0 < LU_NB ? n - k0 : LU_NB;
        const int *sw = swaps + (k0 / LU_NB & 1) * LU_NB;   // two swap lists: panel k+1 writes its own while k's is read
        k_lu_laswp<<<grid_for(n, 256), 256, 0, s>>>(a, n, k0, kb, sw, status);
        ++g_launches;
        const int k1 = k0 + kb, rest = n - k1;
        if (rest <= 0) break;
        k_lu_trsm<<<grid_for(rest, 128), 128, 0, s>>>(a, n, k0, kb, status);
        const int cmid = k1 + LU_NB < n ? k1 + LU_NB : n;   // end of the next panel's columns
        k_lu_gemm<<<dim3(1, grid_for(rest, 64)), 256, 0, s>>>(a, n, k0, kb, k1, cmid, status);
        g_launches += 2;
        if (la) {
            cudaEventRecord(e1, s);
            cudaStreamWaitEvent(sa, e1, 0);
            panel(k1, sa);
            cudaEventRecord(e2, sa);
        }
        if (cmid < n) {
            k_lu_gemm<<<dim3(grid_for(n - cmid, 64), grid_for(rest, 64)), 256, 0, s>>>(a, n, k0, kb, cmid, n, status);
            ++g_launches;
        }
        if (la) cudaStreamWaitEvent(s, e2, 0);
        else panel(k1, s);
    }
    if (la) cudaStreamSynchronize(sa);   // setup path: the helper stream is drained before it is destroyed
    if (sa) cudaStreamDestroy(sa);
    if (e1) cudaEventDestroy(e1);
    if (e2) cudaEventDestroy(e2);
}

}  // namespace mhdp
