// k6_patch_lu.cu -- K6 for the 3D k = 1 stars (32 < n <= 128 DoFs): batched patch LU with a
// look-ahead panel warp.  Same arithmetic as k_patch_lu (kernels.cu): the unblocked
// right-looking LU with partial pivoting of reading R-lu (first index of max |a_ik|, whole
// rows swapped, singular if !(|a_kk| > 1e-14 max|A_i|), l_ik = a_ik / a_kk (IEEE),
// a_ij = fma(-l_ik, a_kj, a_ij) for k ascending), so factors and pivots are bit-identical.
//
// Why another kernel: k_patch_lu spends ~4300 warp instructions per elimination step and
// patch, of which ~120 are the step's DFMAs -- the per-step bookkeeping (staging the pivot
// row, divisions, candidate reduction, two barriers) is replicated in all 8 warps and bounds
// the kernel (profiles/k6/summary.txt).  Here
//   * the matrix is COLUMN-major in shared memory (ld odd), lanes run over rows, so a column
//     is one conflict-free run and a row swap inside a column is two broadcast loads;
//   * warp 0 is the PANEL warp: during phase k (the other warps apply step k to columns
//     j >= k+2) it applies step k to column k+1 in registers, finds the pivot of step k+1
//     (three redux.sync on the bit pattern of |a| and the row index: first maximum), forms
//     the multipliers l_{.,k+1} by IEEE division and publishes them and the pivot row index;
//   * warps 1..7 own the columns j = k+2 + (w-1) + 7m of phase k.  For each they swap rows
//     k / p_k of that column (two broadcast loads, one store; the lane that owns row p_k takes
//     the old a_kj from a register) and update the rows i > k: one LDS, one DFMA, one STS per
//     32 rows, chunks of rows <= k skipped by a uniform switch;
//   * ONE barrier per step; the swaps of the already finished L columns (R-lu swaps whole
//     rows) are applied at the end, column by column in step order.
// The packed store (k2_common.cuh) copies contiguous column pieces.
#include <climits>
#include <cstdio>
#include <type_traits>

#include "k2_common.cuh"
#include "kernels.cuh"

namespace mhdp {

#ifdef MHDP_K6_PROF   // diagnostics build only: SM cycles per phase, summed over CTAs (thread 0)
__device__ unsigned long long g_k6prof[4];
#define K6_STAMP(slot)                                                  \
    do {                                                                \
        if (tid == 0) {                                                 \
            const long long now_ = clock64();                           \
            atomicAdd(&g_k6prof[slot], (unsigned long long)(now_ - stamp_)); \
            stamp_ = now_;                                              \
        }                                                               \
    } while (0)
#else
#define K6_STAMP(slot) do { } while (0)
#endif

template <int NCH>   // 32-row chunks per column: stars up to 32 NCH DoFs
__global__ void __launch_bounds__(256, 2) k_patch_lu_cm(int64_t np, const int *__restrict__ pn,
                                                        const int64_t *__restrict__ poff,
                                                        const int64_t *__restrict__ foff,
                                                        const int *__restrict__ pdofs,
                                                        const int64_t *__restrict__ rowptr,
                                                        const int *__restrict__ col, const double *__restrict__ val,
                                                        double *__restrict__ fac, int *__restrict__ gidx,
                                                        int *__restrict__ perm_out, int *__restrict__ status, int ld,
                                                        int maxn) {
    extern __shared__ double sm[];   // a[maxn][ld] column-major, then dofs / prm / spv / rlen, the hash, rp0
    __shared__ double red[8];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *const a = sm;
    int *const dofs = reinterpret_cast<int *>(sm + (size_t)maxn * ld);
    int *const prm = dofs + 32 * NCH;
    int *const spv = prm + 32 * NCH;
    int *const rlen = spv + 32 * NCH;
    int *const hkey = rlen + 32 * NCH;                                    // 256
    unsigned char *const hval = reinterpret_cast<unsigned char *>(hkey + 256);   // 256
    int64_t *const rp0 = reinterpret_cast<int64_t *>(hval + 256);          // 32 NCH (8-byte aligned)
    for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
        const int n = pn[p];
        const int64_t off = poff[p];
#ifdef MHDP_K6_PROF
        long long stamp_ = clock64();
#endif
        for (int e = tid; e < n * ld; e += 256) a[e] = 0.0;
        hkey[tid] = -1;
        __syncthreads();
        // stage 1: DoF list, CSR row extents and an open-addressing hash DoF -> patch row
        // (256 slots, load <= 1/2), all rows at once: one round of global latency
        for (int e = tid; e < n; e += 256) {
            const int d = pdofs[off + e];
            dofs[e] = d;
            prm[e] = e;
            const int64_t t0 = rowptr[d];
            rp0[e] = t0;
            rlen[e] = (int)(rowptr[d + 1] - t0);
            unsigned h = ((unsigned)d * 2654435761u) >> 24;
            while (atomicCAS(&hkey[h], -1, d) != -1) h = (h + 1) & 255u;
            hval[h] = (unsigned char)e;
        }
        __syncthreads();
        // stage 2: gather A_i = R_i A R_i^T: warp per patch row, lanes over the CSR row;
        // the loads of four rows (up to 96 entries each) are issued before the first lookup
        double mx = 0.0;
        auto place = [&](int rr, int c, double v) {
            unsigned h = ((unsigned)c * 2654435761u) >> 24;
            for (;;) {
                const int kk = hkey[h];
                if (kk == c) {
                    a[(int)hval[h] * ld + rr] = v;
                    mx = fmax(mx, fabs(v));
                    return;
                }
                if (kk == -1) return;
                h = (h + 1) & 255u;
            }
        };
        for (int r0 = wid; r0 < n; r0 += 32) {
            int c[4][3];
            double v[4][3];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rr = r0 + 8 * q;
                const int64_t t0 = rr < n ? rp0[rr] : 0;
                const int len = rr < n ? rlen[rr] : 0;
#pragma unroll
                for (int u = 0; u < 3; ++u) {
                    const int idx = lane + 32 * u;
                    c[q][u] = idx < len ? __ldg(col + t0 + idx) : -1;
                    v[q][u] = idx < len ? __ldg(val + t0 + idx) : 0.0;
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                const int rr = r0 + 8 * q;
#pragma unroll
                for (int u = 0; u < 3; ++u)
                    if (c[q][u] >= 0) place(rr, c[q][u], v[q][u]);
                if (rr < n) {   // rows longer than 96 entries
                    const int64_t t0 = rp0[rr];
                    const int len = rlen[rr];
                    for (int idx = 96 + lane; idx < len; idx += 32) place(rr, __ldg(col + t0 + idx), __ldg(val + t0 + idx));
                }
            }
        }
        for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
        if (lane == 0) red[wid] = mx;
        __syncthreads();
        double amax = red[0];
        for (int w = 1; w < 8; ++w) amax = fmax(amax, red[w]);
        const double thr = 1e-14 * amax;
        K6_STAMP(0);

        // panel warp state: multipliers of the last finished step (rows lane + 32 t) and its pivot row
        double lreg[NCH];
        int pvprev = 0;
        // column j: apply step j-1 (registers), pivot search, multipliers; publishes spv[j]
        auto panel_col = [&](int j) {
            double *cj = a + (size_t)j * ld;
            double c[NCH];
            if (j > 0) {
                const int k = j - 1;
                const double u = cj[pvprev], tt = cj[k];
#pragma unroll
                for (int t = 0; t < NCH; ++t) {
                    const int i = lane + 32 * t;
                    double x = i < n ? cj[i] : 0.0;
                    if (i == pvprev) x = tt;
                    if (i > k && i < n) x = fma(-lreg[t], u, x);
                    c[t] = x;
                }
                __syncwarp();
                if (lane == 0) cj[k] = u;
            } else {
#pragma unroll
                for (int t = 0; t < NCH; ++t) {
                    const int i = lane + 32 * t;
                    c[t] = i < n ? cj[i] : 0.0;
                }
            }
            // first index of max |a_ij| over i >= j (NaN never wins; R-lu / od_lu order)
            double best = -1.0, bs = 0.0, sj = 0.0;   // bs: the signed entry at the lane's first maximum
            int bi = INT_MAX;
#pragma unroll
            for (int t = 0; t < NCH; ++t) {
                const int i = lane + 32 * t;
                const double v = fabs(c[t]);
                if (i == j) sj = c[t];
                if (i >= j && i < n && v > best) { best = v; bi = i; bs = c[t]; }
            }
            const unsigned long long key =
                bi == INT_MAX ? 0ull : (unsigned long long)__double_as_longlong(best) + 1ull;
            const unsigned khi = (unsigned)(key >> 32), klo = (unsigned)key;
            const unsigned mhi = __reduce_max_sync(FULL, khi);
            const unsigned mlo = __reduce_max_sync(FULL, khi == mhi ? klo : 0u);
            int pv = __reduce_min_sync(FULL, (khi == mhi && klo == mlo && bi != INT_MAX) ? bi : INT_MAX);
            const bool none = pv == INT_MAX;   // every candidate is NaN: od_lu keeps p = j (singular)
            if (none) pv = j;
            const double piv = __shfl_sync(FULL, bs, pv & 31);   // the winning lane has bi == pv
            const double ajj = __shfl_sync(FULL, sj, j & 31);
            // od_lu starts from best = |a_jj|: a NaN there keeps p = j and the step is singular
            if (none || !(fabs(piv) > thr) || isnan(ajj)) {
                if (lane == 0) spv[j] = -1;
                return;
            }
#pragma unroll
            for (int t = 0; t < NCH; ++t) {
                const int i = lane + 32 * t;
                double l = 0.0;
                if (i > j && i < n) {
                    l = (i == pv ? ajj : c[t]) / piv;
                    cj[i] = l;
                }
                lreg[t] = l;
            }
            if (lane == 0) {
                cj[j] = piv;
                spv[j] = pv;
                if (pv != j) { const int t = prm[j]; prm[j] = prm[pv]; prm[pv] = t; }
            }
            pvprev = pv;
        };
        bool bad = false;
        for (int k = -1; k < n; ++k) {   // phase -1: the panel warp alone prepares step 0
            int pv = 0;
            if (k >= 0) {
                __syncthreads();   // step k's multipliers and pivot are published; phase k-1's updates are done
                pv = spv[k];
                if (pv < 0) { bad = true; break; }
            }
            if (wid == 0) {
                if (k + 1 < n) panel_col(k + 1);
                continue;
            }
            if (k < 0) continue;
            const double *ck = a + (size_t)k * ld;
            auto cols = [&](auto t0c) {
                constexpr int T0 = decltype(t0c)::value;   // chunks < T0 hold only rows <= k
                double lr[NCH];
                bool act[NCH], isp[NCH];
#pragma unroll
                for (int t = T0; t < NCH; ++t) {
                    const int i = lane + 32 * t;
                    act[t] = i > k && i < n;
                    isp[t] = i == pv;
                    lr[t] = act[t] ? ck[i] : 0.0;
                }
#pragma unroll 2
                for (int j = k + 1 + wid; j < n; j += 7) {
                    double *cj = a + (size_t)j * ld;
                    const double u = cj[pv], tt = cj[k];
#pragma unroll
                    for (int t = T0; t < NCH; ++t) {
                        if (act[t]) {
                            const int i = lane + 32 * t;
                            const double x = isp[t] ? tt : cj[i];
                            cj[i] = fma(-lr[t], u, x);
                        }
                    }
                    __syncwarp();
                    if (lane == 0) cj[k] = u;
                }
            };
            switch ((k + 1) >> 5) {
                case 0: cols(std::integral_constant<int, 0>{}); break;
                case 1: cols(std::integral_constant<int, NCH >= 2 ? 1 : 0>{}); break;
                case 2: cols(std::integral_constant<int, NCH >= 3 ? 2 : 0>{}); break;
                default: cols(std::integral_constant<int, NCH >= 4 ? 3 : 0>{}); break;
            }
        }
        __syncthreads();
        K6_STAMP(1);
        if (bad) {
            if (tid == 0) atomicMin(status, (int)(p + 1 > INT_MAX - 1 ? INT_MAX - 1 : p + 1));
            __syncthreads();
            continue;
        }
        // R-lu swaps whole rows: apply the swaps of steps k > j to the finished L column j
        if (tid < n) {
            double *cj = a + (size_t)tid * ld;
            for (int k = tid + 1; k < n; ++k) {
                const int pv = spv[k];
                if (pv != k) { const double t = cj[k]; cj[k] = cj[pv]; cj[pv] = t; }
            }
        }
        __syncthreads();
        // packed streaming layout (k2_common.cuh): column pieces are contiguous on both sides
        double *F = fac + foff[p];
        for (int j = wid; j < n; j += 8) {
            const double *cj = a + (size_t)j * ld;
            double *Lf = F + pack_fwd(n, j) - (j + 1);   // l_ij at Lf[i], i > j
            for (int i = j + 1 + lane; i < n; i += 32) Lf[i] = cj[i];
            double *Ub = F + pack_bwd(n, j);
            if (lane == 0) { const double v = cj[j]; Ub[0] = v; Ub[1] = 1.0 / v; }
            for (int i = lane; i < j; i += 32) Ub[2 + i] = cj[i];
        }
        for (int e = tid; e < n; e += 256) {
            gidx[off + e] = dofs[prm[e]];
            perm_out[off + e] = prm[e];
        }
        __syncthreads();
        K6_STAMP(2);
    }
}

// stars this kernel takes (launch_patch_lu routes the others to k_patch_lu / k_patch_lu_reg)
bool patch_lu_cm_supported(int max_n) { return max_n > 32 && max_n <= 128; }

void launch_patch_lu_cm(const DevPatches &P, const int64_t *rowptr, const int *col, const double *val, int *status,
                        cudaStream_t s) {
    const int ld = P.max_n | 1;   // odd: the end-of-factorisation swaps run one thread per column
    const int nch = (P.max_n + 31) / 32;
    size_t smem = sizeof(double) * (size_t)P.max_n * ld + sizeof(int) * (4 * 32 * nch + 256) + 256 +
                  sizeof(int64_t) * 32 * nch;
    smem = (smem + 15) & ~(size_t)15;
    const int per_sm = smem > 110 * 1024 ? 1 : (smem > 70 * 1024 ? 2 : (smem > 50 * 1024 ? 3 : 4));
    const int64_t cap = (int64_t)sm_count() * per_sm * 4;
    const unsigned g = (unsigned)(P.np < cap ? P.np : cap);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<g, 256, smem, s>>>(P.np, P.pn, P.poff, P.foff, P.pdofs, rowptr, col, val, P.fac, P.gidx, P.perm,
                                  status, ld, P.max_n);
    };
    if (nch <= 2) go(k_patch_lu_cm<2>);
    else if (nch == 3) go(k_patch_lu_cm<3>);
    else go(k_patch_lu_cm<4>);
    ++g_launches;
#ifdef MHDP_K6_PROF
    cudaStreamSynchronize(s);
    unsigned long long h[4] = {0, 0, 0, 0};
    cudaMemcpyFromSymbol(h, g_k6prof, sizeof(h));
    fprintf(stderr, "K6 prof np=%lld max_n=%d grid=%u: gather %.3e LU %.3e tail %.3e cycles (sum over CTAs)\n",
            (long long)P.np, P.max_n, g, (double)h[0], (double)h[1], (double)h[2]);
    unsigned long long z[4] = {0, 0, 0, 0};
    cudaMemcpyToSymbol(g_k6prof, z, sizeof(z));
#endif
}

}  // namespace mhdp
