// k6_patch_lu.cu -- K6 for the 3D k = 1 stars (32 < n <= 128 DoFs): batched patch LU, blocked
// in panels of B = 4 steps with a look-ahead panel group.  Same arithmetic as k_patch_lu
// (kernels.cu): the unblocked right-looking LU with partial pivoting of reading R-lu (first
// index of max |a_ik|, whole rows swapped, singular if !(|a_kk| > 1e-14 max|A_i|),
// l_ik = a_ik / a_kk (IEEE), a_ij = fma(-l_ik, a_kj, a_ij) for k ascending), so factors and
// pivots are bit-identical.
//
// Why another kernel (profiles/k6/): k_patch_lu is bound by its per-step chain -- pivot
// search, divisions, staging and two barriers per step, replicated in 8 warps (~4300 warp
// instructions per step, ~120 of them DFMAs).  A first rewrite with ONE look-ahead panel warp
// holding four 32-row chunks per lane was bound by that warp's own instruction stream (~320
// dependent instructions per step, 87% of all stall samples on the phase barrier).  Here
//   * one CTA per star, 12 warps; the matrix is COLUMN-major in shared memory (ld odd), lanes
//     run over rows;
//   * warps 0..3 are the PANEL GROUP: warp w owns rows 32w..32w+31, one row per lane, so the
//     four columns of a panel are four registers per thread.  Per step: warp arg-max by
//     redux.sync on the high word of |a| and a ballot (the low word and the position only on
//     ties; first maximum), while every lane forms rcp_nr of its own entry; the four
//     candidates (|a|, reciprocal, position, row: a 64-byte record each) and the entry at
//     position kk meet in a double-buffered exchange area (ONE named barrier per step), the
//     best of the four is picked branch-free, the multipliers follow by PivotDiv's correction
//     step (k2_common.cuh) from the winner's reciprocal, and the panel's remaining columns are
//     updated in registers.  Rows are not moved inside a panel: each thread tracks the position
//     R-lu's swaps would give its row and the write-back scatters rows to positions.  While
//     the other warps apply panel K, the group loads panel K+1's columns with panel K applied
//     (reading through the traced-back swap permutation; the 4 x 4 triangular solve redundantly
//     per thread: no barrier) and factors it;
//   * warps 4..11 apply a finished panel to the trailing columns (a contiguous range of
//     columns per warp): the B row swaps and the 4 x 4 triangular solve for u_{k0..k0+3, j} run
//     with lanes over the warp's columns (stride ld: conflict-free), then element (i, j) takes
//     fma(-l_ik, u_kj, .) for k = k0..k0+3 in ascending order between ONE load and ONE store
//     (the rank-1 form is bound by shared-memory bandwidth: 512 B per 32 DFMAs);
//   * the same warps apply the panel's swaps to the finished L columns on its left (R-lu
//     swaps whole rows), lanes over columns, so the packed store at the end is a plain copy;
//   * ONE CTA barrier per panel.
// The CSR rows are gathered through a 1024-slot hash DoF -> patch row (loads of five rows in
// flight per warp); the next star's DoFs, row extents and an L2 prefetch of its rows are produced
// by the update warps during the first LU phases (registers carried across the star loop).
// Packed factor layout: k2_common.cuh.  Measurements and the variants not kept: DESIGN 6.2,
// profiles/k6/summary.txt; -DMHDP_K6_PROF (tools/k6_prof.sh) prints a cycle timeline.
#include <climits>
#include <cstdint>
#include <cstdio>
#include <type_traits>

#include "k2_common.cuh"
#include "kernels.cuh"

namespace mhdp {

#ifdef MHDP_K6_PROF   // diagnostics build only: SM cycles per phase, summed over CTAs (thread 0)
__device__ unsigned long long g_k6prof[16];
#define K6_STAMP(slot)                                                       \
    do {                                                                     \
        if (tid == 0) {                                                      \
            const long long now_ = clock64();                                \
            atomicAdd(&g_k6prof[slot], (unsigned long long)(now_ - stamp_)); \
            stamp_ = now_;                                                   \
        }                                                                    \
    } while (0)
// finer timeline of the LU phase: thread 0 (panel group) and thread 128 (first update warp)
#define K6_T0() long long t0_ = clock64()
#define K6_LAP(slot, who)                                                    \
    do {                                                                     \
        if (tid == (who)) {                                                  \
            const long long now_ = clock64();                                \
            atomicAdd(&g_k6prof[slot], (unsigned long long)(now_ - t0_));    \
            t0_ = now_;                                                      \
        }                                                                    \
    } while (0)
#else
#define K6_STAMP(slot) do { } while (0)
#define K6_T0() do { } while (0)
#define K6_LAP(slot, who) do { } while (0)
#endif

namespace {
constexpr int K6_B = 4;            // panel width
constexpr int K6_PW = 4;           // panel warps (one 32-row chunk each)
constexpr int K6_UW = 8;           // update warps
constexpr int K6_THREADS = 32 * (K6_PW + K6_UW);
constexpr int K6_HASH = 1024;      // hash slots (load <= 1/8)

// exchange area of the panel group, one per step parity: a 64-byte record per panel warp
struct PanelCand {
    double2 vr;                      // max |a| over the warp's live rows (-1: none), rcp_nr of that entry
    double2 r01, r23;                // that row's entries in the panel's columns
    int pos, pad0;                   // its position
    double pad1;
};
struct PanelXchg {
    PanelCand c[K6_PW];
    double akk, pad;                 // the entry at position kk
};

__device__ __forceinline__ void panel_bar(int threads) { asm volatile("bar.sync 1, %0;" ::"r"(threads) : "memory"); }
}  // namespace

template <int NCH>   // 32-row chunks per column: stars up to 32 NCH DoFs
__global__ void __launch_bounds__(K6_THREADS, 2)
k_patch_lu_cm(int64_t np, const int *__restrict__ pn, const int64_t *__restrict__ poff,
              const int64_t *__restrict__ foff, const int *__restrict__ pdofs, const int64_t *__restrict__ rowptr,
              const int *__restrict__ col, const double *__restrict__ val, double *__restrict__ fac,
              int *__restrict__ gidx, int *__restrict__ perm_out, int *__restrict__ status, int ld, int maxn) {
    constexpr int B = K6_B;
    extern __shared__ double sm[];   // a[maxn][ld] column-major, rp0, the exchange area, int tables, the hash
    __shared__ double red[K6_PW + K6_UW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    double *const a = sm;
    int64_t *const rp0 = reinterpret_cast<int64_t *>(sm + (((size_t)maxn * ld + 1) & ~(size_t)1));   // 128 (16-byte aligned)
    PanelXchg *const xch = reinterpret_cast<PanelXchg *>(rp0 + 128);            // 2
    int *const dofs = reinterpret_cast<int *>(xch + 2);                          // 128
    int *const prm = dofs + 128;
    int *const spv = prm + 128;
    int *const rlen = spv + 128;
    int *const hkey = rlen + 128;                                                // K6_HASH
    unsigned char *const hval = reinterpret_cast<unsigned char *>(hkey + K6_HASH);
    // Update-warp thread 128 + e carries, in registers, DoF e of the star `pt` this CTA factors
    // next, its CSR row start and length, and prefetches that row into L2 -- one step per early
    // LU phase of the current star (stages: 1 size, 2 DoF, 3 row extent, 4 prefetched),
    // so the gather of the next star starts from registers and reads L2-resident rows.
    int64_t nx_t0 = 0;
    int nx_stage = 0, nx_n = 0, nx_d = 0, nx_len = 0;
    auto nx_advance = [&](int want, int64_t pt) {
        const int e = tid - 32 * K6_PW;
        while (nx_stage < want && nx_stage < 4) {
            if (nx_stage == 0) {
                nx_n = pt < np ? pn[pt] : 0;
            } else if (nx_stage == 1) {
                if (e < nx_n) nx_d = pdofs[poff[pt] + e];
            } else if (nx_stage == 2) {
                if (e < nx_n) { nx_t0 = rowptr[nx_d]; nx_len = (int)(rowptr[nx_d + 1] - nx_t0); }
            } else if (e < nx_n) {
                const char *q = reinterpret_cast<const char *>(col + nx_t0), *qe = reinterpret_cast<const char *>(col + nx_t0 + nx_len);
                for (q = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(q) & ~(uintptr_t)127); q < qe; q += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
                q = reinterpret_cast<const char *>(val + nx_t0);
                qe = reinterpret_cast<const char *>(val + nx_t0 + nx_len);
                for (q = reinterpret_cast<const char *>(reinterpret_cast<uintptr_t>(q) & ~(uintptr_t)127); q < qe; q += 128)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(q));
            }
            ++nx_stage;
        }
    };
    for (int64_t p = blockIdx.x; p < np; p += gridDim.x) {
        const int n = pn[p];
        const int64_t off = poff[p];
#ifdef MHDP_K6_PROF
        long long stamp_ = clock64();
#endif
        for (int e = tid; e < n * ld; e += K6_THREADS) a[e] = 0.0;
        for (int e = tid; e < K6_HASH; e += K6_THREADS) hkey[e] = -1;
        __syncthreads();
        // stage 1: DoF list, CSR row extents and an open-addressing hash DoF -> patch row, from
        // the registers filled during the previous star's LU (the CTA's first star loads them here)
        if (tid >= 32 * K6_PW) {
            nx_advance(3, p);   // no-op except for the CTA's first star
            const int e = tid - 32 * K6_PW;
            if (e < n) {
                dofs[e] = nx_d;
                prm[e] = e;
                rp0[e] = nx_t0;
                rlen[e] = nx_len;
                unsigned h = ((unsigned)nx_d * 2654435761u) >> 22;
                while (atomicCAS(&hkey[h], -1, nx_d) != -1) h = (h + 1) & (K6_HASH - 1);
                hval[h] = (unsigned char)e;
            }
            nx_stage = 0;
        }
        __syncthreads();
        // stage 2: gather A_i = R_i A R_i^T: warp per patch row, lanes over the CSR row;
        // the loads of five rows (up to 96 entries each) are issued before the first lookup
        double mx = 0.0;
        auto place = [&](int rr, int c, double v) {
            unsigned h = ((unsigned)c * 2654435761u) >> 22;
            int kk = hkey[h];
            while (kk != c && kk != -1) {   // rare at this load
                h = (h + 1) & (K6_HASH - 1);
                kk = hkey[h];
            }
            if (kk == c) {
                a[(int)hval[h] * ld + rr] = v;
                mx = fmax(mx, fabs(v));
            }
        };
        constexpr int NW = K6_PW + K6_UW, GR = 5;
        for (int r0 = wid; r0 < n; r0 += NW * GR) {
            int c[GR][3];
            double v[GR][3];
#pragma unroll
            for (int q = 0; q < GR; ++q) {
                const int rr = r0 + NW * q;
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
            for (int q = 0; q < GR; ++q) {
                const int rr = r0 + NW * q;
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
#pragma unroll
        for (int w = 1; w < NW; ++w) amax = fmax(amax, red[w]);
        const double thr = 1e-14 * amax;
        K6_STAMP(0);

        // ---------------- blocked LU ----------------
        const int row = tid;         // panel group: the row this thread owns (tid < 128)
        bool bad = false;
        const int nphase = (n + B - 1) / B;
        K6_T0();
        for (int K = -1; K < nphase; ++K) {   // phase -1: the panel group alone factors panel 0
            const int k0 = K * B, k1 = k0 + B;   // panel K = steps k0..k0+3 (published); trailing rows from k1
            int pvk[B] = {0, 0, 0, 0};
            K6_LAP(3, 0);     // panel thread: its phase work (rest)
            K6_LAP(9, 128);   // update thread: its phase work
            if (K >= 0) {
                __syncthreads();   // panel K's multipliers and pivots are published; phase K-1's updates are done
                K6_LAP(8, 0);      // waits at the phase barrier
                K6_LAP(10, 128);
#pragma unroll
                for (int s = 0; s < B; ++s) {
                    pvk[s] = k0 + s < n ? spv[k0 + s] : k0 + s;
                    bad = bad || pvk[s] < 0;
                }
                if (bad) break;
            }
            // rows k0..k0+3 of a trailing column: the B swaps, then u = L11^-1 x (fma chains, k ascending)
            double l10 = 0, l20 = 0, l21 = 0, l30 = 0, l31 = 0, l32 = 0;
            if (K >= 0 && k1 < n) {
                const double *c0 = a + (size_t)k0 * ld + k0, *c1 = c0 + ld, *c2 = c1 + ld;
                l10 = c0[1]; l20 = c0[2]; l30 = c0[3];
                l21 = c1[2]; l31 = c1[3];
                l32 = c2[3];
            }
            auto top_rows = [&](double *cj) {
#pragma unroll
                for (int s = 0; s < B; ++s) {
                    const int A = k0 + s, Bp = pvk[s];
                    if (Bp != A) { const double tA = cj[A], tB = cj[Bp]; cj[A] = tB; cj[Bp] = tA; }
                }
                const double u0 = cj[k0];
                const double u1 = fma(-l10, u0, cj[k0 + 1]);
                const double u2 = fma(-l21, u1, fma(-l20, u0, cj[k0 + 2]));
                const double u3 = fma(-l32, u2, fma(-l31, u1, fma(-l30, u0, cj[k0 + 3])));
                cj[k0 + 1] = u1; cj[k0 + 2] = u2; cj[k0 + 3] = u3;
            };
            if (wid < K6_PW) {
                // ======== panel group: factor panel K+1 (columns k1..k1+nb-1) ========
                // Inside a panel the rows stay with their threads (no register swaps): `mypos` is
                // the position R-lu's physical swaps would have given the thread's row, `live`
                // says it has not been a pivot yet; the write-back scatters the rows to their
                // positions, so shared memory is in R-lu's physical order again at every phase.
                if (k1 >= n) continue;
                // Only the warps owning rows k1..n-1 take part in this panel (warp 0 drops out after
                // row 32, ...): the others would execute every step for nothing and lengthen the
                // exchange barrier.  tl = thread index within the participating warps.
                const int wlo = k1 >> 5, whi = (n - 1) >> 5;
                if (wid < wlo || wid > whi) continue;
                const int pth = 32 * (whi - wlo + 1), tl = tid - 32 * wlo;
                const int nb = min(B, n - k1);
                const bool inb = row < n;
                // Load the panel's columns with panel K applied.  Nothing is swapped in shared memory
                // here: the thread reads the entry that R-lu's four swaps would leave at its position
                // (src_of undoes them in registers), forms u = L11^-1 x for rows k0..k0+3 itself
                // (every thread, redundantly) and applies the four steps to its row.  Thread s stores
                // column s's u after the first exchange barrier; the rows below are rewritten by the
                // panel's write-back, so shared memory is in R-lu's order again when the phase ends.
                auto src_of = [&](int q) {
#pragma unroll
                    for (int s = B - 1; s >= 0; --s) {
                        const int A = k0 + s, Bp = pvk[s];
                        q = q == A ? Bp : (q == Bp ? A : q);
                    }
                    return q;
                };
                double c[B];
                double us0 = 0.0, us1 = 0.0, us2 = 0.0, us3 = 0.0;   // thread s < nb: u of column k1 + s
                if (K >= 0) {
                    double cp0 = 0.0, cp1 = 0.0, cp2 = 0.0, cp3 = 0.0;   // this row's multipliers of panel K
                    if (inb && row >= k1) {
                        const double *lk = a + (size_t)k0 * ld + row;
                        cp0 = lk[0]; cp1 = lk[ld]; cp2 = lk[2 * ld]; cp3 = lk[3 * ld];
                    }
                    const int srow = src_of(row);
                    const int g0 = src_of(k0), g1 = src_of(k0 + 1), g2 = src_of(k0 + 2), g3 = src_of(k0 + 3);
#pragma unroll
                    for (int s = 0; s < B; ++s) {
                        const double *cj = a + (size_t)(k1 + (s < nb ? s : 0)) * ld;
                        const double u0 = cj[g0];
                        const double u1 = fma(-l10, u0, cj[g1]);
                        const double u2 = fma(-l21, u1, fma(-l20, u0, cj[g2]));
                        const double u3 = fma(-l32, u2, fma(-l31, u1, fma(-l30, u0, cj[g3])));
                        double x = (s < nb && inb) ? cj[srow] : 0.0;
                        if (row >= k1) {
                            x = fma(-cp0, u0, x);
                            x = fma(-cp1, u1, x);
                            x = fma(-cp2, u2, x);
                            x = fma(-cp3, u3, x);
                        }
                        c[s] = x;
                        if (tl == s) { us0 = u0; us1 = u1; us2 = u2; us3 = u3; }
                    }
                } else {
#pragma unroll
                    for (int s = 0; s < B; ++s) c[s] = (s < nb && inb) ? a[(size_t)(k1 + s) * ld + row] : 0.0;
                }
                K6_LAP(5, 0);   // panel load + rank-4 update
                int mypos = row;
                bool live = inb && row >= k1;
                int pvs[B] = {0, 0, 0, 0};
                int fail = -1;
#pragma unroll
                for (int s = 0; s < B; ++s) {
                    if (s < nb && fail < 0) {
                        const int kk = k1 + s;
                        PanelXchg &X = xch[s & 1];
                        // Warp arg-max over its live rows (NaN never wins; first maximum by position):
                        // redux.sync on the high word of |a|; the low word and the position only when
                        // several lanes tie.  The winner publishes |a|, rcp_nr(a), its position and row.
                        const double cs = c[s];
                        const unsigned hi = (unsigned)__double2hiint(cs) & 0x7fffffffu, lo = (unsigned)__double2loint(cs);
                        const bool cand = live && !(hi > 0x7ff00000u || (hi == 0x7ff00000u && lo != 0u));
                        const unsigned khi = cand ? hi + 1u : 0u;
                        double rc = rcp_nr(cs);   // every lane, before the reduction: its latency hides this chain
                        asm volatile("" : "+d"(rc));
                        const unsigned mhi = __reduce_max_sync(FULL, khi);
                        bool top = cand && khi == mhi;
                        unsigned ball = __ballot_sync(FULL, top);
                        if (ball & (ball - 1)) {
                            const unsigned klo = top ? lo : 0u;
                            const unsigned mlo = __reduce_max_sync(FULL, klo);
                            top = top && klo == mlo;
                            ball = __ballot_sync(FULL, top);
                            if (ball & (ball - 1)) {
                                const int mp = __reduce_min_sync(FULL, top ? mypos : INT_MAX);
                                top = top && mypos == mp;
                            }
                        }
                        if (top) {
                            PanelCand &W = X.c[wid];
                            W.vr = make_double2(fabs(cs), rc);
                            W.r01 = make_double2(c[0], c[1]);
                            W.r23 = make_double2(c[2], c[3]);
                            W.pos = mypos;
                        }
                        if (ball == 0u && lane == 0) X.c[wid].vr = make_double2(-1.0, 0.0);
                        if (live && mypos == kk) X.akk = cs;
                        panel_bar(pth);
                        if (s == 0 && K >= 0 && tl < nb) {   // every thread has read the columns: store u
                            double *cj = a + (size_t)(k1 + tl) * ld;
                            cj[k0] = us0; cj[k0 + 1] = us1; cj[k0 + 2] = us2; cj[k0 + 3] = us3;
                        }
                        // best of the four candidates: largest |a|, lowest position among equals (branch-free)
                        const double v0 = wlo <= 0 ? X.c[0].vr.x : -1.0, v1 = (wlo <= 1 && whi >= 1) ? X.c[1].vr.x : -1.0;
                        const double v2 = (wlo <= 2 && whi >= 2) ? X.c[2].vr.x : -1.0, v3 = whi >= 3 ? X.c[3].vr.x : -1.0;
                        const int p0 = X.c[0].pos, p1 = X.c[1].pos, p2 = X.c[2].pos, p3 = X.c[3].pos;
                        const double akk = X.akk;
                        const double m01 = v1 > v0 ? v1 : v0, m23 = v3 > v2 ? v3 : v2;
                        const double bv = m23 > m01 ? m23 : m01;
                        const int e0 = v0 == bv ? p0 : INT_MAX, e1 = v1 == bv ? p1 : INT_MAX;
                        const int e2 = v2 == bv ? p2 : INT_MAX, e3 = v3 == bv ? p3 : INT_MAX;
                        const int bp = min(min(e0, e1), min(e2, e3));
                        const int bw = e0 == bp ? 0 : (e1 == bp ? 1 : (e2 == bp ? 2 : 3));
                        const bool none = !(bv >= 0.0);   // every candidate is NaN: od_lu keeps p = kk (singular)
                        const int pv = none ? kk : bp;
                        const PanelCand &W = X.c[bw];
                        const double2 wvr = W.vr, rp01 = W.r01, rp23 = W.r23;
                        const double rowp[B] = {rp01.x, rp01.y, rp23.x, rp23.y};   // the pivot row in the panel's columns
                        const double piv = rowp[s];
                        // od_lu starts from best = |a_kk|: a NaN there keeps p = kk and the step is singular
                        if (none | !(fabs(piv) > thr) | isnan(akk)) {
                            fail = s;
                        } else {
                            // reciprocal of the winner; 0 (-> IEEE division) outside 2^-400 <= |piv| < 2^401
                            const unsigned epv = ((unsigned)__double2hiint(piv) >> 20) & 0x7ffu;
                            const double r = epv - 623u < 801u ? wvr.y : 0.0;
                            // R-lu's swap of positions kk and pv: the row at kk moves to pv, the pivot row retires to kk
                            const bool isp = live && mypos == pv;
                            if (mypos == kk) mypos = pv;
                            if (isp) { mypos = kk; live = false; }
                            if (live) {   // l = a_ik / piv: PivotDiv's arithmetic with the published reciprocal
                                const double x = c[s];
                                const unsigned ex = ((unsigned)__double2hiint(x) >> 20) & 0x7ffu;
                                const double qa = x * r;
                                double q = fma(fma(-qa, piv, x), r, qa);
                                if (x == 0.0) q = qa;
                                if (!(r != 0.0 && (x == 0.0 || ex - 623u < 801u))) q = ieee_div_cold(x, piv);
                                c[s] = q;
#pragma unroll
                                for (int s2 = s + 1; s2 < B; ++s2) c[s2] = fma(-q, rowp[s2], c[s2]);
                            }
                            pvs[s] = pv;
                        }
                    }
                }
                K6_LAP(6, 0);   // the panel's steps
                // write the panel back: every row to its position (rows >= k1: the panel's U and L
                // parts), and publish the pivots
                if (inb && row >= k1) {
#pragma unroll
                    for (int s = 0; s < B; ++s)
                        if (s < nb) a[(size_t)(k1 + s) * ld + mypos] = c[s];
                }
                if (tl == 0) {
#pragma unroll
                    for (int s = 0; s < B; ++s) {
                        if (s < nb && (fail < 0 || s <= fail)) {
                            const int kk = k1 + s;
                            if (s == fail) { spv[kk] = -1; }
                            else spv[kk] = pvs[s];
                        }
                    }
                }
                continue;
            }
            if (K <= 1) nx_advance(K + 3, p + gridDim.x);   // phases -1, 0, 1: the next star's DoFs, row extents, L2 prefetch
            if (K < 0) continue;
            // ======== update warps ========
            const int uw = wid - K6_PW;
            if (tid == K6_THREADS - 32) {   // the row permutation follows the published pivots (read after the LU)
#pragma unroll
                for (int s = 0; s < B; ++s) {
                    const int kk = k0 + s, pv = pvk[s];
                    if (kk < n && pv != kk) { const int t = prm[kk]; prm[kk] = prm[pv]; prm[pv] = t; }
                }
            }
            // panel K's swaps on the finished L columns to its left (16 columns per warp, lanes over
            // columns); after the trailing update: nothing in this phase waits for them
            auto left_swaps = [&]() {
                const int j = 16 * uw + lane;
                if (lane < 16 && j < k0) {
                    double *cj = a + (size_t)j * ld;
#pragma unroll
                    for (int s = 0; s < B; ++s) {
                        const int A = k0 + s, Bp = pvk[s];
                        if (Bp != A) { const double tA = cj[A], tB = cj[Bp]; cj[A] = tB; cj[Bp] = tA; }
                    }
                }
            };
            if (k1 + B >= n) { left_swaps(); continue; }
            // trailing columns beyond the next panel: a contiguous range per warp
            const int ncol = n - (k1 + B), per = (ncol + K6_UW - 1) / K6_UW;
            const int j0 = k1 + B + uw * per, j1 = min(n, j0 + per);
            K6_LAP(11, 128);   // update thread: phase head (prefetch step, ranges)
            if (j0 + lane < j1) top_rows(a + (size_t)(j0 + lane) * ld);
            __syncwarp();
            K6_LAP(12, 128);   // top rows of its columns
            const double *ck = a + (size_t)k0 * ld;
            auto cols = [&](auto t0c) {
                constexpr int T0 = decltype(t0c)::value;   // chunks < T0 hold only rows < k1
                double l[B][NCH];
                bool act[NCH];
#pragma unroll
                for (int t = T0; t < NCH; ++t) {
                    const int i = lane + 32 * t;
                    act[t] = i >= k1 && i < n;
#pragma unroll
                    for (int s = 0; s < B; ++s) l[s][t] = act[t] ? ck[(size_t)s * ld + i] : 0.0;
                }
#pragma unroll 2
                for (int j = j0; j < j1; ++j) {
                    double *cj = a + (size_t)j * ld;
                    const double u0 = cj[k0], u1 = cj[k0 + 1], u2 = cj[k0 + 2], u3 = cj[k0 + 3];
#pragma unroll
                    for (int t = T0; t < NCH; ++t) {
                        if (act[t]) {
                            const int i = lane + 32 * t;
                            double x = cj[i];
                            x = fma(-l[0][t], u0, x);
                            x = fma(-l[1][t], u1, x);
                            x = fma(-l[2][t], u2, x);
                            x = fma(-l[3][t], u3, x);
                            cj[i] = x;
                        }
                    }
                }
            };
            switch (k1 >> 5) {
                case 0: cols(std::integral_constant<int, 0>{}); break;
                case 1: cols(std::integral_constant<int, NCH >= 2 ? 1 : 0>{}); break;
                case 2: cols(std::integral_constant<int, NCH >= 3 ? 2 : 0>{}); break;
                default: cols(std::integral_constant<int, NCH >= 4 ? 3 : 0>{}); break;
            }
            K6_LAP(13, 128);   // trailing columns
            left_swaps();
            K6_LAP(14, 128);   // left swaps
        }
        if (tid >= 32 * K6_PW) nx_advance(4, p + gridDim.x);
        __syncthreads();
        K6_STAMP(1);
        if (bad) {
            if (tid == 0) atomicMin(status, (int)(p + 1 > INT_MAX - 1 ? INT_MAX - 1 : p + 1));
            __syncthreads();
            continue;
        }
        // packed streaming layout (k2_common.cuh): column pieces are contiguous on both sides
        double *F = fac + foff[p];
        for (int j = wid; j < n; j += NW) {
            const double *cj = a + (size_t)j * ld;
            double *Lf = F + pack_fwd(n, j) - (j + 1);   // l_ij at Lf[i], i > j
            double *Ub = F + pack_bwd(n, j);             // [u_jj, RN(1/u_jj), u_0j .. u_{j-1,j}]
#pragma unroll
            for (int t = 0; t < NCH; ++t) {
                const int i = lane + 32 * t;
                if (i < n) {
                    const double v = cj[i];
                    if (i > j) Lf[i] = v;
                    else if (i < j) Ub[2 + i] = v;
                    else { Ub[0] = v; Ub[1] = 1.0 / v; }
                }
            }
        }
        for (int e = tid; e < n; e += K6_THREADS) {
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
    const int ld = P.max_n | 1;   // odd: lanes over columns (swaps, triangular solves) are conflict-free
    const int nch = (P.max_n + 31) / 32;
    size_t smem = sizeof(double) * (((size_t)P.max_n * ld + 1) & ~(size_t)1) + sizeof(int64_t) * 128 + 2 * sizeof(PanelXchg) +
                  sizeof(int) * (4 * 128 + K6_HASH) + K6_HASH;
    smem = (smem + 15) & ~(size_t)15;
    const int per_sm = smem > 110 * 1024 ? 1 : 2;
    const int64_t cap = (int64_t)sm_count() * per_sm * 4;
    const unsigned g = (unsigned)(P.np < cap ? P.np : cap);
    auto go = [&](auto kern) {
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        kern<<<g, K6_THREADS, smem, s>>>(P.np, P.pn, P.poff, P.foff, P.pdofs, rowptr, col, val, P.fac, P.gidx,
                                         P.perm, status, ld, P.max_n);
    };
    if (nch <= 2) go(k_patch_lu_cm<2>);
    else if (nch == 3) go(k_patch_lu_cm<3>);
    else go(k_patch_lu_cm<4>);
    ++g_launches;
#ifdef MHDP_K6_PROF
    cudaStreamSynchronize(s);
    unsigned long long h[16] = {0};
    cudaMemcpyFromSymbol(h, g_k6prof, sizeof(h));
    fprintf(stderr, "K6 prof np=%lld max_n=%d grid=%u: gather %.3e LU %.3e tail %.3e cycles (sum over CTAs)\n",
            (long long)P.np, P.max_n, g, (double)h[0], (double)h[1], (double)h[2]);
    fprintf(stderr, "   panel thread: top rows %.3e load %.3e steps %.3e rest %.3e barrier wait %.3e | update thread: work %.3e "
            "barrier wait %.3e (head %.3e top rows %.3e columns %.3e left swaps %.3e)\n", (double)h[4], (double)h[5], (double)h[6],
            (double)h[3], (double)h[8], (double)h[9], (double)h[10], (double)h[11], (double)h[12], (double)h[13], (double)h[14]);
    unsigned long long z[16] = {0};
    cudaMemcpyToSymbol(g_k6prof, z, sizeof(z));
#endif
}

}  // namespace mhdp
