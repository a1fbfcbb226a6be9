// k8_coarse.cu -- K8: the coarse solve x = A_0^-1 b of the V-cycle's coarsest level
// (SURVEY 8(c.8) "l = 0: return the coarse LU solve", the stand-in for MUMPS) as
// the R-lu forward / back substitution of SURVEY 8(c.6):
//     z = P b;  forward  z_i <- fma(-l_ij, z_j, z_i)            (j ascending)
//               back     z_j <- z_j / u_jj, then z_i <- fma(-u_ij, z_j, z_i)   (j descending)
// Every z_i receives exactly that sequence of roundings, so the result is bit-identical
// to the oracle's od_lu_solve however the work is spread (reading R-order, c.10).  The
// quotient is formed by div_rn from the stored RN(1/u_jj) (Markstein, k2_common.cuh).
//
// Both passes are a chain of n dependent steps, so the kernel is built around the
// chain's latency, not bandwidth (K8).  Rows are taken in "chain order"
// t (forward: row i = t; back: i = n-1-t) in blocks of 32 rows, so both passes are the
// same lower-triangular recurrence on 32x32 tiles M(t, s), s < t:
//   * CTA 0 holds the chain.  Its NW warps take the row blocks round-robin; the warp of
//     block r lane-per-row applies the recent column blocks J (z from shared memory, as
//     soon as the owning warp publishes them four rows at a time), then solves its own
//     32 rows in mini-blocks of 4: the four partial sums are broadcast by shuffles and
//     every lane solves the 4x4 unit-lower (or, back, upper with division) system
//     redundantly, so one step of the chain costs one DFMA (+ one div_rn) and no
//     communication.  The shuffle that starts the next mini-block is the only hop.
//   * the other CTAs ("far" warps, one row block each) stream the older tiles of their
//     row block from HBM and keep pace with the chain through a global progress counter,
//     stopping LF blocks behind their own block; the chain warp claims the partial sums
//     (hflag / hacc) and finishes the last LF-1 blocks itself.
// Co-residency of all CTAs is required (they wait on each other): cooperative launch.
#include <algorithm>
#include <climits>

#include "k2_common.cuh"
#include "kernels.cuh"

namespace mhdp {

namespace {

constexpr int NW = 8;             // chain warps in CTA 0 (and far warps per far CTA)
constexpr int TB = 32;            // rows per block
constexpr int TILE = TB * TB;     // doubles per tile (column-major: (l, c) at c*32 + l)
constexpr int RING = 4;           // far warps: tiles in flight per warp (TMA ring)
constexpr int RING_WARPS = 4;     // far warps 0..3 of a CTA get a ring (4 x 4 x 8 KB = 128 KB)

__device__ __forceinline__ unsigned long long ld_acq(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
// relaxed probe: the publishing lane only needs to see its predecessor's release before it
// releases in turn (release order is all that matters there; no data is read after it)
__device__ __forceinline__ unsigned long long ld_rlx(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_rel(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void *p, unsigned bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

struct K8Args {
    const double *tiles;     // 2 passes x ntile tiles
    const double *rec;       // per (pass, block, mini-block) 32 coefficients, see k8_pack_rec
    const int *perm;         // R-lu row permutation
    const double *b;
    double *x;               // back z by row (output)
    double *zf;              // forward z by row (global copy for the far warps)
    double *hacc;            // 2 * nb * 32 partial sums handed from far warps to CTA 0
    unsigned long long *sync;   // [0] epoch [1] done [2] prog fwd [3] prog back [4..) hflag
    int n, nb;
    long long ntile;         // nb (nb + 1) / 2
    long long *trace;        // optional (diagnostics): globaltimer stamps, 5 per (pass, block)
    int lf;                  // far warps stop lf >= 2 blocks behind their own row block
};

__device__ __forceinline__ long long gtimer() {
    long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
#define K8_STAMP(p, r, k)                                                     \
    do {                                                                      \
        if (A.trace && lane == 0) A.trace[((p) * A.nb + (r)) * 16 + (k)] = gtimer(); \
    } while (0)

__device__ __forceinline__ const double *tile_ptr(const K8Args &A, int p, int R, int J) {
    return A.tiles + ((long long)p * A.ntile + (long long)R * (R + 1) / 2 + J) * TILE;
}

// own-row entries of tile (r, J): m[c] = M(32r + lane, 32J + c)
__device__ __forceinline__ void load_tile(double (&m)[TB], const double *tp, int lane) {
#pragma unroll
    for (int c = 0; c < TB; ++c) m[c] = __ldcg(tp + c * TB + lane);
}

struct K8Shared {
    double *zs;                 // z by row index (nb * 32)
    double *dt;                 // this warp's diagonal tile
    double *rc;                 // this warp's mini-block records (8 x 32)
    volatile int *vblk;         // blocks of the current pass finalised (CTA 0)
    unsigned long long tgt, base;
    uint64_t *dbar = nullptr;         // chain warps: diagonal tile + records staged
    uint32_t dcount = 0;              // (phase of dbar)
    double *ring = nullptr;           // far warps: RING tile slots in shared memory (or null)
    uint64_t *ring_bar = nullptr;     // their mbarriers
    uint32_t ring_count = 0;          // tiles streamed so far by this warp (slot / phase)
};

// row index of chain position s in pass P (forward: s, back: n-1-s)
template <int P>
__device__ __forceinline__ int row_of(int n, int s) { return P == 0 ? s : n - 1 - s; }

// CTA 0, one pass: the warp of block r (r = w, w + NW, ...) claims its partial sums,
// completes the older column blocks, applies block r-1 as its warp solves it, then
// solves block r in mini-blocks of four rows (see the file comment).
template <int P>
__device__ void chain_pass(const K8Args &A, K8Shared &S, int w, int lane) {
    const int n = A.n, nb = A.nb, LF = A.lf;
    unsigned long long *prog = A.sync + 2, *hflag = A.sync + 4;
    double *zs = S.zs, *dt = S.dt;
    for (int r = w; r < nb; r += NW) {
        const int p = P;
        const int t = r * TB + lane;
        K8_STAMP(p, r, 0);
        const int J0 = r >= LF ? r - LF + 1 : 0;   // first column block applied here
        // everything that does not depend on the partial sums first: tiles J0 .. r toward
        // L2, the diagonal tile and the records to this warp's shared-memory slots, and the
        // first catch-up tile into registers -- then wait for the far warp's hand-off
        {
            const char *pb = reinterpret_cast<const char *>(tile_ptr(A, P, r, J0));
            const int lines = (r - J0 + 1) * (TILE * 8 / 128);
            for (int k = lane; k < lines; k += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 128 * (size_t)k));
            if (lane == 0) {            // diagonal tile + records: two bulk copies, one barrier
                mbar_expect_tx(S.dbar, (TILE + 256) * 8);
                bulk_g2s(dt, tile_ptr(A, P, r, r), TILE * 8, S.dbar);
                bulk_g2s(S.rc, A.rec + ((long long)P * nb + r) * 256, 256 * 8, S.dbar);
            }
        }
        double ma[TB], mb[TB];
        if (J0 < r) load_tile(ma, tile_ptr(A, P, r, J0), lane);
        double acc;
        if (r >= LF) {                  // claim the far warp's partial sums (J <= r - LF)
            while (ld_acq(hflag + P * nb + r) != S.tgt) {}
            acc = __ldcg(A.hacc + ((long long)P * nb + r) * TB + lane);
        } else {
            acc = t < n ? (P == 0 ? __ldg(A.b + __ldg(A.perm + t)) : zs[n - 1 - t]) : 0.0;
        }
        __syncwarp();
        K8_STAMP(p, r, 1);
        // ---- column blocks J0 .. r-2 complete (block granularity), then block r-1 live ----
        if (J0 < r) {
            // complete column blocks J0 .. r-2: tiles alternate between two register buffers
            // (no copy between iterations), the next one's loads in flight while the current
            // one is applied
            long long cw = 0;
            const long long cs = clock64();
            auto wait_blk = [&](int J) {
                if (*S.vblk < J + 1) {
                    const long long w0 = clock64();
                    while (*S.vblk < J + 1) __nanosleep(32);
                    cw += clock64() - w0;
                }
                asm volatile("" ::: "memory");
            };
            int J = J0;
#pragma unroll 1
            while (J < r - 1) {
                load_tile(mb, tile_ptr(A, P, r, J + 1), lane);
                wait_blk(J);
#pragma unroll
                for (int c = 0; c < TB; ++c) acc = fma(-ma[c], zs[row_of<P>(n, TB * J + c)], acc);
                ++J;
                if (J >= r - 1) {
#pragma unroll
                    for (int c = 0; c < TB; ++c) ma[c] = mb[c];
                    break;
                }
                load_tile(ma, tile_ptr(A, P, r, J + 1), lane);
                wait_blk(J);
#pragma unroll
                for (int c = 0; c < TB; ++c) acc = fma(-mb[c], zs[row_of<P>(n, TB * J + c)], acc);
                ++J;
            }
            double (&mc)[TB] = ma;
            K8_STAMP(p, r, 13);
            if (A.trace && lane == 0) {
                A.trace[(P * A.nb + r) * 16 + 14] = cw;
                A.trace[(P * A.nb + r) * 16 + 15] = clock64() - cs;
            }
            // block r-1: eight rows at a time as its warp releases them (named barriers
            // 1 + 4 ((r-1) & 1) + h: the two parities keep the hand-off r-1 -> r apart from
            // r -> r+1, whose consumer may reach its barrier before this one has drained)
            const int bid = 1 + 4 * ((r - 1) & 1);
#pragma unroll
            for (int h = 0; h < 4; ++h) {
                asm volatile("bar.sync %0, 64;" ::"r"(bid + h) : "memory");
#pragma unroll
                for (int c = 0; c < 8; ++c)
                    acc = fma(-mc[8 * h + c], zs[row_of<P>(n, TB * (r - 1) + 8 * h + c)], acc);
            }
        }
        // ---- solve the 32 rows of block r ----
        while (!mbar_try(S.dbar, S.dcount & 1)) {}
        ++S.dcount;
        K8_STAMP(p, r, 2);
        const bool consumer = r + 1 < nb;    // the warp of block r+1 waits on us
        double zmine = 0.0;
        const long long c0 = clock64();
        // every lane holds the four partial sums A of the mini-block being solved, and builds
        // those of the next one (B, shuffled from their owners one mini-block ahead) from the
        // new z's itself -- so no shuffle sits between one mini-block's last z and the next
        // mini-block's first (one DFMA per step forward, DFMA + div_rn back).  Records:
        // rec[0..5] = M(q+1,q) M(q+2,q) M(q+3,q) M(q+2,q+1) M(q+3,q+1) M(q+3,q+2),
        // rec[6 + 4i + c] = M(q+4+i, q+c), rec[22 + a] = u (back), rec[26 + a] = RN(1/u).
        double A0 = __shfl_sync(FULL, acc, 0), A1 = __shfl_sync(FULL, acc, 1);
        double A2 = __shfl_sync(FULL, acc, 2), A3 = __shfl_sync(FULL, acc, 3);
#pragma unroll
        for (int mb = 0; mb < 8; ++mb) {
            const int q = 4 * mb;
            const double *R = S.rc + 32 * mb;
            double B0 = __shfl_sync(FULL, acc, (q + 4) & 31), B1 = __shfl_sync(FULL, acc, (q + 5) & 31);
            double B2 = __shfl_sync(FULL, acc, (q + 6) & 31), B3 = __shfl_sync(FULL, acc, (q + 7) & 31);
            double z0, z1, z2, z3;
            if (P == 0) {
                z0 = A0;
                A1 = fma(-R[0], z0, A1);
                z1 = A1;
                A2 = fma(-R[1], z0, A2);
                A2 = fma(-R[3], z1, A2);
                z2 = A2;
                A3 = fma(-R[2], z0, A3);
                A3 = fma(-R[4], z1, A3);
                A3 = fma(-R[5], z2, A3);
                z3 = A3;
            } else {
                z0 = div_rn(A0, R[22], R[26]);
                A1 = fma(-R[0], z0, A1);
                z1 = div_rn(A1, R[23], R[27]);
                A2 = fma(-R[1], z0, A2);
                A2 = fma(-R[3], z1, A2);
                z2 = div_rn(A2, R[24], R[28]);
                A3 = fma(-R[2], z0, A3);
                A3 = fma(-R[4], z1, A3);
                A3 = fma(-R[5], z2, A3);
                z3 = div_rn(A3, R[25], R[29]);
            }
            // next mini-block's partial sums (rows q+4..q+7), columns in order
            B0 = fma(-R[6], z0, B0);  B1 = fma(-R[10], z0, B1); B2 = fma(-R[14], z0, B2); B3 = fma(-R[18], z0, B3);
            B0 = fma(-R[7], z1, B0);  B1 = fma(-R[11], z1, B1); B2 = fma(-R[15], z1, B2); B3 = fma(-R[19], z1, B3);
            B0 = fma(-R[8], z2, B0);  B1 = fma(-R[12], z2, B1); B2 = fma(-R[16], z2, B2); B3 = fma(-R[20], z2, B3);
            B0 = fma(-R[9], z3, B0);  B1 = fma(-R[13], z3, B1); B2 = fma(-R[17], z3, B2); B3 = fma(-R[21], z3, B3);
            // own row (the same four fma's for lanes q+4..q+7 as B above)
            const double *dl = dt + q * TB + lane;
            double v = acc;
            v = fma(-dl[0], z0, v);
            v = fma(-dl[TB], z1, v);
            v = fma(-dl[2 * TB], z2, v);
            v = fma(-dl[3 * TB], z3, v);
            if (lane >= q + 4) acc = v;
            const int sub = lane - q;
            if (sub == 0) zmine = z0;
            if (sub == 1) zmine = z1;
            if (sub == 2) zmine = z2;
            if (sub == 3) zmine = z3;
            if (sub >= 0 && sub < 4 && t < n) zs[row_of<P>(n, t)] = zmine;
            // release every eight rows to the warp of block r+1 (the barrier arrive orders
            // the stores before it)
            if (consumer && (mb & 1)) asm volatile("bar.arrive %0, 64;" ::"r"(1 + 4 * (r & 1) + (mb >> 1)) : "memory");
            if (A.trace && lane == 0) A.trace[(P * A.nb + r) * 16 + 5 + mb] = clock64() - c0;
            A0 = B0; A1 = B1; A2 = B2; A3 = B3;
        }
        K8_STAMP(p, r, 3);
        if (lane == 0) {                    // block r final for the other warps
            __threadfence_block();
            *S.vblk = r + 1;
        }
        // ---- publish block r to the far warps (in block order) ----
        if (t < n) {
            if (P == 0) A.zf[t] = zmine;
            else A.x[n - 1 - t] = zmine;
        }
        __threadfence();
        __syncwarp();
        if (lane == 0) {
            if (r > 0)
                while (ld_rlx(prog + P) < S.base + (unsigned long long)r) __nanosleep(32);
            st_rel(prog + P, S.base + (unsigned long long)r + 1);
        }
        __syncwarp();
    }
}

// far warps, one pass: row block r >= LF, column blocks 0 .. r-LF, z from global memory as
// the chain publishes it; the partial sums go to hacc / hflag
template <int P>
__device__ void far_pass(const K8Args &A, K8Shared &S, int w, int lane) {
    const int n = A.n, nb = A.nb, LF = A.lf;
    unsigned long long *prog = A.sync + 2, *hflag = A.sync + 4;
    const unsigned long long base = S.base;
    const int G1 = gridDim.x - 1;
    for (int idx = w * G1 + (blockIdx.x - 1); LF + idx < nb; idx += G1 * NW) {
        const int p = P;
        const int r = LF + idx, t = r * TB + lane, Jend = r - LF;
        double acc;
        if (P == 0) {
            acc = t < n ? __ldg(A.b + __ldg(A.perm + t)) : 0.0;
        } else {
            while (ld_acq(prog) < base + (unsigned long long)nb) __nanosleep(128);
            acc = t < n ? __ldcg(A.zf + (n - 1 - t)) : 0.0;
        }
        // z of block J: lane c holds z_{32J+c}.  Up to four completed blocks are fetched per
        // poll (loads in flight together) and the window is refilled one block before it
        // runs dry, so a far warp near the front pays about one progress round trip per
        // batch instead of two round trips per block.
        const double *zsrc = P == 0 ? A.zf : A.x;
        auto zaddr = [&](int J) { return zsrc + row_of<P>(n, TB * J + lane); };
        long long done = 0;                       // blocks known complete (all lanes)
        auto poll = [&]() {
            const unsigned long long v = ld_acq(prog + P);
            const long long d = v >= base ? (long long)(v - base) : 0;
            return (long long)__reduce_min_sync(FULL, (unsigned)min(d, (long long)nb));
        };
        double z0 = 0.0, z1 = 0.0, z2 = 0.0, z3 = 0.0;   // window: blocks J .. J+have-1
        int have = 0, nxt = 0;                    // nxt: first block not yet fetched
        auto refill = [&](bool block_until) {
            if (done <= nxt) done = poll();
            while (block_until && done <= nxt) done = poll();
            const int cnt = (int)min((long long)(4 - have), min(done, (long long)Jend + 1) - nxt);
            // append cnt blocks behind the `have` already held
            for (int k = 0; k < cnt; ++k) {
                const double zv = __ldcg(zaddr(nxt + k));
                const int slot = have + k;
                if (slot == 0) z0 = zv;
                else if (slot == 1) z1 = zv;
                else if (slot == 2) z2 = zv;
                else z3 = zv;
            }
            if (cnt > 0) { have += cnt; nxt += cnt; }
        };
        // the row block's tiles 0 .. Jend are one contiguous stream: warps with a ring slot
        // set (RING slots of 8 KB in the far CTA's shared memory) stream them with TMA bulk
        // copies RING tiles ahead; the others double-buffer them in registers
        const bool ring = S.ring != nullptr;
        double mc[TB], mn[TB];
        if (ring) {
            if (lane == 0)
                for (int J = 0; J < RING && J <= Jend; ++J) {
                    const uint32_t slot = (S.ring_count + J) % RING;
                    mbar_expect_tx(S.ring_bar + slot, TILE * 8);
                    bulk_g2s(S.ring + slot * TILE, tile_ptr(A, P, r, J), TILE * 8, S.ring_bar + slot);
                }
        } else {
            if (lane == 0) prefetch_l2(tile_ptr(A, P, r, 0), (unsigned)(min(Jend + 1, 4) * TILE * 8));
            load_tile(mc, tile_ptr(A, P, r, 0), lane);
        }
#pragma unroll 1
        for (int J = 0; J <= Jend; ++J) {
            if (ring) {
                const uint32_t cnt = S.ring_count + J, slot = cnt % RING;
                while (!mbar_try(S.ring_bar + slot, (cnt / RING) & 1)) {}
                const double *src = S.ring + slot * TILE;
#pragma unroll
                for (int c = 0; c < TB; ++c) mc[c] = src[c * TB + lane];
                __syncwarp();
                if (lane == 0 && J + RING <= Jend) {     // refill the slot just read
                    fence_proxy_async();
                    mbar_expect_tx(S.ring_bar + slot, TILE * 8);
                    bulk_g2s(S.ring + slot * TILE, tile_ptr(A, P, r, J + RING), TILE * 8, S.ring_bar + slot);
                }
            } else {
                if (J + 1 <= Jend) load_tile(mn, tile_ptr(A, P, r, J + 1), lane);
                if (lane == 0 && J + 4 <= Jend) prefetch_l2(tile_ptr(A, P, r, J + 4), TILE * 8);
            }
            if (J + 2 == Jend || (Jend < 2 && J == 0)) {
                // the chain CTA's warp finishes this row block with tiles Jend+1 .. r: warm
                // them in L2 now, shortly before it needs them
                const char *pb = reinterpret_cast<const char *>(tile_ptr(A, P, r, Jend + 1));
                const int lines = (r - Jend) * (TILE * 8 / 128);
                for (int k = lane; k < lines; k += 32) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + 128 * (size_t)k));
            }
            if (have == 0) refill(true);
            else if (have == 1 && nxt <= Jend) refill(false);
            const double zj = z0;
#pragma unroll
            for (int c = 0; c < TB; ++c) acc = fma(-mc[c], __shfl_sync(FULL, zj, c), acc);
            if (!ring) {
#pragma unroll
                for (int c = 0; c < TB; ++c) mc[c] = mn[c];
            }
            z0 = z1; z1 = z2; z2 = z3;
            --have;
        }
        if (ring) S.ring_count += Jend + 1;
        A.hacc[((long long)P * nb + r) * TB + lane] = acc;
        __threadfence();
        __syncwarp();
        K8_STAMP(p, r, 4);
        if (lane == 0) st_rel(hflag + P * nb + r, S.tgt);
        __syncwarp();
    }
}

__global__ void __launch_bounds__(NW * 32, 1) k8_solve(K8Args A) {
    extern __shared__ __align__(128) double sm[];
    __shared__ int s_prog;
    __shared__ unsigned long long s_tgt;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_tgt = *(volatile unsigned long long *)A.sync + 1;
    __syncthreads();
    K8Shared S;
    S.zs = sm;
    S.dt = sm + (size_t)A.nb * TB + w * TILE;
    S.rc = sm + (size_t)A.nb * TB + NW * TILE + w * 256;
    S.vblk = &s_prog;
    S.tgt = s_tgt;
    S.base = s_tgt << 10;   // nb <= 1023
    if (blockIdx.x == 0) {
        __shared__ uint64_t dbar[NW];
        S.dbar = dbar + w;
        if (lane == 0) {
            mbar_init(S.dbar, 1);
            fence_mbar_init();
        }
        if (threadIdx.x == 0) s_prog = 0;
        __syncthreads();
        chain_pass<0>(A, S, w, lane);
        __syncthreads();
        if (threadIdx.x == 0) s_prog = 0;
        __syncthreads();
        chain_pass<1>(A, S, w, lane);
    } else {
        __shared__ uint64_t ring_bar[RING_WARPS * RING];
        if (w < RING_WARPS) {
            S.ring = sm + (size_t)w * RING * TILE;
            S.ring_bar = ring_bar + w * RING;
            if (lane == 0) {
                for (int k = 0; k < RING; ++k) mbar_init(S.ring_bar + k, 1);
                fence_mbar_init();
            }
            __syncwarp();
        }
        far_pass<0>(A, S, w, lane);
        far_pass<1>(A, S, w, lane);
    }
    // ---- epoch: the last CTA to finish advances it (the next launch waits for tgt + 1) ----
    __syncthreads();
    if (threadIdx.x == 0) {
        __threadfence();
        const unsigned long long d = atomicAdd(A.sync + 1, 1ULL);
        if (d == gridDim.x - 1) {
            A.sync[1] = 0;
            __threadfence();
            st_rel(A.sync, S.tgt);
        }
    }
}

// tiles of both passes from the row-major R-lu factors
__global__ void k8_pack(const double *__restrict__ a, int n, int nb, long long ntile, double *__restrict__ tiles) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long per = ntile * TILE;
    if (e >= 2 * per) return;
    const int p = (int)(e / per);
    const long long rem = e - p * per, tidx = rem / TILE;
    const int q = (int)(rem % TILE), c = q / TB, l = q % TB;
    int R = (int)((sqrt(8.0 * (double)tidx + 1.0) - 1.0) * 0.5);
    while ((long long)R * (R + 1) / 2 > tidx) --R;
    while ((long long)(R + 1) * (R + 2) / 2 <= tidx) ++R;
    const int J = (int)(tidx - (long long)R * (R + 1) / 2);
    const int t = R * TB + l, s = J * TB + c;
    double v = 0.0;
    if (t < n && s < n) {
        if (p == 0) {
            if (s < t) v = a[(long long)t * n + s];
        } else if (s <= t) {
            v = a[(long long)(n - 1 - t) * n + (n - 1 - s)];
        }
    }
    tiles[e] = v;
}

// M(t, s) of pass p in chain order (forward: strictly lower L; back: U incl. diagonal)
__device__ __forceinline__ double chain_m(const double *a, int n, int p, int t, int s) {
    if (t >= n || s >= n) return 0.0;
    if (p == 0) return s < t ? a[(long long)t * n + s] : 0.0;
    return s <= t ? a[(long long)(n - 1 - t) * n + (n - 1 - s)] : 0.0;
}

// mini-block records: per (pass, block, mini-block) 32 doubles, layout in chain_pass
__global__ void k8_pack_rec(const double *__restrict__ a, int n, int nb, double *__restrict__ rec) {
    const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= 2LL * nb * 256) return;
    const int k = (int)(e % 32), mb = (int)((e / 32) % 8);
    const int R = (int)((e / 256) % nb), p = (int)(e / (256LL * nb));
    const int t0 = R * TB + 4 * mb;
    double v = 0.0;
    if (k < 6) {
        const int ra[6] = {1, 2, 3, 2, 3, 3}, ca[6] = {0, 0, 0, 1, 1, 2};
        v = chain_m(a, n, p, t0 + ra[k], t0 + ca[k]);
    } else if (k < 22) {
        const int i = (k - 6) / 4, c = (k - 6) % 4;
        if (mb < 7) v = chain_m(a, n, p, t0 + 4 + i, t0 + c);
    } else if (k < 26) {
        if (p == 1) v = chain_m(a, n, p, t0 + k - 22, t0 + k - 22);
    } else if (k < 30) {
        if (p == 1) {
            const double u = chain_m(a, n, p, t0 + k - 26, t0 + k - 26);
            v = u != 0.0 ? 1.0 / u : 0.0;   // RN(1/u), IEEE division
        }
    }
    rec[e] = v;
}

}  // namespace

// far-warp lag in blocks, measured on the c5 coarse level (n0 = 7128, tools/k8_trace.py,
// profiles/r02_k8_trace_summary.txt): 6 -> 0.585 ms, 7 -> 0.561, 8 -> 0.593, 9 -> 0.620
int k8_lf() { return 7; }

int k8_max_n() {
    // shared memory: z (nb*32) + NW diagonal tiles and records, within 227 KB
    return (227 * 1024 / 8 - NW * (TILE + 256)) / TB * TB;
}

int64_t k8_tile_doubles(int n) {
    const int64_t nb = (n + TB - 1) / TB;
    return 2 * (nb * (nb + 1) / 2) * TILE;
}

int64_t k8_sync_words(int n) { return 4 + 2 * (int64_t)((n + TB - 1) / TB); }

int64_t k8_rec_doubles(int n) { return 2 * 256 * (int64_t)((n + TB - 1) / TB); }

void launch_k8_pack(const double *lu_rowmajor, int n, double *tiles, double *rec, cudaStream_t s) {
    if (n == 0) return;
    const int nb = (n + TB - 1) / TB;
    const long long ntile = (long long)nb * (nb + 1) / 2;
    const long long tot = 2 * ntile * TILE;
    k8_pack<<<(unsigned)((tot + 255) / 256), 256, 0, s>>>(lu_rowmajor, n, nb, ntile, tiles);
    k8_pack_rec<<<(unsigned)((2LL * nb * 256 + 255) / 256), 256, 0, s>>>(lu_rowmajor, n, nb, rec);
    g_launches += 2;
}

// b and x must not alias; zf: nb*32 doubles; hacc: 2*nb*32 doubles; sync: k8_sync_words
// (zero-initialised once at setup; the kernel keeps it consistent from call to call)
cudaError_t launch_k8_solve(const double *tiles, const double *rec, const int *perm, int n, const double *b,
                            double *x, double *zf, double *hacc, unsigned long long *sync, cudaStream_t s,
                            long long *trace) {
    if (n == 0) return cudaSuccess;
    const int nb = (n + TB - 1) / TB;
    K8Args A;
    A.tiles = tiles; A.rec = rec; A.perm = perm; A.b = b; A.x = x; A.zf = zf; A.hacc = hacc; A.sync = sync;
    A.n = n; A.nb = nb; A.ntile = (long long)nb * (nb + 1) / 2; A.trace = trace;
    const size_t smem = std::max(sizeof(double) * ((size_t)nb * TB + NW * (TILE + 256)),
                                 sizeof(double) * (size_t)RING_WARPS * RING * TILE);
    int dev = 0;
    cudaGetDevice(&dev);
    cudaFuncSetAttribute(k8_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    A.lf = k8_lf();
    const int far_blocks = nb > A.lf ? nb - A.lf : 0;
    const int G = 1 + std::min(sms - 1, far_blocks);
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(NW * 32);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    ++g_launches;
    return cudaLaunchKernelEx(&cfg, k8_solve, A);
}

}  // namespace mhdp
