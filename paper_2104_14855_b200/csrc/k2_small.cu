// k2_small.cu -- K2 for small stars (2D levels): TMA ring feeding a thread-per-patch
// consumer (see the comment below and DESIGN.md §6.1).  A separate translation unit: its
// fully unrolled per-size instantiations dominate the compile time.
#include "kernels.cuh"
#include "k2_common.cuh"

namespace mhdp {

// ------------------------------------------------------------------------------------
// K2 for small stars (2D levels whose patch sizes all lie in LR_SIZES): one THREAD per
// patch runs the R-lu substitution in registers -- per element exactly the operation
// sequence of the warp kernels (forward z_i = fma(-l_ij, z_j, z_i), j ascending;
// backward z_j = div_rn(z_j, u_jj, 1/u_jj), z_i = fma(-u_ij, z_j, z_i), j descending).
// The 32 patches of a warp have the same size n and their packed streams are interleaved
// element by element (facI[gbase[g] + 32 e + lane]), so a group is one contiguous
// stream; each warp's groups are streamed by TMA bulk copies into a per-warp ring of
// 4 KB chunks (16 elements x 32 lanes), and with n a compile-time constant every
// element's ring offset, chunk wait and chunk release is static.
// ------------------------------------------------------------------------------------
static constexpr int LR_CH = 4096;              // bytes per chunk
static constexpr int LR_CD = LR_CH / 8;         // doubles per chunk
static constexpr int LR_EPC = LR_CD / 32;       // elements per chunk
static constexpr int LR_WARPS = 12, LR_STAGES = 4;
static constexpr size_t LR_SMEM = (size_t)LR_WARPS * LR_STAGES * LR_CH + LR_WARPS * LR_STAGES * 8;

struct GroupProducer {               // per-warp producer of the group streams (lane 0)
    const int *gn;
    const int64_t *gbase;
    const double *facI;
    double *ring;
    uint64_t *bar;
    int64_t ng, W, gg;
    const double *src;
    uint32_t left, issued;
    __device__ __forceinline__ void start(int64_t g) {
        gg = g;
        if (g < ng) {
            const int n = gn[g];
            src = facI + gbase[g];
            left = (uint32_t)(256 * ((int64_t)n * n + n));
        } else {
            left = 0;
        }
    }
    __device__ __forceinline__ void top_up(uint32_t limit) {
        while (issued < limit) {
            if (left == 0) {
                if (gg >= ng) return;
                start(gg + W);
                if (left == 0) return;
            }
            const uint32_t sz = left < (uint32_t)LR_CH ? left : (uint32_t)LR_CH;
            const uint32_t slot = issued & (LR_STAGES - 1);
            mbar_expect_tx(bar + slot, sz);
            bulk_g2s(ring + slot * LR_CD, src, sz, bar + slot);
            src += LR_CD;
            left -= sz;
            ++issued;
        }
    }
};

// element descriptors of the packed stream of an N x N factor, in stream order:
// forward l_ij (z_i -= l_ij z_j), then per column j descending u_jj, 1/u_jj (z_j = q),
// u_ij (z_i -= u_ij q)
enum : uint8_t { LR_FWD = 0, LR_UJJ = 1, LR_RJJ = 2, LR_BWD = 3 };
struct LrOp { uint8_t kind, i, j; };
template <int N>
struct LrOps {
    LrOp op[N * N + N];
    constexpr LrOps() : op() {
        int e = 0;
        for (int j = 0; j < N - 1; ++j)
            for (int i = j + 1; i < N; ++i) op[e++] = LrOp{LR_FWD, (uint8_t)i, (uint8_t)j};
        for (int j = N - 1; j >= 0; --j) {
            op[e++] = LrOp{LR_UJJ, (uint8_t)j, (uint8_t)j};
            op[e++] = LrOp{LR_RJJ, (uint8_t)j, (uint8_t)j};
            for (int i = 0; i < j; ++i) op[e++] = LrOp{LR_BWD, (uint8_t)i, (uint8_t)j};
        }
    }
};

// one group of 32 patches of size N; cb = ring chunk index of the group's first chunk.
// Chunks are walked by an outer loop (one wait and one release each), the elements of a
// chunk by an unrolled inner loop over compile-time descriptors.
template <int N>
__device__ __forceinline__ uint32_t lr_group(int64_t g, const int *__restrict__ gpatch,
                                             const int64_t *__restrict__ poff, const int *__restrict__ gidx,
                                             const double *__restrict__ r, double *__restrict__ y,
                                             const double *ring, uint64_t *bar, uint32_t cb, GroupProducer &prod,
                                             int lane) {
    constexpr int L = N * N + N;
    constexpr int NCH = (L + LR_EPC - 1) / LR_EPC;
    constexpr LrOps<N> ops{};
    const int p = gpatch[32 * g + lane];
    const int64_t off = p >= 0 ? poff[p] : 0;
    double z[N];
#pragma unroll
    for (int i = 0; i < N; ++i) z[i] = p >= 0 ? __ldg(r + __ldg(gidx + off + i)) : 0.0;
    double ujj = 1.0, q = 0.0;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
        const uint32_t k = cb + (uint32_t)c;
        while (!mbar_try(bar + (k & (LR_STAGES - 1)), (k / LR_STAGES) & 1)) {
        }
        const double *src = ring + (k & (LR_STAGES - 1)) * LR_CD + lane;
#pragma unroll
        for (int t = 0; t < LR_EPC; ++t) {
            const int e = c * LR_EPC + t;
            if (e < L) {
                const LrOp o = ops.op[e];
                const double x = src[32 * t];
                if (o.kind == LR_FWD) z[o.i] = fma(-x, z[o.j], z[o.i]);
                else if (o.kind == LR_UJJ) ujj = x;
                else if (o.kind == LR_RJJ) { q = div_rn(z[o.j], ujj, x); z[o.j] = q; }
                else z[o.i] = fma(-x, q, z[o.i]);
            }
        }
        __syncwarp();
        if (lane == 0) {
            fence_proxy_async();
            prod.top_up(k + 1 + LR_STAGES);
        }
    }
    if (p >= 0) {
#pragma unroll
        for (int i = 0; i < N; ++i) y[off + i] = z[i];
    }
    return cb + NCH;
}

__global__ void __launch_bounds__(LR_WARPS * 32, 1) k_patch_apply_lring(int64_t ng, const int *__restrict__ gn,
                                                                        const int64_t *__restrict__ gbase,
                                                                        const int *__restrict__ gpatch,
                                                                        const int64_t *__restrict__ poff,
                                                                        const int *__restrict__ gidx,
                                                                        const double *__restrict__ facI,
                                                                        const double *__restrict__ r,
                                                                        double *__restrict__ y) {
    extern __shared__ __align__(128) double lsm[];
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    double *ring = lsm + (size_t)w * LR_STAGES * LR_CD;
    uint64_t *bar = reinterpret_cast<uint64_t *>(lsm + (size_t)LR_WARPS * LR_STAGES * LR_CD) + w * LR_STAGES;
    if (lane == 0) {
        for (int st = 0; st < LR_STAGES; ++st) mbar_init(bar + st, 1);
        fence_mbar_init();
    }
    __syncwarp();
    const int64_t W = (int64_t)gridDim.x * LR_WARPS;
    const int64_t gw = (int64_t)blockIdx.x * LR_WARPS + w;
    GroupProducer prod;
    prod.gn = gn; prod.gbase = gbase; prod.facI = facI; prod.ring = ring; prod.bar = bar;
    prod.ng = ng; prod.W = W; prod.issued = 0;
    if (lane == 0) {
        prod.start(gw);
        prod.top_up(LR_STAGES);
    }
    uint32_t cb = 0;
    for (int64_t g = gw; g < ng; g += W) {
        switch (gn[g]) {
#define LR_CASE(N) case N: cb = lr_group<N>(g, gpatch, poff, gidx, r, y, ring, bar, cb, prod, lane); break;
            LR_CASE(1) LR_CASE(2) LR_CASE(3) LR_CASE(4) LR_CASE(7) LR_CASE(9) LR_CASE(12) LR_CASE(15) LR_CASE(31)
            LR_CASE(36)
#undef LR_CASE
            default: __trap();
        }
    }
}

bool lring_size_supported(int n) {
    switch (n) {
        case 1: case 2: case 3: case 4: case 7: case 9: case 12: case 15: case 31: case 36: return true;
        default: return false;
    }
}

__global__ void k_interleave(const int *__restrict__ gn, const int64_t *__restrict__ gbase,
                             const int *__restrict__ gpatch, const int64_t *__restrict__ foff,
                             const double *__restrict__ fac, double *__restrict__ facI) {
    const int64_t g = blockIdx.x;
    const int64_t len = 32 * pack_len(gn[g]);
    for (int64_t k = threadIdx.x; k < len; k += blockDim.x) {
        const int lane = (int)(k & 31);
        const int p = gpatch[32 * g + lane];
        facI[gbase[g] + k] = p >= 0 ? fac[foff[p] + (k >> 5)] : 0.0;
    }
}

void launch_interleave(const DevPatches &P, cudaStream_t s) {
    if (P.ng == 0) return;
    k_interleave<<<(unsigned)P.ng, 256, 0, s>>>(P.gn, P.gbase, P.gpatch, P.foff, P.fac, P.facI);
    ++g_launches;
}

void apply_lring(const DevPatches &P, const double *r, cudaStream_t s) {
    static unsigned long long init = 0;
    if (first_use_on_device(init)) {
        cudaFuncSetAttribute(k_patch_apply_lring, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)LR_SMEM);
    }
    const int64_t need = (P.ng + LR_WARPS - 1) / LR_WARPS;
    const int sms = sm_count();
    const unsigned g = (unsigned)(need < sms ? need : sms);
    k_patch_apply_lring<<<g, LR_WARPS * 32, LR_SMEM, s>>>(P.ng, P.gn, P.gbase, P.gpatch, P.poff, P.gidx, P.facI, r,
                                                          P.y);
}


}  // namespace mhdp
