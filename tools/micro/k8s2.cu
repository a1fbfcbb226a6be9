#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
constexpr int TB = 32;
__device__ __forceinline__ double div_rn(double z, double u, double y) {
    const double q = z * y; const double r = fma(-q, u, z); return fma(r, y, q);
}
// chain with mini-blocks of 2 rows: record per mini-block [e10, N00, N01, N10, N11, d0, d1, y0, y1] (+pad)
template <int P>
__global__ void __launch_bounds__(32) k(double *out, long long *cyc, int nblk) {
    __shared__ double dt[TB * TB];
    __shared__ __align__(16) double rec[16 * 16];
    const int lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) dt[e] = 1e-3 * ((e * 7919) % 101);
    for (int e = threadIdx.x; e < 256; e += blockDim.x) rec[e] = (e % 16 == 5 || e % 16 == 6) ? 2.0 : ((e % 16 == 7 || e % 16 == 8) ? 0.5 : 1e-3 * (e % 17));
    __syncwarp();
    double acc = 1.0 + lane;
    long long c0 = clock64();
    for (int r = 0; r < nblk; ++r) {
        double zmine = 0;
        double A0 = __shfl_sync(FULL, acc, 0), A1 = __shfl_sync(FULL, acc, 1);
#pragma unroll
        for (int mb = 0; mb < 16; ++mb) {
            const int q = 2 * mb;
            const double *R = rec + 16 * mb;
            double B0 = __shfl_sync(FULL, acc, (q + 2) & 31), B1 = __shfl_sync(FULL, acc, (q + 3) & 31);
            double z0, z1;
            if (P == 0) { z0 = A0; A1 = fma(-R[0], z0, A1); z1 = A1; }
            else { z0 = div_rn(A0, R[5], R[7]); A1 = fma(-R[0], z0, A1); z1 = div_rn(A1, R[6], R[8]); }
            B0 = fma(-R[1], z0, B0); B1 = fma(-R[3], z0, B1);
            B0 = fma(-R[2], z1, B0); B1 = fma(-R[4], z1, B1);
            const double *dl = dt + q * TB + lane;
            double v = acc;
            v = fma(-dl[0], z0, v); v = fma(-dl[TB], z1, v);
            if (lane >= q + 2) acc = v;
            if (lane == q) zmine = z0;
            if (lane == q + 1) zmine = z1;
            A0 = B0; A1 = B1;
        }
        acc += zmine * 1e-9;
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
    out[threadIdx.x] = acc;
}
template <int P> void run(const char *name) {
    double *out; long long *cyc; cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 8);
    const int nblk = 2000;
    k<P><<<1, 32>>>(out, cyc, nblk); k<P><<<1, 32>>>(out, cyc, nblk);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s: %.1f cycles per row\n", name, (double)h / nblk / TB);
}
int main() { run<0>("S2 fwd"); run<1>("S2 back"); return 0; }
