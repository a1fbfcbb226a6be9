#include <cstdio>
#include <cuda_runtime.h>
#define FULL 0xffffffffu
constexpr int TB = 32;
__device__ __forceinline__ double div_rn(double z, double u, double y) {
    const double q = z * y; const double r = fma(-q, u, z); return fma(r, y, q);
}
// chain v3: redundant next-mini-block accs; P = 1 back (division)
template <int P, int PF>
__global__ __launch_bounds__(32) void k(double *out, long long *cyc, int nblk) {
    __shared__ double dt[TB * TB];
    __shared__ __align__(16) double rec[8 * 32];
    const int lane = threadIdx.x & 31;
    for (int e = threadIdx.x; e < TB * TB; e += blockDim.x) dt[e] = 1e-3 * ((e * 7919) % 101);
    for (int e = threadIdx.x; e < 256; e += blockDim.x) rec[e] = (e % 32 >= 22 && e % 32 < 26) ? 2.0 : ((e % 32 >= 26 && e % 32 < 30) ? 0.5 : 1e-3 * (e % 17));
    __syncwarp();
    double acc = 1.0 + lane;
    long long c0 = clock64();
    for (int r = 0; r < nblk; ++r) {
        double zmine = 0;
        double A0 = __shfl_sync(FULL, acc, 0), A1 = __shfl_sync(FULL, acc, 1), A2 = __shfl_sync(FULL, acc, 2), A3 = __shfl_sync(FULL, acc, 3);
#pragma unroll
        for (int mb = 0; mb < 8; ++mb) {
            const int q = 4 * mb;
            const double2 *R = reinterpret_cast<const double2 *>(rec + 32 * mb);
            double B0 = 0, B1 = 0, B2 = 0, B3 = 0;
            const bool more = PF ? true : mb < 7;
            if (more) {
                B0 = __shfl_sync(FULL, acc, (q + 4) & 31); B1 = __shfl_sync(FULL, acc, (q + 5) & 31);
                B2 = __shfl_sync(FULL, acc, (q + 6) & 31); B3 = __shfl_sync(FULL, acc, (q + 7) & 31);
            }
            const double2 e01 = R[0], e23 = R[1], e45 = R[2];
            const double2 n0 = R[3], n1 = R[4], n2 = R[5], n3 = R[6], n4 = R[7], n5 = R[8], n6 = R[9], n7 = R[10];
            const double l0 = dt[q * TB + lane], l1 = dt[(q + 1) * TB + lane], l2 = dt[(q + 2) * TB + lane], l3 = dt[(q + 3) * TB + lane];
            double z0, z1, z2, z3;
            if (P == 0) {
                z0 = A0;
                A1 = fma(-e01.y, z0, A1); z1 = A1;
                A2 = fma(-e23.x, z0, A2); A2 = fma(-e45.x, z1, A2); z2 = A2;
                A3 = fma(-e23.y, z0, A3); A3 = fma(-e45.y, z1, A3); A3 = fma(-e01.x, z2, A3); z3 = A3;
            } else {
                const double2 d01 = R[11], d23 = R[12], y01 = R[13], y23 = R[14];
                z0 = div_rn(A0, d01.x, y01.x);
                A1 = fma(-e01.y, z0, A1); z1 = div_rn(A1, d01.y, y01.y);
                A2 = fma(-e23.x, z0, A2); A2 = fma(-e45.x, z1, A2); z2 = div_rn(A2, d23.x, y23.x);
                A3 = fma(-e23.y, z0, A3); A3 = fma(-e45.y, z1, A3); A3 = fma(-e01.x, z2, A3); z3 = div_rn(A3, d23.y, y23.y);
            }
            if (more) {
                B0 = fma(-n0.x, z0, B0); B1 = fma(-n2.x, z0, B1); B2 = fma(-n4.x, z0, B2); B3 = fma(-n6.x, z0, B3);
                B0 = fma(-n0.y, z1, B0); B1 = fma(-n2.y, z1, B1); B2 = fma(-n4.y, z1, B2); B3 = fma(-n6.y, z1, B3);
                B0 = fma(-n1.x, z2, B0); B1 = fma(-n3.x, z2, B1); B2 = fma(-n5.x, z2, B2); B3 = fma(-n7.x, z2, B3);
                B0 = fma(-n1.y, z3, B0); B1 = fma(-n3.y, z3, B1); B2 = fma(-n5.y, z3, B2); B3 = fma(-n7.y, z3, B3);
            }
            double v = acc;
            v = fma(-l0, z0, v); v = fma(-l1, z1, v); v = fma(-l2, z2, v); v = fma(-l3, z3, v);
            if (lane >= q + 4) acc = v;
            const int sub = lane - q;
            if (sub == 0) zmine = z0;
            if (sub == 1) zmine = z1;
            if (sub == 2) zmine = z2;
            if (sub == 3) zmine = z3;
            A0 = B0; A1 = B1; A2 = B2; A3 = B3;
        }
        acc += zmine * 1e-9;
    }
    long long c1 = clock64();
    if (threadIdx.x == 0) cyc[0] = c1 - c0;
    out[threadIdx.x] = acc;
}
template <int P, int PF> void run(const char *name) {
    double *out; long long *cyc; cudaMalloc(&out, 64 * 8); cudaMalloc(&cyc, 8);
    const int nblk = 2000;
    k<P, PF><<<1, 32>>>(out, cyc, nblk);
    k<P, PF><<<1, 32>>>(out, cyc, nblk);
    long long h; cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s: %.1f cycles per row, %.1f per mini-block\n", name, (double)h / nblk / TB, (double)h / nblk / 8);
}
int main() {
    run<0, 0>("v3 fwd unrolled");
    run<1, 0>("v3 back unrolled");
    run<0, 1>("v3 fwd unrolled branchless");
    run<1, 1>("v3 back unrolled branchless");
    return 0;
}
